# A/B of an environment knob on one box: bash /tmp/abenv.sh VAR "v1 v2" "c2 c3" reps
var=$1; vals=$2; cfgs=$3; reps=${4:-1}
mkdir -p gpurun_out/ab
for i in $(seq $reps); do for c in $cfgs; do for v in $vals; do
  env $var=$v timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-mb --no-asm > gpurun_out/ab/env_${v}_${c}_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab/env_${v}_${c}_$i.json')); print('$var=$v $c $i', round(d['value'],1), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms'],4), 'solve ms/it', round(d['solve']['ms_per_iteration'],3))"
done; done; done
