#!/bin/bash
# A/B of library builds on one box: tools/ab_bench.sh "base u32" "c2 c3" [reps]
# (libmehdg_b200.<v>.so, "base" = libmehdg_b200.so); prints value / element GB/s per run
vars=$1; cfgs=$2; reps=${3:-2}
mkdir -p gpurun_out/ab
for i in $(seq $reps); do for c in $cfgs; do for v in $vars; do
  if [ "$v" = base ]; then unset MEHDG_LIB_VARIANT; else export MEHDG_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-mb --no-asm \
    > gpurun_out/ab/${v}_${c}_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab/${v}_${c}_$i.json')); print('$v $c $i', round(d['value'],1), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms'],4))"
done; done; done
