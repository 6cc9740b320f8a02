#!/bin/bash
# Round-2 GPU evidence session: bench lines (c2 default, c3, c5 n=20, c4), the ncu
# launch list of the default bench, and ncu --set full summaries of the top kernels.
#   gpurun --timeout 3600 -- 'bash tools/profile_round2.sh'
out=gpurun_out/prof2
mkdir -p $out
python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in c3 c5n20 c4; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-mb --no-asm > $out/bench_$c.json 2> $out/bench_$c.err
done
python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_c2_reference.json 2> $out/bench_c2_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv \
  python bench.py --steps 5 --warmup 3 --warmup-seconds 0 --no-cpu-baseline --no-mb --no-asm > $out/ncu_launch.log 2>&1
NB="--steps 3 --warmup 3 --warmup-seconds 0 --no-cpu-baseline --no-mb --no-asm"
ncu --set full --import-source on --clock-control none -k element_kernel -s 1 -c 1 \
  -o $out/element_c2 python bench.py $NB > $out/ncu_el.log 2>&1
for c in c3 c5n20 c4; do
  ncu --set full --import-source on --clock-control none -k element_kernel -s 1 -c 1 \
    -o $out/element_$c python bench.py --config $c $NB > $out/ncu_el_$c.log 2>&1
done
for c in c5n20 c4; do
  ncu --set full --import-source on --clock-control none -k regex:face_bulk -c 1 \
    -o $out/face_$c python bench.py --config $c $NB > $out/ncu_face_$c.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:lu_tile -c 1 \
  -o $out/lu_tile_c5n20 python tools/lu_probe.py c5n20 1 > $out/ncu_lu.log 2>&1
MEHDG_LU=cta ncu --set full --import-source on --clock-control none -k regex:lu_cta -c 1 \
  -o $out/lu_cta_c5n20 python tools/lu_probe.py c5n20 1 > $out/ncu_lucta.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/gmres_c2.csv python tools/gmres_probe.py c2 > $out/ncu_gmres.log 2>&1
for c in c2 c3 c5n20; do MEHDG_GMRES_TRACE=1 python tools/gmres_probe.py $c >> $out/gmres_probe.txt 2>&1; done
for c in c2 c3 c5n20; do for v in tile cta; do MEHDG_LU=$v python tools/lu_probe.py $c 4 >> $out/lu_probe.txt 2>&1; done; done
for r in $out/*.ncu-rep; do
  python tools/ncu_hot.py $r "" 30 > ${r%.ncu-rep}_hot.txt 2>&1
  python profiles/ncu_summary.py $r 0 > ${r%.ncu-rep}_sum.txt 2>&1
  ncu -i $r --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > ${r%.ncu-rep}_dram.csv 2>/dev/null
done
find $out -name "*.ncu-rep" -delete
ls -la $out
