#!/bin/bash
# Round-2 final GPU evidence session (after the MB-mode and LU changes): bench lines
# (c2 default, c3, c5 n=20, c4, reference arm), the ncu launch list of the default
# bench, ncu --set full summaries of the element kernel (apply and MB modes), the MB
# form kernel and the tile LU, LU probes of the three LU kernels.
#   gpurun --timeout 3600 -- 'bash tools/profile_round2b.sh'
out=gpurun_out/prof2b
mkdir -p $out
python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in c3 c5n20 c4; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-asm > $out/bench_$c.json 2> $out/bench_$c.err
done
python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_c2_reference.json 2> $out/bench_c2_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv \
  python bench.py --steps 5 --warmup 3 --warmup-seconds 0 --no-cpu-baseline --no-asm > $out/ncu_launch.log 2>&1
NB="--steps 3 --warmup 3 --warmup-seconds 0 --no-cpu-baseline --no-asm"
ncu --set full --import-source on --clock-control none -k regex:element_kernel -s 1 -c 1 \
  -o $out/element_c2 python bench.py $NB --no-mb > $out/ncu_el.log 2>&1
for c in c2 c3 c5n20 c4; do
  ncu --set full --import-source on --clock-control none -k regex:form_dmma -s 1 -c 1 \
    -o $out/form_$c python bench.py --config $c $NB > $out/ncu_form_$c.log 2>&1
done
for c in c2 c5n20; do
  ncu --set full --import-source on --clock-control none -k "regex:element_kernel<[0-9], 3" -s 2 -c 1 \
    -o $out/mbapply_$c python bench.py --config $c $NB > $out/ncu_mb_$c.log 2>&1
done
for c in c2 c5n20; do
  ncu --set full --import-source on --clock-control none -k regex:lu_tile -c 1 \
    -o $out/lu_tile_$c python tools/lu_probe.py $c 1 > $out/ncu_lu_$c.log 2>&1
done
for c in c2 c3 c5n20 c4; do for v in tile cta pipe; do MEHDG_LU=$v python tools/lu_probe.py $c 4 2>&1 | tail -1 | sed "s/^/$v /" >> $out/lu_probe.txt; done; done
for r in $out/*.ncu-rep; do
  python tools/ncu_hot.py $r "" 30 > ${r%.ncu-rep}_hot.txt 2>&1
  python profiles/ncu_summary.py $r 0 > ${r%.ncu-rep}_sum.txt 2>&1
done
find $out -name "*.ncu-rep" -delete
ls -la $out
