#!/bin/bash
# One GPU session of round evidence: bench lines for c2..c5, the ncu launch list of
# the default bench, and ncu --set full captures of the top kernels.
#   gpurun --timeout 3000 -- 'bash tools/profile_round.sh'
out=gpurun_out/prof
mkdir -p $out
python bench.py > $out/bench_c2.json 2> $out/bench_c2.err
for c in c3 c5n20 c4; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-mb --no-asm > $out/bench_$c.json 2> $out/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-mb --no-asm > $out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k element_kernel -s 1 -c 1 \
  -o $out/element_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-mb --no-asm > $out/ncu_el.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"face_small|face_reduce" -c 2 \
  -o $out/face_c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-mb --no-asm > $out/ncu_face.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:lu_tile -c 1 \
  -o $out/lu_c2 python tools/lu_probe.py c2 1 > $out/ncu_lu.log 2>&1
ncu --set full --import-source on --clock-control none -k element_kernel -s 1 -c 1 \
  -o $out/element_c3 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-mb --no-asm > $out/ncu_el3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:assemble_macro -c 1 \
  -o $out/assembly python tools/asm_probe.py 128 2 3 1 > $out/ncu_asm.log 2>&1
python tools/asm_probe.py 128 2 3 3 > $out/asm_probe.txt 2>&1
for c in c2 c3 c5n20; do python tools/lu_probe.py $c 4 >> $out/lu_probe.txt 2>&1; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu && ./tools/fp64_peak > $out/fp64_peak.txt 2>&1
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back);
# only the element-kernel c2 report travels back
for r in $out/*.ncu-rep; do
  python tools/ncu_hot.py $r "" 30 > ${r%.ncu-rep}_hot.txt 2>&1
  python profiles/ncu_summary.py $r 0 > ${r%.ncu-rep}_sum.txt 2>&1
  ncu -i $r --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > ${r%.ncu-rep}_dram.csv 2>/dev/null
done
find $out -name "*.ncu-rep" ! -name element_c2.ncu-rep -delete
ls -la $out
