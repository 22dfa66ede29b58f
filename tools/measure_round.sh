#!/bin/bash
# Round measurement: every bench config, the reference arm, the ncu launch list of
# the default bench command and one full ncu capture of each dominant kernel.
# Usage (under gpurun): bash tools/measure_round.sh <outdir under gpurun_out>
out=${1:-gpurun_out/round}
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > $out/gpu.csv
for c in box2d heat2d star2d heat3d box3d box3d1024; do
  timeout 600 python bench.py --config $c --no-sweep > $out/bench_$c.json 2> $out/bench_$c.err
done
timeout 300 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_box2d.csv \
  python bench.py --no-sweep --steps 8 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 1 -c 1 \
  -o $out/prof_box2d python bench.py --no-sweep --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d -s 1 -c 1 \
  -o $out/prof_box3d python bench.py --no-sweep --config box3d --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 1 -c 1 \
  -o $out/prof_star2d python bench.py --no-sweep --config star2d --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_step -s 1 -c 1 \
  -o $out/prof_heat2d python bench.py --no-sweep --config heat2d --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
# (each capture: launch 1 of the warm-up run = a steady binary16 launch, binary16 in and out)
# summaries on the box (gpurun copies back at most 64 MiB: the .ncu-rep files would exceed it)
for k in box2d box3d star2d heat2d; do
  python tools/ncu_summary.py $out/prof_$k.ncu-rep > $out/ncu_${k}_full.txt 2>&1
  python tools/ncu_smem.py $out/prof_$k.ncu-rep 20 > $out/smem_${k}.txt 2>&1
done
rm -f $out/*.ncu-rep
