#!/bin/bash
# ncu evidence for the bench command: launch list (all launches, serialised) + one --set full
# capture of K4, K5, K6 of one step.  Plain runs first (ncu only after an exit-0 plain run).
set -e
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-classical --no-variants"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/prof_launch.log 2>&1
CMD1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-classical --no-variants"
$CMD1 > gpurun_out/prof_plain1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"premix|leaf|postmix" -c 4 -o gpurun_out/prof_full -f $CMD1 > gpurun_out/prof_full.log 2>&1
echo done
