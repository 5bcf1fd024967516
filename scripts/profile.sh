#!/bin/bash
# ncu evidence for the bench workload (B200_PROFILING.md recipe). Run under gpurun.
set -e
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:patch_solve -s 20 -c 1 -o gpurun_out/prof_patch $CMD > gpurun_out/ncu_patch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_q -s 20 -c 1 -o gpurun_out/prof_apply $CMD > gpurun_out/ncu_apply.log 2>&1
echo done
