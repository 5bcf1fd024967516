#!/bin/bash
# ncu evidence for the bench workload (B200_PROFILING.md recipe). Run under gpurun, 1 GPU.
# 1) plain run (must exit 0), 2) launch list with per-launch durations (cold, serialised),
# 3) one --set full capture of the patch kernel and of the apply kernel.
set -e
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:patch_stream -s 2 -c 1 -o gpurun_out/prof_patch $CMD > gpurun_out/ncu_patch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_q -s 20 -c 1 -o gpurun_out/prof_apply $CMD > gpurun_out/ncu_apply.log 2>&1
echo done
