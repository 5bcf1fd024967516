#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config 4 --secondary 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_batch -s 8 -c 1 -o gpurun_out/prof_batch_cfg4 $CMD > gpurun_out/ncu_b4.log 2>&1
echo done
