#!/bin/bash
# round-2 pass U: ncu of the cfg2 k = 0 apply (one launch) and the skeleton gather
mkdir -p gpurun_out
CMD="python bench.py --config 2 --secondary 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"apply_q_kernel|tri_gather_sc" -s 2 -c 2 -o gpurun_out/prof_apply_q_cfg2 $CMD > gpurun_out/ncu_q.log 2>&1
echo done
