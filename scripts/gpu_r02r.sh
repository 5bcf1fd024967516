#!/bin/bash
# round-2 pass R: ncu of the cfg5 memory-bound kernels around the patch solve (SC pre / post, gather, combine)
mkdir -p gpurun_out
CMD="python bench.py --config 5 --secondary 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sc_cell|sc_face|sc_post|tri_gather|unpad" -s 5 -c 5 -o gpurun_out/prof_sc_cfg5 $CMD > gpurun_out/ncu_sc.log 2>&1
echo done
