#!/bin/bash
# pass AO: ncu --set full with source of the class-batched kernel (cfg4 NCE8 edge-star potential family)
mkdir -p gpurun_out
C4="python bench.py --config 4 --secondary 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_batch -s 26 -c 1 -o gpurun_out/prof_batch_cfg4_ao $C4 > gpurun_out/ao_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
echo done
