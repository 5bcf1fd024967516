#!/bin/bash
# ncu --set full of the trilinear apply kernel at cfg5 shape (8^3 mesh keeps setup short; the
# kernel's per-cell work is the same). Usage under gpurun: bash scripts/ncu_tri.sh NAME [MESH]
NAME=${1:-tri}; MESH=${2:-8}
mkdir -p gpurun_out
CMD="python bench.py --config 5 --mesh $MESH --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:apply_tri -s 3 -c 1 -o gpurun_out/prof_$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1
tail -1 gpurun_out/ncu_$NAME.log
