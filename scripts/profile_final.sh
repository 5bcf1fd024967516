#!/bin/bash
# Final round evidence (1 GPU): default bench line (cfg2, full contract), cfg5 line, reference
# arm, launch lists of both configs and --set full captures of the dominant kernels.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg2.log 2>&1; tail -1 gpurun_out/bench_cfg2.log > gpurun_out/bench_cfg2.json
python bench.py --config 5 > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log > gpurun_out/bench_cfg5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
for c in 2 5; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > gpurun_out/plain_cfg$c.log 2>&1 || continue
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > /dev/null 2>&1
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:patch_stream -s 2 -c 1 -o gpurun_out/prof_patch_cfg$c $CMD > /dev/null 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:apply_tri -s 3 -c 1 -o gpurun_out/prof_apply_tri_cfg5 \
  python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
