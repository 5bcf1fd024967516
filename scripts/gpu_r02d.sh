#!/bin/bash
# round-2 pass D: full parity suite, eps study, all bench lines, launch lists, ncu --set full captures
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python scripts/eps_study.py > gpurun_out/eps_study.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
for c in 5 2; do
  CMD="python bench.py --config $c --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_launch$c.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:patch_stream -s 2 -c 1 -o gpurun_out/prof_patch_cfg$c $CMD > gpurun_out/ncu_patch$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_tri -s 3 -c 1 -o gpurun_out/prof_apply_tri_cfg5 \
  python bench.py --config 5 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tri.log 2>&1
echo done
