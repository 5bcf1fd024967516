#!/bin/bash
# round-2 pass K: k = 0 pointwise-stage apply (Cartesian) -- parity suite, cfg2 bench, cfg2 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --config 2 --secondary 0 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; tail -1 gpurun_out/bench2.log > gpurun_out/bench2.json
RM_APPLY_COLOURS=1 timeout 600 python bench.py --config 2 --secondary 0 --no-cpu-baseline > gpurun_out/bench2c.log 2>&1; tail -1 gpurun_out/bench2c.log > gpurun_out/bench2c.json
CMD="python bench.py --config 2 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_q_pw -s 2 -c 1 -o gpurun_out/prof_applyq_cfg2 $CMD > gpurun_out/ncu_a2.log 2>&1
echo done
