#!/bin/bash
# round-2 pass I: balanced even/odd pointwise slots; trilinear parity subset, cfg5 bench, launch list, ncu
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg5 or trilinear" > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --secondary 0 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
CMD="python bench.py --config 5 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_tri -s 3 -c 1 -o gpurun_out/prof_apply_tri_cfg5 $CMD > gpurun_out/ncu_tri.log 2>&1
echo done
