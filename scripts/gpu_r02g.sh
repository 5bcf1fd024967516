#!/bin/bash
# round-2 pass G: compressed static-condensation couplings (cfg5): parity subset, default bench, launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg5 or sc or trilinear or slab" > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
CMD="python bench.py --config 5 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch5.log 2>&1
echo done
