#!/bin/bash
# round-2 pass W: out-of-place combine (no u copy), full suite, default bench, cfg3/cfg4 bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
echo done
