#!/bin/bash
# round-2 pass Z: cfg5 after the sc_post 32-bit decode -- cfg5 parity, cfg5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg5" > gpurun_out/gpu_z.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_z.log
timeout 600 python bench.py --config 5 --secondary 0 --no-cpu-baseline --no-e2e > gpurun_out/bench5.log 2>&1; tail -1 gpurun_out/bench5.log > gpurun_out/bench5.json
echo done
