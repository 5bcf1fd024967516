#!/bin/bash
# round-2 pass AD: 5 tile warps in the persistent patch kernel -- H(grad) parity, cfg2 + cfg5 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg1 or cfg2 or stream or nbox1" > gpurun_out/gpu_ad.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_ad.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
echo done
