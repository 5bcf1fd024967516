#!/bin/bash
# round-2 pass AB: overlapped host copies in rm_relax_host (SC-fused path) -- test, cfg5 e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "host" > gpurun_out/gpu_ab.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_ab.log
timeout 600 python bench.py --config 5 --secondary 0 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; tail -1 gpurun_out/bench5.log > gpurun_out/bench5.json
echo done
