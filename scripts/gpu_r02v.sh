#!/bin/bash
# round-2 pass V: block-diagonal final blocks (edge stars) in the class-batched kernel -- H(curl)/H(div) parity, cfg3/cfg4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg3 or cfg4" > gpurun_out/gpu_34.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_34.log
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
echo done
