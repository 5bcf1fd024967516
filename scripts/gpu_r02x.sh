#!/bin/bash
# round-2 pass X: post step writes u_out (SC), apply_q register cap -- H(grad) parity, cfg5 + cfg2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg1 or cfg2 or cfg5 or sc" > gpurun_out/gpu_x.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_x.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
echo done
