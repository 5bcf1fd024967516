#!/bin/bash
# round-2 pass AF: k-form apply CTA size -- H(curl)/H(div) parity (cfg3/cfg4 shapes), cfg3/cfg4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep and (cfg3 or cfg4)" > gpurun_out/gpu_af.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_af.log
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline --no-e2e > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
echo done
