#!/bin/bash
# round-2 pass P: SC-PH product (sweep parity + PCG counts), then the dsetup timing breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "scph" > gpurun_out/gpu_scph.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_scph.log
RM_VERBOSE=1 timeout 600 python bench.py --config 2 --secondary 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1
echo done
