#!/bin/bash
# round-2 pass O: device-resident numeric setup (dsetup.cu) -- parity vs host setup and oracle, full suite, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k device_setup > gpurun_out/gpu_dsetup.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_dsetup.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
echo done
