#!/bin/bash
# round-2 first GPU pass: parity suite, default bench (cfg5 + nested cfg2), FP64 peak log, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
./scripts/fp64_bench > gpurun_out/fp64_bench.txt 2>&1 || (nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64b scripts/fp64_bench.cu && /tmp/fp64b > gpurun_out/fp64_bench.txt 2>&1)
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
