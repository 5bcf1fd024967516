#!/bin/bash
# round-2 pass T: k = 0 Cartesian apply as one launch + skeleton-only gather -- H(grad) parity, cfg2 bench, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg1 or cfg2 or coarse or slab or precondition or interior_only" > gpurun_out/gpu_k0.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_k0.log
timeout 600 python bench.py --config 2 --secondary 0 --no-cpu-baseline > gpurun_out/bench2.log 2>&1; tail -1 gpurun_out/bench2.log > gpurun_out/bench2.json
CMD="python bench.py --config 2 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch2.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg2.csv > gpurun_out/launches_cfg2.txt 2>&1
echo done
