#!/bin/bash
# round-2 pass S: SC-fused residual (cfg5) -- trilinear parity cases, cfg5 bench, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg5" > gpurun_out/gpu_cfg5.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_cfg5.log
timeout 600 python bench.py --config 5 --secondary 0 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; tail -1 gpurun_out/bench5.log > gpurun_out/bench5.json
CMD="python bench.py --config 5 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch5.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5.txt 2>&1
echo done
