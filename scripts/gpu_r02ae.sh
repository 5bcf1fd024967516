#!/bin/bash
# round-2 pass AE: row-per-warp Hiptmair D / D^T -- H(curl)/H(div) parity, cfg3/cfg4 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "cfg3 or cfg4 or scph or pafw or cfg1" > gpurun_out/gpu_ae.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_ae.log
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline --no-e2e > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
CMD="python bench.py --config 4 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg4.csv > gpurun_out/launches_cfg4.txt 2>&1
echo done
