#!/bin/bash
# round-2 pass C: full parity suite, cfg3/cfg4 bench, launch lists, ncu of the k-form apply
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
for c in 3 4; do
  CMD="python bench.py --config $c --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > gpurun_out/ncu_launch$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_ncf -s 3 -c 1 -o gpurun_out/prof_apply_ncf_cfg4 \
  python bench.py --config 4 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ncf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:patch_stream -s 4 -c 1 -o gpurun_out/prof_patch_cfg4 \
  python bench.py --config 4 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p4.log 2>&1
echo done
