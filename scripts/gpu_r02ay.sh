#!/bin/bash
# round-2 pass AY (final state: pass AW + programmatic dependent launches of the batched colours; look-ahead sliced loop, loads-first
# pivot / ZERO loops, third CTA per SM): full GPU suite, default bench, cfg3/cfg4 bench, reference arm,
# launch lists, ncu --set full of the class-batched kernel (cfg4 potential family), smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
for c in 5 2 3 4; do
  CMD="python bench.py --config $c --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$c.csv $CMD > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/launches_cfg$c.csv > gpurun_out/launches_cfg$c.txt 2>&1
done
C4="python bench.py --config 4 --secondary 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:patch_batch -s 26 -c 1 -o gpurun_out/prof_batch_cfg4_ay $C4 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log
echo done
