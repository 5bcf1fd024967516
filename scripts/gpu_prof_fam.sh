#!/bin/bash
# instrumentation pass: per-family patch-kernel counters (RM_PROFILE) and plans (RM_VERBOSE) for cfg3 / cfg4
mkdir -p gpurun_out
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_EXPERIMENTS=1 python paper_2211_14284_b200/build.py > gpurun_out/build_exp.log 2>&1 || exit 1
for c in 3 4; do
  RM_PROFILE=1 RM_VERBOSE=1 timeout 600 python bench.py --config $c --secondary 0 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_fam_cfg$c.log 2>&1
done
echo done
