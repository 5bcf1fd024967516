#!/bin/bash
# pass AV: class-batched kernel with two 384-thread CTAs per SM where three 256-thread CTAs do not fit (-DRM_BATCH_384)
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_384" RM_BUILD_EXPERIMENTS=1 python paper_2211_14284_b200/build.py > gpurun_out/av_build.log 2>&1 || exit 1
RM_VERBOSE=1 timeout 600 $B34 > gpurun_out/av.log 2>&1; tail -1 gpurun_out/av.log > gpurun_out/av.json
grep "batched" gpurun_out/av.log | head -12
python - <<'PY'
import json
b = json.load(open("gpurun_out/av.json"))
for x in (b, b["secondary"]):
    print(x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
echo done
