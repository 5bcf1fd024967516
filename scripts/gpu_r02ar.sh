#!/bin/bash
# round-2 pass AR: class-batched kernel with two 512-thread CTAs per SM (64-register cap), -DRM_BATCH_512X2
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_512X2" python paper_2211_14284_b200/build.py > gpurun_out/ar_build.log 2>&1 || exit 1
RM_VERBOSE=1 timeout 600 $B34 > gpurun_out/ar_x2.log 2>&1; tail -1 gpurun_out/ar_x2.log > gpurun_out/ar_x2.json
grep -i "batch" gpurun_out/ar_x2.log | head -8
python - <<'PY'
import json
b = json.load(open("gpurun_out/ar_x2.json"))
for x in (b, b["secondary"]):
    print("x2", x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
echo done
