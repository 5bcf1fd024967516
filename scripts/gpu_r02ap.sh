#!/bin/bash
# round-2 pass AP: class-batched kernel with S slices per warp at once, pivot / ZERO loops with all loads first
# (A/B: -DRM_BATCH_SLICES=4 (default) / 2 / 1)
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B34 > gpurun_out/ap_s4.log 2>&1; tail -1 gpurun_out/ap_s4.log > gpurun_out/ap_s4.json
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl or pcg" > gpurun_out/ap_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/ap_tests.log
for S in 2 1; do
  rm -f paper_2211_14284_b200/_build/patch_solve.cu.o paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="-DRM_BATCH_SLICES=$S" python paper_2211_14284_b200/build.py > gpurun_out/ap_build$S.log 2>&1 || exit 1
  timeout 600 $B34 > gpurun_out/ap_s$S.log 2>&1; tail -1 gpurun_out/ap_s$S.log > gpurun_out/ap_s$S.json
done
python - <<'PY'
import json
for n in ("s4", "s2", "s1"):
    b = json.load(open(f"gpurun_out/ap_{n}.json"))
    for x in (b, b["secondary"]):
        print(n, x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/ap_tests.log
echo done
