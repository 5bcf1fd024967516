#!/bin/bash
# round-2 pass AQ: class-batched kernel knobs on top of the look-ahead loop: serpentine slice -> warp map, U
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
run() {  # name, defs
  if [ -n "$2" ]; then
    rm -f paper_2211_14284_b200/_build/patch_solve.cu.o paper_2211_14284_b200/librm.so
    RM_BUILD_DEFS="$2" python paper_2211_14284_b200/build.py > gpurun_out/aq_build_$1.log 2>&1 || return 1
  fi
  timeout 600 $B34 > gpurun_out/aq_$1.log 2>&1; tail -1 gpurun_out/aq_$1.log > gpurun_out/aq_$1.json
}
run base ""
run serp "-DRM_BATCH_SERP"
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl" > gpurun_out/aq_tests_serp.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/aq_tests_serp.log
run serp_u8 "-DRM_BATCH_SERP -DRM_BATCH_U=8"
run u8 "-DRM_BATCH_U=8"
run u2 "-DRM_BATCH_U=2"
python - <<'PY'
import json
for n in ("base", "serp", "serp_u8", "u8", "u2"):
    try:
        b = json.load(open(f"gpurun_out/aq_{n}.json"))
    except Exception as e:
        print(n, "failed", e); continue
    for x in (b, b["secondary"]):
        print(n, x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/aq_tests_serp.log
echo done
