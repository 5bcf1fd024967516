#!/bin/bash
# round-2 pass AN: class-batched sliced loop with a one-step look-ahead (A/B against -DRM_BATCH_NOPIPE)
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B34 > gpurun_out/an_pipe.log 2>&1; tail -1 gpurun_out/an_pipe.log > gpurun_out/an_pipe.json
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl or pcg" > gpurun_out/an_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/an_tests.log
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_NOPIPE" python paper_2211_14284_b200/build.py > gpurun_out/an_build.log 2>&1 || exit 1
timeout 600 $B34 > gpurun_out/an_nopipe.log 2>&1; tail -1 gpurun_out/an_nopipe.log > gpurun_out/an_nopipe.json
python - <<'PY'
import json
for n in ("pipe", "nopipe"):
    b = json.load(open(f"gpurun_out/an_{n}.json"))
    for x in (b, b["secondary"]):
        print(n, x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/an_tests.log
echo done
