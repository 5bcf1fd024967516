#!/bin/bash
# pass AT: class-batched kernel, third 256-thread CTA per SM where shared memory allows (A/B -DRM_BATCH_CTA3=0)
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B34 > gpurun_out/at_cta3.log 2>&1; tail -1 gpurun_out/at_cta3.log > gpurun_out/at_cta3.json
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl" > gpurun_out/at_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/at_tests.log
rm -f paper_2211_14284_b200/_build/patch_solve.cu.o paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_CTA3=0" python paper_2211_14284_b200/build.py > gpurun_out/at_build.log 2>&1 || exit 1
timeout 600 $B34 > gpurun_out/at_cta2.log 2>&1; tail -1 gpurun_out/at_cta2.log > gpurun_out/at_cta2.json
python - <<'PY'
import json
for n in ("cta3", "cta2"):
    b = json.load(open(f"gpurun_out/at_{n}.json"))
    for x in (b, b["secondary"]):
        print(n, x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/at_tests.log
echo done
