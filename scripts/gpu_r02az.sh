#!/bin/bash
# pass AZ: the colour chain continued across orientation families (A/B -DRM_BATCH_CHAINF=0)
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B34 > gpurun_out/az_chainf.log 2>&1; tail -1 gpurun_out/az_chainf.log > gpurun_out/az_chainf.json
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl or pcg" > gpurun_out/az_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/az_tests.log
rm -f paper_2211_14284_b200/_build/patch_solve.cu.o paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_CHAINF=0" python paper_2211_14284_b200/build.py > gpurun_out/az_build.log 2>&1 || exit 1
timeout 600 $B34 > gpurun_out/az_nochainf.log 2>&1; tail -1 gpurun_out/az_nochainf.log > gpurun_out/az_nochainf.json
python - <<'PY'
import json
for n in ("chainf", "nochainf"):
    b = json.load(open(f"gpurun_out/az_{n}.json"))
    for x in (b, b["secondary"]):
        print(n, x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/az_tests.log
echo done
