#!/bin/bash
# pass AU: third-CTA fix (B = 8 keeps two CTAs): k-form parity subset + cfg3/cfg4 bench
mkdir -p gpurun_out
B34="python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B34 > gpurun_out/au.log 2>&1; tail -1 gpurun_out/au.log > gpurun_out/au.json
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "apply_and_sweep or hcurl" > gpurun_out/au_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/au_tests.log
python - <<'PY'
import json
b = json.load(open("gpurun_out/au.json"))
for x in (b, b["secondary"]):
    print(x["config"]["workload"][:5], "%.3f ms" % x["ms_per_step"], x["roofline"]["phase_ms_per_step"])
PY
tail -3 gpurun_out/au_tests.log
echo done
