#!/bin/bash
# round-2 pass AM (re-entry check of HEAD after the container was re-created): full GPU suite, default bench, smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; python - <<'PY'
import json
b=json.load(open('gpurun_out/bench.json'))
print(b['value'], b['ms_per_step'], b['e2e']['value'], b['secondary']['value'], b['roofline']['frac'], b['roofline']['secondary']['frac'])
PY
echo done
