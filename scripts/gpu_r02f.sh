#!/bin/bash
# round-2 pass F: parity suite (incl. H(curl)/H(div) slabs), cfg3/cfg4 bench after the multi-rank refactor
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --config 3 --secondary 4 --no-cpu-baseline --steps 5 > gpurun_out/bench34.log 2>&1; tail -1 gpurun_out/bench34.log > gpurun_out/bench34.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
echo done
