#!/bin/bash
# experiments build: class-batched kernel configurations (B, threads) on cfg3 / cfg4
mkdir -p gpurun_out
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_EXPERIMENTS=1 python paper_2211_14284_b200/build.py > gpurun_out/build_exp.log 2>&1 || exit 1
for cfgs in auto 8,512 4,512 2,512 8,256 4,256 2,256; do
  if [ $cfgs != auto ]; then export RM_BATCH_CFG=$cfgs; else unset RM_BATCH_CFG; fi
  RM_VERBOSE=1 timeout 300 python bench.py --config 3 --secondary 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$cfgs.log 2>&1
  python - $cfgs <<'PY'
import json, sys
l = open(f"gpurun_out/sweep_{sys.argv[1]}.log").read().splitlines()
d = json.loads(l[-1])
print(sys.argv[1], "cfg3 %.3f ms" % d["ms_per_step"], "cfg4 %.3f ms" % d["secondary"]["ms_per_step"],
      [x for x in l if "batched" in x][:6])
PY
done > gpurun_out/batch_sweep.txt 2>&1
echo done
