#!/bin/bash
# pass AS: class-batched configurations again on the look-ahead kernel (experiments build reads RM_BATCH_CFG)
mkdir -p gpurun_out
rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
RM_BUILD_EXPERIMENTS=1 python paper_2211_14284_b200/build.py > gpurun_out/as_build.log 2>&1 || exit 1
for cfgs in auto 4,512 2,512 4,256; do
  if [ $cfgs != auto ]; then export RM_BATCH_CFG=$cfgs; else unset RM_BATCH_CFG; fi
  RM_VERBOSE=1 timeout 300 python bench.py --config 3 --secondary 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/as_$cfgs.log 2>&1
  python - $cfgs <<'PY'
import json, sys
l = open(f"gpurun_out/as_{sys.argv[1]}.log").read().splitlines()
d = json.loads(l[-1])
print(sys.argv[1], "cfg3 %.3f ms" % d["ms_per_step"], "cfg4 %.3f ms" % d["secondary"]["ms_per_step"],
      d["secondary"]["roofline"]["phase_ms_per_step"], [x for x in l if "batched" in x][:6])
PY
done
echo done
