#!/bin/bash
# tuning sweep of the transfer units of the persistent patch kernel (cfg2: tile + sparse channels; cfg5: ICC)
mkdir -p gpurun_out
run() {
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$2" python paper_2211_14284_b200/build.py > gpurun_out/build_$1.log 2>&1 || { echo "$1 build failed"; return; }
  for c in 2 5; do
    timeout 300 python bench.py --config $c --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/unit_$1_$c.log 2>&1
    python - $1 $c <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/unit_{sys.argv[1]}_{sys.argv[2]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "cfg" + sys.argv[2], "%.4f ms" % d["ms_per_step"], "patch kernel %.4f" % ph["patch_kernel"])
PY
  done
}
{
run base ""
run tile8192 "-DRM_UNIT_VALS_TILE=8192"
run tile2048 "-DRM_UNIT_VALS_TILE=2048"
run sp4096 "-DRM_UNIT_VALS=4096"
run nd8 "-DRM_NDESC=8"
run nd32 "-DRM_NDESC=32"
} > gpurun_out/unit_sweep.txt 2>&1
echo done
