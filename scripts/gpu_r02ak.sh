#!/bin/bash
# round-2 pass AK: L2 eviction-priority hints of the persistent patch kernel (RM_L2_VALS: factor
# values evict_first; RM_L2_BOX: r window boxes evict_last; RM_L2_RED: c reduce-adds evict_last)
mkdir -p gpurun_out
run() {   # $1 name, $2 defs, $3.. configs
  local name=$1 defs=$2; shift 2
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$defs" python paper_2211_14284_b200/build.py > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; return; }
  for c in "$@"; do
    timeout 300 python bench.py --config $c --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ak_${name}_$c.log 2>&1
    python - $name $c <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ak_{sys.argv[1]}_{sys.argv[2]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "cfg" + sys.argv[2], "%.4f ms" % d["ms_per_step"], {k: round(v, 4) for k, v in ph.items() if v})
PY
  done
}
{
run base "" 2 5
run V "-DRM_L2_VALS=1" 2 5
run VB "-DRM_L2_VALS=1 -DRM_L2_BOX=1" 2 5
run VBR "-DRM_L2_VALS=1 -DRM_L2_BOX=1 -DRM_L2_RED=1" 2 5
run B "-DRM_L2_BOX=1" 2 5
run VR "-DRM_L2_VALS=1 -DRM_L2_RED=1" 2 5
run base2 "" 2 5
} > gpurun_out/ak_sweep.txt 2>&1
echo done
