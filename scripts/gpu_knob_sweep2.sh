#!/bin/bash
# tuning sweep 2: SC post CTA size, skeleton gather residency (cfg5, cfg2), Hiptmair row kernels (cfg4)
mkdir -p gpurun_out
run() {   # $1 name, $2 defs, $3.. configs
  local name=$1 defs=$2; shift 2
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$defs" python paper_2211_14284_b200/build.py > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; return; }
  for c in "$@"; do
    timeout 300 python bench.py --config $c --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/k2_${name}_$c.log 2>&1
    python - $name $c <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/k2_{sys.argv[1]}_{sys.argv[2]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "cfg" + sys.argv[2], "%.4f ms" % d["ms_per_step"], {k: round(v, 4) for k, v in ph.items() if v})
PY
  done
}
{
run base "" 5 2 4
run scp128 "-DRM_SCP_THREADS=128" 5
run gsc4 "-DRM_GSC_MINB=4" 5 2
run gsc8 "-DRM_GSC_MINB=8" 5 2
run hip4 "-DRM_HIP_WARPS=4" 4
run hip16 "-DRM_HIP_WARPS=16" 4
run base2 "" 5 2 4
run scp128b "-DRM_SCP_THREADS=128" 5
} > gpurun_out/knob_sweep2.txt 2>&1
echo done
