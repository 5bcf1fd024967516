#!/bin/bash
# tuning sweep of launch sizes (rebuilt on the box with -D overrides): k = 0 apply CTA (cfg2),
# SC pre / post CTAs (cfg5); prints ms per sweep and the phase split per variant
mkdir -p gpurun_out
run() {   # $1 = name, $2 = -D definitions, $3 = config
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$2" python paper_2211_14284_b200/build.py > gpurun_out/build_$1.log 2>&1 || { echo "$1 build failed"; return; }
  timeout 300 python bench.py --config $3 --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/knob_$1.log 2>&1
  python - $1 <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/knob_{sys.argv[1]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "%.4f ms" % d["ms_per_step"], {k: round(v, 4) for k, v in ph.items() if v})
PY
}
{
run q256 "" 2
run q512 "-DRM_Q_THREADS=512 -DRM_Q_MINB=2" 2
run q128 "-DRM_Q_THREADS=128 -DRM_Q_MINB=10" 2
run sc256 "" 5
run scc128 "-DRM_SCC_THREADS=128" 5
run scc512 "-DRM_SCC_THREADS=512" 5
run scp128 "-DRM_SCP_THREADS=128" 5
run scp512 "-DRM_SCP_THREADS=512" 5
} > gpurun_out/knob_sweep.txt 2>&1
echo done
