#!/bin/bash
# round-2 pass AJ: the ICC-SC pre step inside the trilinear apply (RM_APPLY_SC_FUSE) and SC post
# DoFs per thread (RM_SCP_DOFS): parity of the cfg5-shaped cases, then a knob sweep on cfg5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "cfg5 or trilinear or host or smoke or dsetup" > gpurun_out/aj_tests.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/aj_tests.log
run() {   # $1 name, $2 defs, $3.. configs
  local name=$1 defs=$2; shift 2
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$defs" python paper_2211_14284_b200/build.py > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; return; }
  for c in "$@"; do
    timeout 300 python bench.py --config $c --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/aj_${name}_$c.log 2>&1
    python - $name $c <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/aj_{sys.argv[1]}_{sys.argv[2]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "cfg" + sys.argv[2], "%.4f ms" % d["ms_per_step"], "launches", d["gpu_launches"], {k: round(v, 4) for k, v in ph.items() if v})
PY
  done
}
{
run nofuse "-DRM_APPLY_SC_FUSE=0" 5
run fuse "" 5
run fuse_d2 "-DRM_SCP_DOFS=2" 5
run fuse_d4 "-DRM_SCP_DOFS=4" 5
run nofuse2 "-DRM_APPLY_SC_FUSE=0" 5
run fuse2 "" 5
} > gpurun_out/aj_sweep.txt 2>&1
CMD="python bench.py --config 5 --secondary 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/aj_launches_cfg5.csv $CMD > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/aj_launches_cfg5.csv > gpurun_out/aj_launches_cfg5.txt 2>&1
echo done
