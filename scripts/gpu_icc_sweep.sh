#!/bin/bash
# tuning sweep of the ICC piece layout (cfg5 patch kernel): chunks per piece / values per piece
mkdir -p gpurun_out
run() {
  rm -rf paper_2211_14284_b200/_build paper_2211_14284_b200/librm.so
  RM_BUILD_DEFS="$2" python paper_2211_14284_b200/build.py > gpurun_out/build_$1.log 2>&1 || { echo "$1 build failed"; return; }
  timeout 300 python bench.py --config 5 --secondary 0 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/icc_$1.log 2>&1
  python - $1 <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/icc_{sys.argv[1]}.log").read().splitlines()[-1])
ph = d["roofline"]["phase_ms_per_step"]
print(sys.argv[1], "%.4f ms" % d["ms_per_step"], "patch kernel %.4f" % ph["patch_kernel"])
PY
}
{
run c4v4096 ""
run c4v8192 "-DRM_ICC_PIECE_VALS=8192"
run c4v12288 "-DRM_ICC_PIECE_VALS=12288"
run c4v16384 "-DRM_ICC_PIECE_VALS=16384"
run c4v4096b ""
run c4v8192b "-DRM_ICC_PIECE_VALS=8192"
} > gpurun_out/icc_sweep.txt 2>&1
echo done
