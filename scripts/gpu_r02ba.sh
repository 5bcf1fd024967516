#!/bin/bash
# pass BA: sweeps without the library's timing events (cross-family colour chain on / off; cfg5 / cfg2 for reference)
mkdir -p gpurun_out
( for c in 3 4 5 2; do timeout 300 python scripts/time_relax_plain.py $c 20 2>&1 | tail -1; done ) > gpurun_out/ba_chainf.txt
rm -f paper_2211_14284_b200/_build/patch_solve.cu.o paper_2211_14284_b200/librm.so
RM_BUILD_DEFS="-DRM_BATCH_CHAINF=0" python paper_2211_14284_b200/build.py > gpurun_out/ba_build.log 2>&1 || exit 1
( for c in 3 4; do timeout 300 python scripts/time_relax_plain.py $c 20 2>&1 | tail -1; done ) > gpurun_out/ba_nochainf.txt
echo "chain across families:"; cat gpurun_out/ba_chainf.txt; echo "no chain across families:"; cat gpurun_out/ba_nochainf.txt
echo done
