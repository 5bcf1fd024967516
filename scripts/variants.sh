#!/bin/bash
# ring / occupancy / unit-size variants of the bench (one line each)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in ${VARIANTS:-"X=1" "RM_CTAS_PER_SM=2"}; do
  echo "== $v"
  env $(echo $v | tr , " ") RM_VERBOSE=1 timeout 300 $B 2>&1 | grep -E "patch plan|^\{" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3e ms %.3f patch_ms %.3f frac %.3f'%(d['value'],d['ms_per_step'],d['roofline']['phase_ms_per_step'][1],d['roofline']['frac']))
    else: print(l.strip())"
done
