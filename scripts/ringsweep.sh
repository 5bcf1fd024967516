for nb in "" "RM_NBOX2=1"; do for a in 0 40 90 110; do
  envs="$nb"; [ "$a" != "0" ] && envs="$envs RM_RING_A_KB=$a"
  r=$(env $envs RM_VERBOSE=1 timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1)
  plan=$(echo "$r" | grep "patch plan" | tail -1 | grep -o "ringA=[0-9]* ringB=[0-9]*")
  echo "[$envs] $plan $(echo "$r" | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["roofline"]["launch_ms_avg"],3))')"
done; done
