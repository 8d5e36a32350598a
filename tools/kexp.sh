# A/B experiments at config 4 (5 warm-up + 20 timed SIMP iterations): env settings per line
for cfg in "TOPO_TINY_NODES=0" "TOPO_TINY_NODES=12000" "TOPO_TINY_NODES=80000"; do
  echo "== $cfg"
  env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --matvec-reps 2 --no-clocks 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],4), d['cg_iters_per_step'], [round(x,2) for x in d['ms_per_cg_iter']][::4])"
done
