# A/B experiments at config 4 (5 warm-up + 20 timed SIMP iterations): one env setting per argument
#   bash tools/kexp.sh "TOPO_KMAX=3" "TOPO_KMAX=4"
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --matvec-reps 2 --no-clocks 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],4), d['cg_iters_per_step'], [round(x,2) for x in d['ms_per_cg_iter']][::4], [round(p['ms_mg_setup'],1) for p in d['phase_ms']][::5])"
done
