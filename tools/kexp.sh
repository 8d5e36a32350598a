# multigrid coarsest-size / K-depth experiments at config 4 (5 warm-up + 20 timed SIMP iterations)
for cfg in "X=1 --mg-coarse-max 1000" "TOPO_KMAX=4 --mg-coarse-max 1000" "TOPO_KMAX=3 --mg-coarse-max 1000" "TOPO_KMAX=3 --mg-coarse-max 2000"; do
  echo "== $cfg"
  envs=$(echo $cfg | tr ' ' '\n' | grep = | tr '\n' ' '); args=$(echo $cfg | tr ' ' '\n' | grep -v = | tr '\n' ' ')
  env $envs python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --matvec-reps 2 --no-clocks $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],4), d['solver']['mg_levels'][-1], d['cg_iters_per_step'], [round(x,2) for x in d['ms_per_cg_iter']][::4], round(d['phase_ms'][-1]['ms_mg_setup'],1))"
done
