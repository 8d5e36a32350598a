timeout 900 python -m pytest tests/test_gpu_dist_mg.py tests/test_dist_host.py -q -p no:cacheprovider 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -4
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 --matvec-reps 5 --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print(round(d['value'],4), 'ms/cg', round(s.mean(d['ms_per_cg_iter']),3), d['cg_iters_per_step'], 'launches', d['gpu_launches'])"; }
run TOPO_X=1
