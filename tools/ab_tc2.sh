cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mg.py -q -x -p no:cacheprovider -k "galerkin or vcycle or loop_parity" 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 --matvec-reps 5 --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print(round(d['value'],4), 'ms/cg', round(s.mean(d['ms_per_cg_iter']),3), d['cg_iters_per_step'], 'setup', [round(p['ms_mg_setup'],3) for p in d['phase_ms']])"; }
run TOPO_TC2=0
run TOPO_TC2=1
run TOPO_TC2=0
run TOPO_TC2=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dgemm_nt64 -c 2 python tools/prof_mg.py 4 2>&1 | grep -E "k_dgemm|duration|bytes" | head -12
