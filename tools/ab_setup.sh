#!/bin/bash
# A/B of multigrid-setup changes on one box: parity tests of the hierarchy,
# then config-4 bench lines with the toggles given as arguments (VAR=0 VAR=1 ...)
timeout 900 python -m pytest tests/test_gpu_mg.py -q -x -p no:cacheprovider -k "galerkin or vcycle or solve_parity or loop_parity" 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 --matvec-reps 5 --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print(round(d['value'],4), 'ms/cg', round(s.mean(d['ms_per_cg_iter']),3), d['cg_iters_per_step'], 'setup', [round(p['ms_mg_setup'],3) for p in d['phase_ms']])"; }
for v in "$@"; do run $v; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_mg_dense_fill|k_sw_block_inv" -c 4 python tools/prof_mg.py 4 2>&1 | grep -E "^  k_|duration" | head -12
