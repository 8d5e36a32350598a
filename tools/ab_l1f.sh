#!/bin/bash
# A/B of the level-1 face operator's cp.async operand prefetch (TOPO_L1F_ASYNC) on one box.
timeout 1200 python -m pytest tests/test_gpu_mg.py tests/test_gpu_dist_mg.py -q -x -p no:cacheprovider 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 --matvec-reps 5 --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print(round(d['value'],5), 'ms/cg', round(s.mean(d['ms_per_cg_iter']),3), d['cg_iters_per_step'], 'c', d.get('c_last'))"; }
run TOPO_L1F_ASYNC=0
run TOPO_L1F_ASYNC=1
run TOPO_L1F_ASYNC=0
run TOPO_L1F_ASYNC=1
