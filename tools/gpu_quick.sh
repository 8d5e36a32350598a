M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
q() { tag=$1; shift; env "$@" timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"$K" --launch-skip 20 -c 3 python tools/prof_mg.py 4 > gpurun_out/q_$tag.csv 2>/dev/null; echo "$tag rc=$?"; python tools/ncu_csv_table.py gpurun_out/q_$tag.csv; }
K="k_mg_l1_elem"; q l1p2 TOPO_X=1
K="k_mg_l1_elem"; q l1old TOPO_L1_P2=0
K="k_mg_apply_st"; q ap2 TOPO_X=1
K="k_mg_apply_st"; q ap4 TOPO_APPLY_UNROLL=4
K="k_mg_apply_st"; q ap13 TOPO_APPLY_UNROLL=13
K="k_mg_deep"; q deep3 TOPO_X=1
run() { echo "== $*"; env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 0 --matvec-reps 5 --no-clocks 2>/dev/null | tail -1 | python -c "import json,sys,statistics as s; d=json.loads(sys.stdin.read()); print(round(d['value'],4), 'ms/cg', round(s.mean(d['ms_per_cg_iter']),3), d['cg_iters_per_step'], 'launches', d['gpu_launches'])"; }
run TOPO_DEEP=0 TOPO_L1_P2=0
run TOPO_DEEP=0
run TOPO_DEEP=0 TOPO_APPLY_UNROLL=13
run TOPO_X=1
timeout 600 python -m pytest tests/test_gpu_mg.py -q -x -p no:cacheprovider 2>&1 | tail -3
