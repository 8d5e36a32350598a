#!/bin/bash
# Round-2 evidence on one B200 (gpurun from the repo root): default bench line,
# the bench launch list, ncu --set full of the hot kernels, the paper protocol
# (both variants, oracle timed beside).  Output under gpurun_out/$TAG*.
TAG=${1:-r02}
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1
  tail -2 gpurun_out/${TAG}_gpu_tests.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
  timeout 600 python tools/run_configs.py 0 1 2 3 > gpurun_out/${TAG}_configs.jsonl 2>&1
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.jsonl 2> gpurun_out/${TAG}_bench_default.err
tail -c 600 gpurun_out/${TAG}_bench.jsonl
timeout 600 python tools/paper_protocol.py --variant both --oracle-iters 2 > gpurun_out/${TAG}_paper_protocol.jsonl 2>&1
tail -c 300 gpurun_out/${TAG}_paper_protocol.jsonl
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --matvec-reps 5 --no-clocks > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launch list rc=$?"
python tools/ncu_agg_grid.py gpurun_out/${TAG}_launches_bench.csv 60 > gpurun_out/${TAG}_kernel_shares_bench.txt
gzip -f gpurun_out/${TAG}_launches_bench.csv
K=0
for spec in "k_mv_wht<.int.8, .int.2, .bool.1, .int.0,::2" "k_mv_wht<.int.8, .int.3, .bool.0, .int.2,::2" \
            "k_mv_wht<.int.8, .int.0, .bool.0, .int.1,::2" "k_mg_l1_face<float::4" "k_filt25::1" \
            "k_sens_x::1" "k_update<.bool.1, .bool.1::2" "k_mg_apply_st<float::4" "k_dgemm_nt64_tc::0" \
            "k_mg_sweep_st8::40"; do
  re="${spec%%::*}"; skip="${spec##*::}"
  K=$((K+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$re" --launch-skip $skip -c 1 -o gpurun_out/${TAG}_full_$K python tools/prof_mg.py 4 > gpurun_out/${TAG}_full_$K.log 2>&1
  echo "full $K ($re, skip $skip) rc=$?"
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_$K.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/${TAG}_full_$K.ncu-rep > gpurun_out/${TAG}_full_$K.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/${TAG}_full_$K.ncu-rep >> gpurun_out/${TAG}_full_$K.txt 2>&1
  python tools/ncu_json.py gpurun_out/${TAG}_full_$K.ncu-rep gpurun_out/${TAG}_full_$K.json "${TAG} capture" > /dev/null 2>&1
  rm -f gpurun_out/${TAG}_full_$K.ncu-rep gpurun_out/${TAG}_full_$K.raw.csv
done
python - "$TAG" <<'PY'
import glob, json, sys
tag = sys.argv[1]
out = {"_source": "ncu --set full --clock-control none, config 4, tools/prof_mg.py 4 (second design), capture " + tag}
for fn in sorted(glob.glob("gpurun_out/%s_full_*.json" % tag)):
    for k, v in json.load(open(fn)).items():
        if not k.startswith("_"):
            out.setdefault(k, v)
json.dump(out, open("gpurun_out/%s_ncu_cfg4_mg.json" % tag, "w"), indent=1)
print(sorted(k for k in out if not k.startswith("_")))
PY
