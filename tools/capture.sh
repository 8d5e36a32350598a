#!/bin/bash
# Round evidence on one B200 (run through gpurun from the repo root):
#   tests, default bench line, launch list of the bench command, ncu --set full
#   captures of the hot kernels.  Output under gpurun_out/$TAG*.
TAG=${1:-cap}
python -m paper_2504_05604_b200.build --force > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.log 2>&1
tail -2 gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
tail -c 400 gpurun_out/${TAG}_bench.jsonl
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --matvec-reps 5 > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launch list rc=$?"
K=0
# "regex::launch-skip" (prof_mg.py runs two designs; skip into the second one)
for spec in "k_mv_wht<.int.8, .int.2, .bool.1, .int.0,::2" "k_mv_wht<.int.8, .int.3, .bool.0, .int.2,::2" \
            "k_mv_wht<.int.8, .int.0, .bool.0, .int.1,::2" "k_mg_l1_elem<float>::4" "k_mg_restrict0<float::2" \
            "k_mg_prolong0<float::2" "k_update<.bool.1, .bool.1>::2" "k_oc_pass<.int.1>::6" \
            "k_mg_sweep_st8<.bool.1, float>::40" "k_mg_asm_galerkin_t::3" "k_sw_block_inv::61" \
            "k_mg_apply_st<float>::20" "k_sens::1"; do
  re="${spec%%::*}"; skip="${spec##*::}"
  K=$((K+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$re" --launch-skip $skip -c 1 -o gpurun_out/${TAG}_full_$K python tools/prof_mg.py 4 > gpurun_out/${TAG}_full_$K.log 2>&1
  echo "full $K ($re, skip $skip) rc=$?"
  # keep the copy-back under gpurun's 64 MiB: raw metrics as CSV, stall/source
  # attribution as text, per-kernel JSON; the reports themselves are dropped
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_$K.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/${TAG}_full_$K.ncu-rep > gpurun_out/${TAG}_full_$K.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/${TAG}_full_$K.ncu-rep >> gpurun_out/${TAG}_full_$K.txt 2>&1
  python tools/ncu_json.py gpurun_out/${TAG}_full_$K.ncu-rep gpurun_out/${TAG}_full_$K.json "${TAG} capture" > /dev/null 2>&1
  rm -f gpurun_out/${TAG}_full_$K.ncu-rep
done
# one JSON with every captured kernel (bench.py reads roofline.traffic from it)
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
