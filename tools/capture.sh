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
for re in "k_mv_wht<.int.8, .int.2, .bool.1, .int.0>" "k_mv_wht<.int.8, .int.3, .bool.0, .int.2>" "k_mv_wht<.int.8, .int.0, .bool.0, .int.1>" "k_mg_l1_elem<float>" "k_mg_restrict0<float>" "k_mg_prolong0<float>" "k_update<.bool.1, .bool.1>" "k_oc_pass<.int.1>" "k_mg_apply_st<float>" "k_filt_apply<.int.2>" "k_sens"; do
  K=$((K+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$re" --launch-skip 2 -c 1 -o gpurun_out/${TAG}_full_$K python tools/prof_mg.py 4 > gpurun_out/${TAG}_full_$K.log 2>&1
  echo "full $K ($re) rc=$?"
  # keep the copy-back under gpurun's 64 MiB: raw metrics as CSV, stall/source
  # attribution as text, the report itself only for the PCG matvec
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_$K.raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/${TAG}_full_$K.ncu-rep > gpurun_out/${TAG}_full_$K.txt 2>&1
  python tools/ncu_stalls.py gpurun_out/${TAG}_full_$K.ncu-rep >> gpurun_out/${TAG}_full_$K.txt 2>&1
  [ $K -eq 1 ] || rm -f gpurun_out/${TAG}_full_$K.ncu-rep
done
python tools/ncu_json.py "gpurun_out/${TAG}_full_1.ncu-rep" gpurun_out/${TAG}_ncu_pcg.json "${TAG} capture" > /dev/null 2>&1
rm -f gpurun_out/${TAG}_full_1.ncu-rep
