# ncu of the Helmholtz P=5 dip (hex / pyr P=5 vs P=6)
mkdir -p gpurun_out/r2run68
bash tools/prof_kernels.sh gpurun_out/r2run68 \
  "helm_hex5|k_|1||--op helm --shape hex --order 5 --elements 150000 --reps 4" \
  "helm_pyr5|k_|1||--op helm --shape pyr --order 5 --elements 200000 --reps 4"
for f in gpurun_out/r2run68/*_raw.csv; do python tools/ncu_summary.py $f; done > gpurun_out/r2run68/summary.txt 2>&1
cat gpurun_out/r2run68/summary.txt
