# DRAM traffic of the dominant Helmholtz launches (roofline.traffic): tet P=4 (headline), the mixed6 blocks (P=6), hex P=4
mkdir -p gpurun_out/r2run71
bash tools/prof_kernels.sh gpurun_out/r2run71 \
  "tet4|k_|1||--op helm --shape tet --order 4 --elements 1048576 --reps 6" \
  "hex6|k_|1||--op helm --shape hex --order 6 --elements 131072 --reps 6" \
  "prism6|k_|1||--op helm --shape prism --order 6 --elements 131072 --reps 6" \
  "pyr6|k_|1||--op helm --shape pyr --order 6 --elements 131072 --reps 6" \
  "tet6|k_|1||--op helm --shape tet --order 6 --elements 131072 --reps 6" \
  "hex4|k_|1||--op helm --shape hex --order 4 --elements 262144 --reps 6"
for f in gpurun_out/r2run71/*_raw.csv; do python tools/ncu_summary.py $f; done > gpurun_out/r2run71/summary.txt 2>&1
grep -E "^==|time |dram_rd |dram_wr " gpurun_out/r2run71/summary.txt
