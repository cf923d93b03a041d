# ncu of the hex P=6 Helmholtz kernel the TMA driver replaces (SK_HELM_TMA=0)
mkdir -p gpurun_out/r2run67
bash tools/prof_kernels.sh gpurun_out/r2run67 \
  "helm_hex6_tile|k_tile|1|SK_HELM_TMA=0|--op helm --shape hex --order 6 --elements 100000 --reps 4" \
  "helm_hex6_persist|k_persist|1|SK_HELM_TMA=0|--op helm --shape hex --order 6 --elements 100000 --reps 4"
for f in gpurun_out/r2run67/*_raw.csv; do python tools/ncu_summary.py $f; done > gpurun_out/r2run67/summary.txt 2>&1
grep -E "^==|time |fp64|warps_active|inst |stalls" gpurun_out/r2run67/summary.txt
