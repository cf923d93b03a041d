# ncu --set full of the round-2 TMA kernels vs the kernels they replace (mass pyr P=3, Helmholtz hex P=6)
mkdir -p gpurun_out/r2run66
bash tools/prof_kernels.sh gpurun_out/r2run66 \
  "mass_pyr3_tma|k_mass_tma|1||--op mass --shape pyr --order 3 --elements 1000000 --reps 4" \
  "mass_pyr3_cta|k_tile|1|SK_MASS_TMA=0|--op mass --shape pyr --order 3 --elements 1000000 --reps 4" \
  "helm_hex6_tma|k_persist_tma|1||--op helm --shape hex --order 6 --elements 100000 --reps 4" \
  "helm_hex6_default|k_(tile|persist)|1|SK_HELM_TMA=0|--op helm --shape hex --order 6 --elements 100000 --reps 4"
ls -la gpurun_out/r2run66
for f in gpurun_out/r2run66/*_raw.csv; do python tools/ncu_summary.py $f; done > gpurun_out/r2run66/summary.txt 2>&1
cat gpurun_out/r2run66/summary.txt | head -60
