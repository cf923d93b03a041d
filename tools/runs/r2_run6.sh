timeout 900 python bench.py > gpurun_out/r2run6_bench.json 2> gpurun_out/r2run6_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2run6_ref.json 2> gpurun_out/r2run6_ref.err; echo "ref rc=$?"
for w in hex4 mixed6 c0hex tet4max; do timeout 900 python bench.py --workload $w --sweep off > gpurun_out/r2run6_$w.json 2> gpurun_out/r2run6_$w.err; echo "$w rc=$?"; done
SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --sweep on --sweep-quick > gpurun_out/r2run6_share2.json 2> gpurun_out/r2run6_share2.err; echo "share2 rc=$?"
SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload c0hex --elements 32768 > gpurun_out/r2run6_share2_c0.json 2> gpurun_out/r2run6_share2_c0.err; echo "share2 c0 rc=$?"
mkdir -p gpurun_out/ncu_r2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_r2/bench_launches.csv python bench.py --steps 2 --warmup 1 --sweep off > gpurun_out/ncu_r2/bench_under_ncu.log 2>&1; echo "launches rc=$?"
bash tools/prof_kernels.sh gpurun_out/ncu_r2 \
  "helm_hex10_fused|k_tile|1||--op helm --shape hex --order 10 --elements 12000 --reps 4" \
  "helm_hex10_staged|k_tile|3||--op helmstaged --shape hex --order 10 --elements 12000 --reps 2" \
  "helm_tet10_fused|k_tile|1||--op helm --shape tet --order 10 --elements 16000 --reps 4" \
  "helm_tet10_staged|k_tile|3||--op helmstaged --shape tet --order 10 --elements 16000 --reps 2" \
  "helm_tet4_fused|k_tile|1||--op helm --shape tet --order 4 --elements 1048576 --reps 4" \
  "mass_pyr2_dense|k_mass_dense|1|SK_MASS_DENSE=1|--op mass --shape pyr --order 2 --elements 2000000 --reps 4" \
  "mass_pyr2_sumfac|k_tile|1|SK_MASS_DENSE=0|--op mass --shape pyr --order 2 --elements 2000000 --reps 4" \
  "helmreg_tet3_dense|k_helm_dense|1|SK_HELM_DENSE=1|--op helm --geo regular --shape tet --order 3 --elements 1000000 --reps 4" \
  "helmreg_tet3_sumfac|k_tile|1|SK_HELM_DENSE=0|--op helm --geo regular --shape tet --order 3 --elements 1000000 --reps 4"
du -sh gpurun_out
echo done
