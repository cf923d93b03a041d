# ncu --set full of the C0 hex scatter (k_c0_scatter_t) and the fused-gather Helmholtz kernel
mkdir -p gpurun_out/r2run88
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_c0_scatter_t" -c 1 -o /tmp/sc -f python bench.py --workload c0hex --steps 1 --warmup 0 --sweep off > gpurun_out/r2run88/sc.log 2>&1; echo "rc=$?"
ncu -i /tmp/sc.ncu-rep --page raw --csv > gpurun_out/r2run88/scatter_raw.csv 2>&1
ncu -i /tmp/sc.ncu-rep --page source --print-source sass --csv > gpurun_out/r2run88/scatter_sass.csv 2>&1
python tools/ncu_summary.py gpurun_out/r2run88/scatter_raw.csv
