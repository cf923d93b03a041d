# ncu source-level (SASS) capture of the sum-factorised mass, tet P=4 deformed
mkdir -p gpurun_out/r2run30
SK_MASS_DENSE=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(persist|tile)" -s 2 -c 1 \
  -o /tmp/mass_tet4 -f python tools/profile_op.py --shape tet --order 4 --op mass --elements 262144 > gpurun_out/r2run30/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/mass_tet4.ncu-rep --page source --print-source sass --csv > gpurun_out/r2run30/mass_tet4_sass.csv 2>&1
ncu -i /tmp/mass_tet4.ncu-rep --page raw --csv > gpurun_out/r2run30/mass_tet4_raw.csv 2>&1
ls -la gpurun_out/r2run30; tail -3 gpurun_out/r2run30/ncu.log
