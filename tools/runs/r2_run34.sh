# ncu source-level (SASS) captures: deformed Helmholtz pyr P=8 and tet P=9
mkdir -p gpurun_out/r2run34
for c in "pyr 8" "tet 9"; do set -- $c
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(persist|tile)" -s 2 -c 1 \
  -o /tmp/helm_$1$2 -f python tools/profile_op.py --shape $1 --order $2 --op helm --elements 16384 > gpurun_out/r2run34/ncu_$1$2.log 2>&1; echo "ncu $1 $2 rc=$?"
ncu -i /tmp/helm_$1$2.ncu-rep --page source --print-source sass --csv > gpurun_out/r2run34/helm_$1$2_sass.csv 2>&1
ncu -i /tmp/helm_$1$2.ncu-rep --page raw --csv > gpurun_out/r2run34/helm_$1$2_raw.csv 2>&1
done
ls -la gpurun_out/r2run34
