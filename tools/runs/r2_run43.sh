# even-odd from P=2 / P=3 in the mass kernels A/B (sum-factorised, deformed)
SK_MASS_DENSE=0 timeout 900 python tools/tune_eb.py --variants op1,op1_eo2,op1_eo3,op1 --ops mass --orders 2-4 --gbytes 1.0 > gpurun_out/r2run43_eo.jsonl 2> gpurun_out/r2run43_eo.err; echo "tune rc=$?"
