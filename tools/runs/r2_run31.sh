# TMA-fed deformed mass (k_mass_tma) A/B: parity of the forced variant, then the sweep
SK200_LIB=paper_2604_04644_b200/libsk200_op1_mtma1.so SK_MASS_DENSE=0 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "mass" 2>&1 | tail -3
SK_MASS_DENSE=0 timeout 1500 python tools/tune_eb.py --variants op1,op1_mtma1,op1 --ops mass --orders 1-8 --gbytes 1.0 > gpurun_out/r2run31_mtma.jsonl 2> gpurun_out/r2run31_mtma.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run31_mtma.err
