# DMMA mass: next group's W held in registers (dwpf) / plus coefficient prefetch (dpf), dense forced on, P=1-4; parity of the forced variant
SK200_LIB=paper_2604_04644_b200/libsk200_op1_dwpf1_dpf1.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "dense_dmma_mass" 2>&1 | tail -1
SK200_LIB=paper_2604_04644_b200/libsk200_op1_dwpf1.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "dense_dmma_mass" 2>&1 | tail -1
SK_MASS_DENSE=1 timeout 1500 python tools/tune_eb.py --variants op1,op1_dwpf1,op1_dwpf1_dpf1,op1 --ops mass --orders 1-4 --gbytes 1.0 > gpurun_out/r2run91_dw.jsonl 2> gpurun_out/r2run91_dw.err; echo "tune rc=$?"
