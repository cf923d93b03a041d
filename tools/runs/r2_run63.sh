# TMA-staged driver for regular-geometry Helmholtz / stiffness A/B (+ parity of the forced variant)
SK200_LIB=paper_2604_04644_b200/libsk200_op0_htmar1.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "regular and (helm or Helm) and not dense and not staged" 2>&1 | tail -1
timeout 1500 python tools/tune_eb.py --variants op0,op0_htmar1,op0 --ops helm,stiff --geo regular --orders 2-10 --gbytes 1.0 > gpurun_out/r2run63_reg.jsonl 2> gpurun_out/r2run63_reg.err; echo "tune rc=$?"
