# persistent TMA-staged Helmholtz driver (k_persist_tma) A/B: parity of the forced variant, helm + stiffness sweep
SK200_LIB=paper_2604_04644_b200/libsk200_op0_htma1.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "helm or persistent" 2>&1 | tail -2
timeout 1500 python tools/tune_eb.py --variants op0,op0_htma1,op0 --ops helm,stiff --orders 2-10 --gbytes 1.0 > gpurun_out/r2run35_htma.jsonl 2> gpurun_out/r2run35_htma.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run35_htma.err
