# ragged-sweep switches re-check at high order (pyr / tet P=6-10): dispatch max order 7/10, split from P=7, smem tables from P=7/9
timeout 2000 python tools/tune_eb.py --variants op0,op0_rd7,op0_rd10,op0_sp7,op0_smt7,op0_smt9,op0 --ops helm,stiff --shapes pyr,tet --orders 6-10 --gbytes 1.0 > gpurun_out/r2run99_rag.jsonl 2> gpurun_out/r2run99_rag.err; echo "tune rc=$?"
