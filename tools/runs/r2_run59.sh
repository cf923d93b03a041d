# item-loop unroll 2 (two lines per thread per iteration) re-check, Helmholtz deformed P=4-10
timeout 1500 python tools/tune_eb.py --variants op0,op0_iu2,op0 --ops helm --orders 4-10 --gbytes 1.0 > gpurun_out/r2run59_iu.jsonl 2> gpurun_out/r2run59_iu.err; echo "tune rc=$?"
