# thread divisor / min-blocks grid for the other operators (class 2 table + non-collocated Helmholtz)
timeout 2400 python tools/tune_eb.py --variants nt1,nt2,nt4,mb0 --ops bwd,iprod,pderiv,ipderiv,helmnc --orders 1-10 --gbytes 0.5 --reps 6 > gpurun_out/r2run47_ops.jsonl 2> gpurun_out/r2run47_ops.err; echo "tune rc=$?"
tail -2 gpurun_out/r2run47_ops.err
