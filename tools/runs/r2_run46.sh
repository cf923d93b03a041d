# the other reference operators (bwd_trans, iproduct_wrt_base, phys_deriv, iproduct_wrt_deriv_base, noncollocated Helmholtz), deformed, every shape, P=1..10
timeout 1500 python tools/sweep.py --ops bwd,iprod,pderiv,ipderiv,helmnc --orders 1-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run46_ops.jsonl 2> gpurun_out/r2run46_ops.err; echo "sweep rc=$?"
tail -3 gpurun_out/r2run46_ops.err
