# bwd_trans tile-width grid (its own table now)
timeout 1500 python tools/tune_eb.py --variants op2,op2_eb16,op2_eb8,op2_eb4,op2_eb2,op2_eb1 --ops bwd --orders 1-10 --gbytes 0.5 --reps 6 > gpurun_out/r2run49_bwd.jsonl 2> gpurun_out/r2run49_bwd.err; echo "tune rc=$?"
tail -2 gpurun_out/r2run49_bwd.err
