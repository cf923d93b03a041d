# non-collocated Helmholtz tile-width grid, EB 16/8/4 (five-plane fit)
timeout 1800 python tools/tune_eb.py --variants op6,op6_eb16,op6_eb8,op6_eb4 --ops helmnc --orders 1-10 --gbytes 0.5 --reps 6 > gpurun_out/r2run52_nc.jsonl 2> gpurun_out/r2run52_nc.err; echo "tune rc=$?"
