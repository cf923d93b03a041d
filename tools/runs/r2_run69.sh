# P=5 dip grid: row stride 9/11, tile width 4/1, min-blocks cap 8 (Helmholtz + stiffness, P=4-6)
timeout 1800 python tools/tune_eb.py --variants op0,op0_s9,op0_s11,op0_eb4,op0_eb1,op0_mb1_cap8,op0 --ops helm,stiff --orders 4-6 --gbytes 1.0 > gpurun_out/r2run69_p5.jsonl 2> gpurun_out/r2run69_p5.err; echo "tune rc=$?"
