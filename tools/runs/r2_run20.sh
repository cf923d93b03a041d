# high-order deformed Helmholtz: low-register M2 x geometry chunk / min-blocks cap / tile width grid, P=7-10
timeout 1500 python tools/tune_eb.py --variants op0,op0_lowreg0,op0_lowreg1_ch2,op0_lowreg1_ch6,op0_lowreg1_ch8,op0_lowreg1_eb1,op0_lowreg1_eb2,op0_lowreg1_eb4,op0_lowreg1_mb1_cap2,op0_lowreg1_mb1_cap3,op0_lowreg1_mb1_cap4,op0_mb1_cap3 --ops helm --orders 7-10 --gbytes 1.0 > gpurun_out/r2run20_grid.jsonl 2> gpurun_out/r2run20_grid.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run20_grid.err
echo done
