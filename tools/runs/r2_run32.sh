# TMA-fed mass: tile width x thread divisor grid
SK_MASS_DENSE=0 timeout 1500 python tools/tune_eb.py --variants op1,op1_mtma1,op1_mtma1_eb16,op1_mtma1_eb16_nt2,op1_mtma1_eb4,op1_mtma1_eb4_nt2,op1_mtma1_eb8,op1_mtma1_eb8_nt2 --ops mass --orders 1-8 --gbytes 1.0 > gpurun_out/r2run32_mtma.jsonl 2> gpurun_out/r2run32_mtma.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run32_mtma.err
