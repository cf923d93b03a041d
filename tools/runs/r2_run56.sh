# high-order prism / pyr / tet: TMA-staged driver without the register cap, with the low-register metric sweep
timeout 1500 python tools/tune_eb.py --variants op0,op0_htma1_mb0,op0_htma1_lowreg1,op0_htma1_lowreg1_mb0 --ops helm --shapes prism,pyr,tet --orders 7-10 --gbytes 1.0 > gpurun_out/r2run56_hp.jsonl 2> gpurun_out/r2run56_hp.err; echo "tune rc=$?"
