# M2 low-register metric sweep A/B (deformed Helmholtz, P=4-10, all shapes)
timeout 1500 python tools/tune_eb.py --variants op0,op0_lowreg1,op0_lowreg0 --ops helm --orders 4-10 --gbytes 1.0 > gpurun_out/r2run18_lowreg.jsonl 2> gpurun_out/r2run18_lowreg.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run18_lowreg.err
echo done
