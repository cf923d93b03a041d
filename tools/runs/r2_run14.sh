SK_MASS_DENSE=0 timeout 1500 python tools/tune_eb.py --variants op1,op1_eb16,op1_eb8,op1_eb4,op1_eb2,op1_nt2,op1_eb8_nt2,op1_eb4_nt2 --ops mass --shapes prism,pyr --orders 2-8 --gbytes 1.0 --reps 10 > gpurun_out/r2run14_mass_tune.jsonl 2>&1
echo done
