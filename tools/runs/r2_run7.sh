SK_MASS_DENSE=1 timeout 1200 python tools/tune_eb.py --variants op1,op1_dpf1,op1_dminb5,op1_dminb5_dpf1,op1_dminb4_dpf1 --ops mass --orders 1-3 --gbytes 1.0 --reps 10 > gpurun_out/r2run7_dense_tune_def.jsonl 2>&1
SK_MASS_DENSE=1 timeout 1200 python tools/tune_eb.py --variants op1,op1_dpf1,op1_dminb5,op1_dminb5_dpf1,op1_dminb4_dpf1 --ops mass --orders 1-6 --geo regular --shapes tet,pyr --gbytes 0.3 --reps 10 > gpurun_out/r2run7_dense_tune_reg.jsonl 2>&1
echo done
