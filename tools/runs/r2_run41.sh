# even-odd contractions at hex P=5 (SK_EO_MINP=5) A/B, Helmholtz + stiffness + mass
timeout 900 python tools/tune_eb.py --variants op0,op0_eo5,op0 --ops helm,stiff --shapes hex --orders 4-6 --gbytes 1.0 > gpurun_out/r2run41_eo.jsonl 2> gpurun_out/r2run41_eo.err; echo "tune rc=$?"
SK_MASS_DENSE=0 timeout 900 python tools/tune_eb.py --variants op1,op1_eo5,op1 --ops mass --shapes hex --orders 4-6 --gbytes 1.0 >> gpurun_out/r2run41_eo.jsonl 2>> gpurun_out/r2run41_eo.err; echo "tune rc=$?"
