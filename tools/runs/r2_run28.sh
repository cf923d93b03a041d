# warp-tile mass (k_mass_warp) A/B: parity of the forced variants, then the sweep (deformed, sum-fac only)
for v in op1_mwg1 op1_mwg2 op1_mwg4; do SK200_LIB=paper_2604_04644_b200/libsk200_$v.so SK_MASS_DENSE=0 timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "mass" 2>&1 | tail -1; done
SK_MASS_DENSE=0 timeout 1500 python tools/tune_eb.py --variants op1,op1_mwg1,op1_mwg2,op1_mwg2_mwb2,op1_mwg2_mwb3,op1_mwg2_mwc4,op1_mwg4,op1_mwg4_mwb2 --ops mass --orders 1-8 --gbytes 1.0 > gpurun_out/r2run28_mw.jsonl 2> gpurun_out/r2run28_mw.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run28_mw.err
