# even-odd threshold A/B for the Helmholtz / stiffness kernel (EO from P=2/3/4/7 for every shape)
timeout 1500 python tools/tune_eb.py --variants op0,op0_eo2,op0_eo3,op0_eo4,op0_eo7,op0 --ops helm,stiff --orders 2-8 --gbytes 1.0 > gpurun_out/r2run45_eo.jsonl 2> gpurun_out/r2run45_eo.err; echo "tune rc=$?"
