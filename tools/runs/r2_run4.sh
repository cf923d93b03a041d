timeout 1800 python tools/tune_eb.py --variants op0,op0_ring2,op0_ring3,op0_ring4,op0_eb1,op0_ring3_eb1,op0_ring4_eb1,op0_ring6_eb1 --ops helm,stiff --orders 4-10 --gbytes 1.0 --reps 8 > gpurun_out/r2run4_ring.jsonl 2> gpurun_out/r2run4_ring.err
echo done
