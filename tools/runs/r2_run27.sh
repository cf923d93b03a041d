# high-order occupancy grid: tile width 1/2/4 x forced min-blocks caps x thread divisor, P=7-10
timeout 1500 python tools/tune_eb.py --variants op0,op0_eb1_mb1_cap4,op0_eb1_mb1_cap6,op0_eb2_mb1_cap2,op0_eb2_mb1_cap3,op0_eb2_mb1_cap4,op0_eb2_nt2_mb1_cap4,op0_eb4_nt2 --ops helm --orders 7-10 --shapes prism,pyr,tet --gbytes 1.0 > gpurun_out/r2run27_grid.jsonl 2> gpurun_out/r2run27_grid.err; echo "tune rc=$?"
tail -3 gpurun_out/r2run27_grid.err
