# tet slice dispatch threshold (compile-time dispatch vs compact L1-table loop) at high order
timeout 1500 python tools/tune_eb.py --variants op0,op0_td7,op0_td8,op0_td10,op0 --ops helm,stiff --shapes tet --orders 6-10 --gbytes 1.0 > gpurun_out/r2run58_td.jsonl 2> gpurun_out/r2run58_td.err; echo "tune rc=$?"
