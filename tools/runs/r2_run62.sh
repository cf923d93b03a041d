# persistent (register-staged next tile) vs one-tile CTAs at high order, re-check
timeout 1500 python tools/tune_eb.py --variants op0,op0_ps0,op0_ps1,op0 --ops helm --shapes prism,pyr,tet --orders 6-10 --gbytes 1.0 > gpurun_out/r2run62_ps.jsonl 2> gpurun_out/r2run62_ps.err; echo "tune rc=$?"
