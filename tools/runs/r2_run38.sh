# driver-equivalent: reference arm, default bench (all per_shape_P tables), smoke
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2run38_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2run38_ref.json 2> gpurun_out/r2run38_ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/r2run38_bench.json 2> gpurun_out/r2run38_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2run38_bench.err
