export PYTHONUNBUFFERED=1
timeout 300 python tools/check_helm.py > gpurun_out/c9_check.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c9_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/c9_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c9_smoke.log 2>&1; echo rc=$? >> gpurun_out/c9_smoke.log
timeout 400 python bench.py > gpurun_out/c9_bench.json 2> gpurun_out/c9_bench.err
timeout 400 python bench.py --workload mixed6 > gpurun_out/c9_bench_mixed6.json 2>> gpurun_out/c9_bench.err
timeout 400 python bench.py --workload c0hex > gpurun_out/c9_bench_c0hex.json 2>> gpurun_out/c9_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c9_bench_ref.json 2>> gpurun_out/c9_bench.err
timeout 1500 python tools/sweep.py --ops helm,stiff,mass --orders 1-10 --gbytes 1.5 > gpurun_out/c9_sweep.jsonl 2> gpurun_out/c9_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c9_bench_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/c9_bench_ncu.log 2>&1
bash tools/prof_batch.sh gpurun_out/c9_prof "helm tet 4 1048576" "helm hex 10 60000" "helm prism 8 100000"
