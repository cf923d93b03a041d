# every bench workload with the round-2 final kernels, the multi-rank path on one GPU, ncu launch list of the default bench
for w in hex4 mixed6 c0hex c0prism c0tet c0pyr tet4max; do timeout 900 python bench.py --workload $w --sweep off > gpurun_out/r2run57_$w.json 2> gpurun_out/r2run57_$w.err; echo "$w rc=$?"; done
SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --sweep off > gpurun_out/r2run57_share2.json 2> gpurun_out/r2run57_share2.err; echo "share2 rc=$?"
mkdir -p gpurun_out/r2run57
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2run57/bench_launches.csv python bench.py --steps 2 --warmup 1 --sweep off > gpurun_out/r2run57/bench_under_ncu.log 2>&1; echo "launches rc=$?"
echo done
