# multi-rank bench path with every per_shape_P table (two ranks sharing one GPU over gloo), c0 workloads at N=2
SK_BENCH_SHARE_GPU=1 timeout 1500 python bench.py --gpus 2 --steps 3 --warmup 3 --sweep on --sweep-quick > gpurun_out/r2run97_share2.json 2> gpurun_out/r2run97_share2.err; echo "share2 rc=$?"
python3 -c "
import json; l=json.loads(open('gpurun_out/r2run97_share2.json').read().strip().splitlines()[-1]); print(l['n_gpus'], round(l['value'],2), sorted(k for k in l['per_shape_P'] if isinstance(l['per_shape_P'][k], dict)))"
for w in c0tet c0hex; do SK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload $w > gpurun_out/r2run97_$w.json 2>/dev/null; echo "$w rc=$?"; done
tail -c 300 gpurun_out/r2run97_share2.err
