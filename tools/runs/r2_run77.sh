# c0tet / c0prism step breakdown (ncu launch list)
mkdir -p gpurun_out/r2run77
for w in c0tet c0prism; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2run77/${w}_launches.csv python bench.py --workload $w --steps 2 --warmup 1 --sweep off > /dev/null 2>&1; echo "$w rc=$?"
python3 - $w <<'PY'
import csv, collections, sys
w=sys.argv[1]
rows=list(csv.reader(open(f'gpurun_out/r2run77/{w}_launches.csv')))
h=[r for r in rows if r and r[0]=='ID'][0]; i=rows.index(h)
kn=h.index('Kernel Name'); mn=h.index('Metric Name'); mv=h.index('Metric Value')
agg=collections.defaultdict(lambda: collections.defaultdict(float)); cnt=collections.Counter()
for r in rows[i+1:]:
    if len(r)<=mv: continue
    try: v=float(r[mv].replace(',',''))
    except: continue
    agg[r[kn][:70]][r[mn]]+=v
    if r[mn]=='gpu__time_duration.sum': cnt[r[kn][:70]]+=1
for k,d in sorted(agg.items(), key=lambda x:-x[1]['gpu__time_duration.sum']/max(cnt[x[0]],1))[:8]:
    n=max(cnt[k],1); print(f"{d['gpu__time_duration.sum']/n/1000:9.1f} us  rd {d['dram__bytes_read.sum']/n/1e6:8.1f} MB  wr {d['dram__bytes_write.sum']/n/1e6:7.1f} MB  x{n:3d}  {k}")
PY
done
