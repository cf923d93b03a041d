# c0hex step breakdown: ncu launch list (per-kernel durations) of one short bench run
mkdir -p gpurun_out/r2run75
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2run75/c0hex_launches.csv python bench.py --workload c0hex --steps 2 --warmup 1 --sweep off > gpurun_out/r2run75/c0hex.log 2>&1; echo "rc=$?"
python3 - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/r2run75/c0hex_launches.csv')))
h=[r for r in rows if r and r[0]=='ID']
if h:
    hdr=h[0]; i=rows.index(hdr)
    kn=hdr.index('Kernel Name'); mv=hdr.index('Metric Value')
    tot=collections.defaultdict(float); cnt=collections.Counter()
    for r in rows[i+1:]:
        if len(r)>mv:
            try: v=float(r[mv].replace(',',''))
            except: continue
            k=r[kn][:60]; tot[k]+=v; cnt[k]+=1
    for k,v in sorted(tot.items(), key=lambda x:-x[1])[:10]: print(f"{v/cnt[k]/1000:9.1f} us x{cnt[k]:3d}  {k}")
PY
