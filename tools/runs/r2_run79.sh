# c0tet / c0pyr / c0prism per-apply kernel durations (my kernels only)
mkdir -p gpurun_out/r2run79
for w in c0tet c0prism; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_c0|k_tile|k_persist" -c 30 --csv --log-file gpurun_out/r2run79/${w}.csv python bench.py --workload $w --steps 2 --warmup 1 --sweep off > /dev/null 2>&1; echo "$w rc=$?"
python3 - $w <<'PY'
import csv, collections, sys
w=sys.argv[1]
rows=list(csv.reader(open(f'gpurun_out/r2run79/{w}.csv')))
h=[r for r in rows if r and r[0]=='ID'][0]; i=rows.index(h)
kn=h.index('Kernel Name'); mv=h.index('Metric Value')
tot=collections.defaultdict(float); cnt=collections.Counter()
for r in rows[i+1:]:
    if len(r)<=mv: continue
    try: v=float(r[mv].replace(',',''))
    except: continue
    tot[r[kn][:60]]+=v; cnt[r[kn][:60]]+=1
for k in tot: print(f"{tot[k]/cnt[k]/1000:8.1f} us x{cnt[k]:2d}  {k}")
PY
done
