# DMMA mass on at tet P=3 deformed: mass GPU tests + mass table
timeout 900 python -m pytest tests -m gpu -q -k "mass or Mass or streamed" 2>&1 | tail -1
timeout 1200 python bench.py --sweep on --sweep-tables mass_deformed --steps 5 > gpurun_out/r2run93_sweep.json 2>/dev/null; echo "sweep rc=$?"
python3 -c "
import json; l=json.loads(open('gpurun_out/r2run93_sweep.json').read().strip().splitlines()[-1]); t=l['per_shape_P']['mass_deformed']
for s in ['hex','prism','pyr','tet']: print(s, ' '.join(f'{r[0]}:{r[2]:.2f}' for r in t[s]))
print(t['max_parity'])"
