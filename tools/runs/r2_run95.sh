timeout 900 python -m pytest tests -m gpu -q -k "mass or Mass or streamed or regular" 2>&1 | tail -1
timeout 600 python tools/sweep.py --ops mass --geo regular --shapes hex --orders 2-4 --gbytes 1.0 --reps 10 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print(r['shape'], r['P'], round(r['roofline_frac'],3))"
