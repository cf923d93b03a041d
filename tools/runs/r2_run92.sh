# DMMA vs sum-factorised deformed mass at tet / pyr / prism P=2-4, same box, alternating
for i in 1 2; do for d in 0 1; do SK_MASS_DENSE=$d timeout 600 python tools/sweep.py --ops mass --shapes tet,pyr,prism --orders 2-4 --gbytes 1.0 --reps 10 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('dense=$d', r['shape'], r['P'], round(r['roofline_frac'],3))"; done; done
