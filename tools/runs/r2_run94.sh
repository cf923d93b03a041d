# DMMA vs sum-factorised re-check, same box: regular Helmholtz / stiffness (SK_HELM_DENSE) and regular mass (SK_MASS_DENSE), P=2-6
for d in 0 1; do SK_HELM_DENSE=$d timeout 900 python tools/sweep.py --ops helm,stiff --geo regular --orders 2-6 --gbytes 1.0 --reps 10 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('helmdense=$d', r['op'], r['shape'], r['P'], round(r['roofline_frac'],3))"; done
for d in 0 1; do SK_MASS_DENSE=$d timeout 900 python tools/sweep.py --ops mass --geo regular --orders 2-6 --gbytes 1.0 --reps 10 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    r=json.loads(l); print('massdense=$d', r['op'], r['shape'], r['P'], round(r['roofline_frac'],3))"; done
