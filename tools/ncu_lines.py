"""Aggregate warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass`:
  python tools/ncu_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, out, tot, hdr = None, [], 0, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name" or not r[0]:
        continue
    try:
        s = int(r[4])
    except (ValueError, IndexError):
        continue
    reasons = {}
    if hdr:
        for h, v in zip(hdr, r):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    if int(v) > 0:
                        reasons[h[6:]] = int(v)
                except ValueError:
                    pass
    why = " ".join(f"{k}:{v}" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:3])
    out.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], why))
    tot += s
out.sort(reverse=True)
print(f"total samples {tot}")
for s, loc, src, why in out[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {loc:22s} {src:70s} [{why}]")
