"""Aggregate warp-stall samples per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass`:
  python tools/ncu_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, out, tot = None, [], 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No") or not r[0]:
        continue
    try:
        s = int(r[4])
    except (ValueError, IndexError):
        continue
    out.append((s, f"{fname}:{r[0]}", r[1].strip()[:90], r[7] if len(r) > 7 else ""))
    tot += s
out.sort(reverse=True)
print(f"total samples {tot}")
for s, loc, src, inst in out[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {loc:22s} {src}")
