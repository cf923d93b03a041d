"""Per-opcode and per-barrier-segment breakdown of an ncu source page
(--page source --print-source sass --csv): instructions and warp stall
samples.  python tools/sass_breakdown.py <sass.csv> <elements>"""

import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
E = int(sys.argv[2])
hdr, data = rows[1], rows[2:]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
tot = totst = 0
seg, cur, after = [], [0, 0, 0], []
for idx, r in enumerate(data):
    src = r[iS].strip()
    n, st = int(r[iE] or 0), int(r[iW] or 0)
    tok = src.split()
    op = (tok[1] if tok and tok[0].startswith("@") else tok[0]) if tok else "?"
    base = op.split(".")[0]
    ops[base] += n
    stall[base] += st
    tot += n
    totst += st
    cur[0] += n
    cur[1] += st
    if base in ("DFMA", "DMUL", "DADD"):
        cur[2] += n
    if base == "BAR":
        seg.append(tuple(cur))
        cur = [0, 0, 0]
        after.append(int(data[idx + 1][iW] or 0))
seg.append(tuple(cur))
print(rows[0][1][:200])
fp = ops["DFMA"] + ops["DMUL"] + ops["DADD"]
print(f"warp instructions per element {tot / E:.1f}, FP64 {fp / E:.1f} ({100 * fp / tot:.1f} %), stall samples {totst}")
for k, v in ops.most_common(16):
    print(f"  {k:8s} {v / E:9.1f}/el {100 * v / tot:5.1f}% inst {100 * stall[k] / totst:5.1f}% stalls")
print("segments between CTA barriers (inst/el, stall share incl. the wait at its start, FP64/el):")
for i, s in enumerate(seg):
    print(f"  seg{i:2d} {s[0] / E:9.1f} {100 * s[1] / totst:5.1f}% {s[2] / E:8.1f}")
print(f"stall samples on the instruction after each BAR.SYNC: {100 * sum(after) / totst:.1f}%")
top = sorted(((int(r[iW] or 0), i, r[iS].strip()[:70]) for i, r in enumerate(data)), reverse=True)[:12]
for st, i, src in top:
    print(f"  {100 * st / totst:5.1f}%  #{i:5d}  {src}")
