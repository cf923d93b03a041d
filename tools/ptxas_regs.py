"""Compile one (shape, order) translation unit with -Xptxas -v and print
registers / spills per kernel:  python tools/ptxas_regs.py 3 4 [extra nvcc flags]"""
import re
import subprocess
import sys
import os

csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2604_04644_b200", "csrc")
S, P = sys.argv[1], sys.argv[2]
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
       f"-DSK_S={S}", f"-DSK_P={P}", "-c", "inst.cu", "-o", f"/tmp/ptxas_{S}_{P}.o"] + sys.argv[3:]
out = subprocess.run(cmd, cwd=csrc, capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = (m.group(1), m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        k = re.search(r"k_(?:tile|persist)INS_\d+(k_\w+?)I", name)
        if k:
            short = k.group(1) + " " + re.sub(r"ILi|Li|E|NS_|Lb", " ", name[name.index(k.group(1)) + len(k.group(1)):][:90])
            print(f"{m.group(1):>4} regs  spill {spill[0]}/{spill[1]}  {short}")
        name = None
if "error" in out:
    print(out[-3000:])
