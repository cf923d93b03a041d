"""Summarise `ncu --page raw --csv` exports: time, DRAM, pipes, occupancy,
stall reasons (pc-sampling counts, descending).

  python tools/ncu_summary.py gpurun_out/prof1/*_raw.csv
"""

import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__bytes_read.sum.per_second", "dram_rd_bw"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "threads"),
    ("launch__shared_mem_per_block_dynamic", "smem/blk"),
    ("launch__occupancy_limit_registers", "occ_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_smem"),
    ("launch__occupancy_limit_warps", "occ_warps"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__func_cache_config", "cache"),
]


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        summarise_row(path, hdr, units, vals)


def summarise_row(path, hdr, units, vals):
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(f"== {path}  {d.get('Kernel Name', '')[:140]}")
    for k, name in KEYS:
        if k in d:
            print(f"  {name:16s} {d[k]} {u[k]}")
    for h, v in d.items():  # tensor-pipe (DMMA) activity, when the kernel uses it
        if "pipe_tensor" in h and "pct_of_peak_sustained_active" in h and v not in ("", "0"):
            print(f"  {h[:60]:60s} {v} {u[h]}")
    stalls = []
    for h, v in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    print("  stalls: " + ", ".join(f"{n} {s / tot:.0%}" for s, n in sorted(stalls, reverse=True)[:8]))


for p in sys.argv[1:]:
    summarise(p)
