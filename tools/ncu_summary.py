"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, rows = r[0], r[2:]
keys = {
    "gpu__time_duration.sum": "duration_ns",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__thread_inst_executed.sum": "thread_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "regs",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
for row in rows:
    name = row[hdr.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    print("=====", name.split("(")[0])
    for k, short in keys.items():
        if k in hdr:
            print(f"  {short:22s} {row[hdr.index(k)]}")
    st = []
    for i, h in enumerate(hdr):
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio$", h)
        if m:
            try:
                v = float(row[i])
            except ValueError:
                continue
            if v > 0.05:
                st.append((v, m.group(1)))
    print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)))
