"""Summarise an ncu report: key metrics (with units), stall reasons, and
optionally a JSON of per-launch DRAM traffic for bench.py's roofline.

    python tools/ncu_summary.py REPORT [kernel-regex] [--json OUT.json]
"""
import csv
import io
import json
import re
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rep = args[0]
kre = args[1] if len(args) > 1 else "."
out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
if out_json in args:
    args.remove(out_json)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, rows = r[0], r[1], r[2:]
keys = {
    "gpu__time_duration.sum": "duration",
    "smsp__inst_executed.sum": "warp_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "pipe_lsu_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "regs",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1.0}


def si(i, row):
    """value of column i in base units (bytes, seconds) when the unit is known"""
    try:
        v = float(row[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(units[i], 1.0)


traffic = {}
for row in rows:
    name = row[hdr.index("Kernel Name")]
    if not re.search(kre, name):
        continue
    short_name = name.split("(")[0].split("::")[-1]
    print("=====", short_name)
    for k, short in keys.items():
        if k in hdr:
            i = hdr.index(k)
            print(f"  {short:22s} {row[i]} {units[i]}")
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
    if "dram__bytes_read.sum" in hdr:
        rd = si(hdr.index("dram__bytes_read.sum"), row)
        wr = si(hdr.index("dram__bytes_write.sum"), row)
        dur = si(hdr.index("gpu__time_duration.sum"), row)
        traffic.setdefault(short_name, {"dram_bytes": rd + wr, "duration_s": dur,
                                        "dram_read": rd, "dram_write": wr})
if out_json:
    with open(out_json, "w") as f:
        json.dump(traffic, f, indent=1)
    print("wrote", out_json)
