"""Bucket an ncu source-page profile of the forward / backward raster kernel
into phases by source line ranges (inlined device functions count where
they are defined).

    python tools/ncu_phases.py REPORT KERNEL_REGEX
"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
# (file, first line, last line, phase)
RANGES = [
    ("shade.cuh", 1, 103, "shade helpers (arc/eval/ellipse)"),
    ("shade.cuh", 104, 173, "shade_at / shade_from_log"),
    ("shade.cuh", 174, 277, "exact: refine/confirm/marginal"),
    ("shade.cuh", 278, 370, "coarse stage 1/2"),
    ("shade.cuh", 371, 413, "exact: hit_exact_from/refined"),
    ("shade.cuh", 414, 439, "normal_curv32"),
    ("shade.cuh", 440, 9999, "pixel dir / box"),
    ("raster_warp.cu", 1, 199, "staging / block masks / conic rows"),
    ("raster_warp.cu", 199, 320, "ring"),
    ("raster_warp.cu", 320, 441, "frag helpers / setup"),
    ("raster_warp.cu", 442, 493, "fwd composite"),
    ("raster_warp.cu", 494, 559, "fwd pass 1 loop"),
    ("raster_warp.cu", 560, 611, "fwd pass 2 (exact+accept)"),
    ("raster_warp.cu", 612, 693, "fwd pass 0 (list, conic queue)"),
    ("raster_warp.cu", 694, 770, "fwd drain / epilogue"),
    ("raster_warp.cu", 770, 99999, "backward body"),
]
cur, hdr, agg = None, None, {}
tot_s = tot_e = 0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit() or row[2] != "-":
        continue
    try:
        s = int(row[hdr.index("# Samples")])
        e = int(row[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    ln = int(row[0])
    ph = next((p for f, a, b, p in RANGES if f == cur and a <= ln <= b), f"{cur} other")
    v = agg.setdefault(ph, [0, 0])
    v[0] += s
    v[1] += e
    tot_s += s
    tot_e += e
for ph, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{100 * s / max(tot_s, 1):5.1f}% samples {100 * e / max(tot_e, 1):5.1f}% inst  {ph}")
