"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [N]
"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
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
        samp = int(row[hdr.index("# Samples")])
        ex = int(row[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    key = (cur, int(row[0]))
    a = agg.setdefault(key, [0, 0, row[1][:70]])
    a[0] += samp
    a[1] += ex
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts}  warp-inst {te:.3e}")
for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{s / ts * 100:5.1f}% samp {e / te * 100:5.1f}% inst  {f}:{ln:<4d} {src}")
