"""Print a compact summary of gpurun_out/{parity.json, bench_c3.json, launches_c3.csv}."""
import collections
import csv
import json
import os

D = "gpurun_out"
if os.path.exists(f"{D}/parity.json"):
    for x in json.load(open(f"{D}/parity.json")):
        if x["scene"].startswith("s_"):
            continue
        im, g = x["image"], x["grads"]
        print(x["scene"], "bin", x["tile_prims_equal"], "flip", im["count_flip_pixels"], "col",
              im["color"]["over_tol_same_count"], "gradviol", g["violations"], "/", g["n"])
for f in ("bench_c3", "bench_c2"):
    p = f"{D}/{f}.json"
    if not os.path.exists(p):
        continue
    try:
        b = json.load(open(p))
        r = b["roofline"]
        print(f, "value %.1f" % b["value"], "ms/step %.1f" % b["ms_per_step"],
              "fwd %.1f bwd %.1f" % (r["fwd_ms_per_step"], r["bwd_ms_per_step"]),
              "frac %.3f sfu %.3f roof %.3f step %.3f" % (r["frac"], r["sfu_frac"], r["roof_frac"],
                                                         r["step_roofline_frac"]),
              "e2e", b.get("e2e", {}).get("value"))
    except Exception as e:  # noqa: BLE001
        print(f, "ERROR", e, open(f"{D}/{f}.err").read()[-600:])
p = f"{D}/launches_c3.csv"
if os.path.exists(p):
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    data = data[len(data) // 2:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    for r in data:
        tot[r[ki].split("(")[0].replace("void ", "")[:40]] += float(r[vi].replace(",", "")) / 1e6
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:6]:
        print("  %-40s %7.2f ms" % (k, v))
