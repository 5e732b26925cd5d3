"""One small view through every path of the CUDA rasterizer: prepare,
forward (exact and fp32 decisions, a page pool that runs dry), backward
(atomics, deterministic, log and replay), chain, the exports.  Run with
QGS_LIB_VARIANT=debug for the bounds-checking build (tests/test_debug_checks.py).

    python tools/sanitize_view.py [--config c1] [--n N] [--res R]
"""
import argparse
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--res", type=int, default=None)
a = ap.parse_args()
kw = {}
if a.n:
    kw["n"] = a.n
if a.res:
    kw["res"] = a.res
sc = scenes.CONFIGS[a.config](**kw)
cam, up = sc.cams[0], sc.upstream[0]
check, det = [], []
for st in (rz.RenderSettings(), rz.RenderSettings(exact_decisions=False),
           rz.RenderSettings(deterministic=True), rz.RenderSettings(resort=False),
           rz.RenderSettings(euclidean_density=True, background=np.array([0.2, 0.3, 0.4]))):
    prep = rz.prepare(sc.prims, cam, st)
    tg = rz.forward(prep)
    g = rz.backward(prep, tg, up)
    check.append(float(tg.color.double().sum()))          # the forward is deterministic
    if st.deterministic:
        det.append(float(g.centers.double().abs().sum()))
    tg.frag_prim = tg.frag_t = None           # replay path
    g2 = rz.backward(prep, tg, up)
    for f in ("R", "ohat", "M", "Nmat", "wv", "lam", "view_dirs", "view_dist", "clamped",
              "color_clamped", "dirs", "scales", "alphas", "colors", "pix_bbox", "planar"):
        getattr(prep, f)
    prep.sorted_keys()
    prep.trace_pixel(cam.width // 2, cam.height // 2)
# a fragment-log pool far too small: most blocks overflow -> replay
prep = rz.prepare(sc.prims, cam)
rz._FORCE_POOL_PAGES = 8
try:
    tg = rz.forward(prep)
finally:
    rz._FORCE_POOL_PAGES = None
g3 = rz.backward(prep, tg, up)
torch.cuda.synchronize()
from paper_2411_16392_b200 import _lib  # noqa: E402
print("lib", os.path.basename(_lib.LIB_PATH))
print("det", " ".join(f"{v:.17g}" for v in det))
print("ok", prep.n_pairs, " ".join(f"{v:.17g}" for v in check))
