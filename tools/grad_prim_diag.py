"""Gradient of selected primitives under the backward's variants vs the
float64 oracle (diagnostics for unexplained gradient violations).

    python tools/grad_prim_diag.py --config c4 --prims 1269412 [--view 0]

Variants: default (fp32 re-shade from the logged hit point), all fragments
re-shaded from the float64 geometry (QGS_NO_FRAG_XY), deterministic fp64
reduction.  Prints each group's values and the relative error per variant.
"""
import argparse
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--view", type=int, default=0)
ap.add_argument("--prims", default="")
a = ap.parse_args()
kw = {"views": a.view + 1}
sc = scenes.CONFIGS[a.config](**kw)
cam, up = sc.cams[a.view], sc.upstream[a.view]
idx = [int(x) for x in a.prims.split(",") if x]
st = rz.RenderSettings()
prep = rz.prepare(sc.prims, cam, st)
out = {}
tg = rz.forward(prep)
out["default"] = rz.backward(prep, tg, up).to_numpy()
os.environ["QGS_NO_FRAG_XY"] = "1"
tg64 = rz.forward(prep)
out["fp64_reshade"] = rz.backward(prep, tg64, up).to_numpy()
del os.environ["QGS_NO_FRAG_XY"]
pd = dataclasses.replace(prep, settings=dataclasses.replace(st, deterministic=True))
out["deterministic"] = rz.backward(pd, tg, up).to_numpy()
tg.frag_prim = tg.frag_t = None
out["replay"] = rz.backward(prep, tg, up).to_numpy()
torch.cuda.synchronize()
vw = qo.prepare(sc.prims.astype(np.float64), cam)
ref = qo.forward(vw)
kg, kga = qo.kernel_grads(vw, ref, {k: np.asarray(v, np.float64) for k, v in up.items()},
                          with_abs=True)
rg = qo.chain(vw, kg)
for p in idx:
    print(f"=== prim {p}: kg_abs max {kga[p].max():.3e}")
    for g in ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "screen_center"):
        o = np.asarray(rg[g][p], np.float64).ravel()
        line = f"  {g:13s} ref {np.array2string(o, precision=6)}"
        for k, v in out.items():
            e = np.abs(np.asarray(v[g][p], np.float64).ravel() - o)
            line += f" | {k} {np.max(e / (1e-5 + 1e-3 * np.abs(o))):.2f}"
        print(line)
