"""Gradient parity of the backward's two re-shading paths (fp32 from the
logged hit point vs float64 geometry) against the reference golden fixtures.

    python tools/grad_xy_check.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz  # noqa: E402
from tests import golden_io, parity  # noqa: E402

for name in golden_io.names():
    gc = golden_io.load(name)
    if "grad_centers" not in gc.g:
        continue
    s = gc.settings
    st = rz.RenderSettings(background=np.asarray(s.background), resort=s.resort,
                           euclidean_density=s.euclidean_density)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    ref = {k: gc.g[f"grad_{k}"] for k in parity.GRAD_GROUPS + ("screen_center",)}
    out = []
    for mode in ("xy", "fp64"):
        if mode == "fp64":
            tg.frag_xy = None
        gr = rz.backward(prep, tg, gc.upstream)
        torch.cuda.synchronize()
        rep = parity.grad_report(gr.to_numpy(), ref)
        out.append(f"{mode}: {rep['violations']}/{rep['n']} worst group-rel "
                   f"{max(rep[k]['group_rel'] for k in parity.GRAD_GROUPS):.2e}")
    print(f"{name:14s}", " | ".join(out))
