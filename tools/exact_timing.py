"""Raster kernel times of one C3 view with and without exact decisions."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

sc = scenes.CONFIGS["c3"]()
dev = rz.DevicePrimitives.from_host(sc.prims)
up = {k: torch.from_numpy(v).cuda() for k, v in sc.upstream[0].items()}
for ex in (False, True):
    st = rz.RenderSettings(exact_decisions=ex)
    prep = rz.prepare(dev, sc.cams[0], st)
    tg = rz.forward(prep)
    rz.backward(prep, tg, up)
    del tg                                # the timed forward reuses the cached blocks
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    tg = rz.forward(prep)
    e[1].record()
    rz.kernel_grads(prep, tg, up)
    e[2].record()
    torch.cuda.synchronize()
    print("exact", ex, "fwd ms", round(e[0].elapsed_time(e[1]), 3), "bwd ms", round(e[1].elapsed_time(e[2]), 3))
