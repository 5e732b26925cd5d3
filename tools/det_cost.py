"""Cost of RenderSettings(deterministic=True): backward (kernel gradients) of
one view with fp32 atomics vs the bitwise-repeatable row reduction, CUDA
events, after warm-up.

    python tools/det_cost.py [--config c3] [--reps 5]
"""
import argparse
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
sc = scenes.CONFIGS[a.config](views=1)
dev = rz.DevicePrimitives.from_host(sc.prims)
up = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in sc.upstream[0].items()}
out = {"config": a.config}
for det in (False, True):
    st = dataclasses.replace(rz.RenderSettings(), deterministic=det)
    prep = rz.prepare(dev, sc.cams[0], st)
    tg = rz.forward(prep)
    for _ in range(2):
        rz.kernel_grads(prep, tg, up)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        kg = rz.kernel_grads(prep, tg, up)
    e1.record()
    torch.cuda.synchronize()
    out["deterministic" if det else "atomics"] = {"ms": e0.elapsed_time(e1) / a.reps,
                                                  "fragments": int(tg.n_fragments.sum().item())}
print(json.dumps(out))
