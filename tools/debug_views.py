"""Run prepare / forward / backward view by view with a sync and a print
after each stage (locates a stage that fails or does not finish).

    python tools/debug_views.py [--config c3] [--no-cull]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--no-cull", action="store_true")
ap.add_argument("--counters", action="store_true")
a = ap.parse_args()
sc = scenes.CONFIGS[a.config]()
dev = rz.DevicePrimitives.from_host(sc.prims)
st = rz.RenderSettings(conic_cull=not a.no_cull)
for v, cam in enumerate(sc.cams):
    up = {k: torch.from_numpy(np.ascontiguousarray(x)).cuda() for k, x in sc.upstream[v].items()}
    t0 = time.time()
    prep = rz.prepare(dev, cam, st)
    torch.cuda.synchronize()
    print(f"view {v} prepare ok pairs={prep.n_pairs} {time.time() - t0:.3f}s", flush=True)
    cnt = torch.zeros(5, dtype=torch.int64, device="cuda") if a.counters else None
    tg = rz.forward(prep, counters=cnt)
    torch.cuda.synchronize()
    print(f"view {v} forward ok max_frag={int(tg.n_fragments.max())} cnt={None if cnt is None else cnt.tolist()} {time.time() - t0:.3f}s", flush=True)
    kg = rz.kernel_grads(prep, tg, up)
    torch.cuda.synchronize()
    print(f"view {v} backward ok {time.time() - t0:.3f}s", flush=True)
