"""Run prepare/forward/backward on one view (for ncu captures).

    python tools/profile_view.py [--config c2] [--view 0] [--reps 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--view", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
sc = scenes.CONFIGS[a.config]()
dev = rz.DevicePrimitives.from_host(sc.prims)
up = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in sc.upstream[a.view].items()}
for _ in range(a.reps):
    prep = rz.prepare(dev, sc.cams[a.view])
    tg = rz.forward(prep)
    gr = rz.backward(prep, tg, up)
torch.cuda.synchronize()
print("ok pairs", prep.n_pairs)
