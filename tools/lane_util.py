"""Lane utilisation of the per-block loops: for each 8x4 raster block, the
composited fragments of its pixels over 32 x the deepest pixel (the
backward's steps), for one view.

    python tools/lane_util.py [--config c3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
a = ap.parse_args()
sc = scenes.CONFIGS[a.config]()
cam = sc.cams[0]
tg = rz.forward(rz.prepare(rz.DevicePrimitives.from_host(sc.prims), cam), keep_aux=False)
nf = tg.n_fragments.cpu().numpy()
H, W = nf.shape
Hp, Wp = (H + 3) // 4 * 4, (W + 7) // 8 * 8
pad = np.zeros((Hp, Wp), np.int64)
pad[:H, :W] = nf
blk = pad.reshape(Hp // 4, 4, Wp // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
tot, steps = blk.sum(), (blk.max(axis=1) * 32).sum()
print(f"fragments {tot}, block steps x32 {steps}, backward lane utilisation {tot / steps:.3f}")
print("mean/max per block quantiles:", np.percentile(blk.mean(1) / np.maximum(blk.max(1), 1), [10, 50, 90]))
