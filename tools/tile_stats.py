"""Tile-list length distribution of one view (sort / raster load balance).

    python tools/tile_stats.py [--config c4] [--view 0]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--view", type=int, default=0)
a = ap.parse_args()
sc = scenes.CONFIGS[a.config]()
dev = rz.DevicePrimitives.from_host(sc.prims)
prep = rz.prepare(dev, sc.cams[a.view])
torch.cuda.synchronize()
off = prep.tile_offsets.cpu().numpy().astype(np.int64)
c = np.diff(off)
q = np.percentile(c, [50, 90, 99, 99.9])
print(f"{a.config}: tiles {len(c)} pairs {off[-1]} mean {c.mean():.0f} p50 {q[0]:.0f} p90 {q[1]:.0f} "
      f"p99 {q[2]:.0f} p99.9 {q[3]:.0f} max {c.max()}  >8192: {(c > 8192).sum()} "
      f">32768: {(c > 32768).sum()}  items in >8192 tiles: {c[c > 8192].sum() / off[-1]:.2f}")
