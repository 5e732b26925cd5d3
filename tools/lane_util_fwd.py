"""Lane utilisation of the forward's passes 1 and 2 (build with
QGS_NVCC_EXTRA=-DQGS_UTIL_COUNTERS=1): pass 1 tests candidates the warp's
lanes share (a lane idles on the candidates not in its pixel's mask); pass 2
runs as many iterations as the busiest lane has coarse survivors.

    python tools/lane_util_fwd.py [--config c3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
a = ap.parse_args()
sc = scenes.CONFIGS[a.config](views=1)
dev = rz.DevicePrimitives.from_host(sc.prims)
prep = rz.prepare(dev, sc.cams[0])
import ctypes  # noqa: E402
from paper_2411_16392_b200 import _lib  # noqa: E402
diag = (ctypes.c_ulonglong * 4)()
_lib.load().qgs_diag_counters(diag, 4)                   # clear
cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
rz.forward(prep, counters=cnt)
torch.cuda.synchronize()
n = _lib.load().qgs_diag_counters(diag, 4)
c = cnt.cpu().tolist()
if n >= 2:
    print(f"fp64 band re-decisions {diag[0]:.3e} ({diag[0] / max(c[4], 1):.2e} per exact test), "
          f"near-tangent fp64 roots {diag[1] & 0xffffffff:.3e}")
if n >= 4:
    print(f"coarse rejects: stage 1 {diag[2]:.3e} (of which the ray misses the quadric: "
          f"{diag[1] >> 32:.3e}), stage 2 (geodesic 3 sigma) {diag[3]:.3e}")
print(f"in-box {c[0]:.3e} conic {c[3]:.3e} coarse {c[4]:.3e} accepted {c[1]:.3e} composited {c[2]:.3e}")
if c[5]:
    print(f"pass 1: {c[3]:.3e} lane-candidates in {c[5]:.3e} lane slots -> utilisation {c[3] / c[5]:.3f}")
    print(f"pass 2: {c[4]:.3e} exact tests in {c[6]:.3e} lane slots -> utilisation {c[4] / c[6]:.3f}")
