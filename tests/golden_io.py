"""Load the committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference implementation)."""

import glob
import os
from types import SimpleNamespace

import numpy as np

from paper_2411_16392_b200.cameras import Camera
from paper_2411_16392_b200.model import PrimitiveSet

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
UP_KEYS = ("color", "alpha", "depth", "normal", "curvature", "distortion")


def names():
    # scenes only (losses / optim / multiview fixtures belong to their own tests)
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if os.path.basename(p) not in ("losses.npz", "optim.npz", "multiview.npz"))


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    g = {k: z[k] for k in z.files}
    prims = PrimitiveSet(*(g[k].astype(np.float64) for k in
                           ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")))
    fx, fy, cx, cy = g["cam_intr"]
    W, H = (int(v) for v in g["cam_size"])
    cam = Camera(fx=fx, fy=fy, cx=cx, cy=cy, width=W, height=H, world_to_camera=g["w2c"])
    st = SimpleNamespace(background=tuple(g["background"]), t_near_clip=0.01,
                         alpha_floor=1.0 / 255.0, alpha_clamp=0.999, t_term=1e-4,
                         resort=bool(g["resort"]), euclidean_density=bool(g["euclid"]))
    up = {k: g[f"up_{k}"].astype(np.float64) for k in UP_KEYS if f"up_{k}" in g}
    return SimpleNamespace(prims=prims, cam=cam, settings=st, upstream=up, g=g)
