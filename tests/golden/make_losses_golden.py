"""Generate the loss-producer fixtures (tests/golden/losses.npz) by running
the REFERENCE qgsplat.losses / qgsplat.ssim (losses.py, ssim.py).

Run in the build container (where /root/reference exists):

    python tests/golden/make_losses_golden.py

Inputs are float32-representable (the device path reads fp32 maps) and are
handed to the reference as float64.  Cases: random images for the
photometric / SSIM terms (3- and 1-channel, both SSIM weights), a
distortion map, and a depth / alpha / normal / curvature set taken from
the c1 fixture's reference-rendered maps (depth_to_normal and the
curvature-guided consistency, guided and not).  Nothing on the GPU box
reads /root/reference.
"""

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qgs_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qgsplat import losses as ls  # noqa: E402
from qgsplat import ssim as ssim_mod  # noqa: E402
from qgsplat.cameras import Camera as RefCamera  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32)


def main():
    rng = np.random.default_rng(2411)
    out = {}
    # photometric / SSIM on random images
    x = f32(rng.uniform(0, 1, (40, 52, 3)))
    y = f32(np.clip(x + rng.normal(0, 0.08, x.shape), 0, 1))
    y[3, 4] = x[3, 4]                                   # exact ties: sign(0) = 0
    out["ph_x"], out["ph_y"] = x, y
    for tag, m in (("m02", 0.2), ("m0", 0.0), ("m1", 1.0)):
        v, g = ls.photometric(x.astype(np.float64), y.astype(np.float64), m)
        out[f"ph_{tag}_value"], out[f"ph_{tag}_grad"] = np.float64(v), g
    x1 = f32(rng.uniform(0.2, 0.8, (24, 30)))
    y1 = f32(np.clip(x1 + rng.normal(0, 0.05, x1.shape), 0, 1))
    s, gs = ssim_mod.ssim(x1.astype(np.float64), y1.astype(np.float64), return_grad=True)
    out["ss_x"], out["ss_y"], out["ss_value"], out["ss_grad"] = x1, y1, np.float64(s), gs
    # distortion
    d = f32(rng.exponential(0.01, (33, 17)))
    v, g = ls.depth_distortion(d.astype(np.float64))
    out["di_map"], out["di_value"], out["di_grad"] = d, np.float64(v), g
    # depth -> normal and the consistency loss on reference-rendered maps
    c1 = np.load(os.path.join(HERE, "c1.npz"))
    fx, fy, cx, cy = c1["cam_intr"]
    W, H = (int(v) for v in c1["cam_size"])
    cam = RefCamera(fx=fx, fy=fy, cx=cx, cy=cy, width=W, height=H, world_to_camera=c1["w2c"])
    depth = f32(c1["map_depth_median"])
    alpha = f32(c1["map_alpha"])
    normal = f32(c1["map_normal"])
    curv = f32(c1["map_curvature"])
    out.update(nc_intr=c1["cam_intr"], nc_size=c1["cam_size"], nc_w2c=c1["w2c"],
               nc_depth=depth, nc_alpha=alpha, nc_normal=normal, nc_curv=curv)
    N, mask = ls.depth_to_normal(depth.astype(np.float64), alpha.astype(np.float64), cam)
    out["nc_N"], out["nc_mask"] = N, mask
    for tag, guided in (("g", True), ("u", False)):
        v, da, dn, dk = ls.curvature_guided_normal_consistency(
            alpha.astype(np.float64), normal.astype(np.float64), curv.astype(np.float64), N,
            mask, 1e-6, guided=guided)
        out[f"nc_{tag}_value"] = np.float64(v)
        out[f"nc_{tag}_da"], out[f"nc_{tag}_dn"], out[f"nc_{tag}_dk"] = da, dn, dk
    path = os.path.join(HERE, "losses.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, "mask pixels", int(mask.sum()), "of", mask.size)


if __name__ == "__main__":
    main()
