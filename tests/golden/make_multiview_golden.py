"""Generate the multi-view loss fixtures (tests/golden/multiview.npz) by
running the REFERENCE qgsplat.multiview.multiview_loss (multiview.py:108).

Run in the build container (where /root/reference exists):

    python tests/golden/make_multiview_golden.py

Two seeded cameras look at a textured plane; the maps are the plane's
analytic depth / alpha / normal plus seeded noise (so the reprojection and
NCC terms are non-zero), stored as float32 and handed to the reference as
float64.  Cases: full chain on and off, RGB vs gray photos, different
neighbour size, and pixels made invalid (low alpha, zero normal, zero
depth).  Nothing on the GPU box reads /root/reference.
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

from qgsplat import multiview as mv  # noqa: E402
from qgsplat.cameras import Camera, look_at  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32)


def cam(eye, target, W, H, focal):
    return Camera(fx=focal, fy=focal * 1.05, cx=W / 2 + 0.3, cy=H / 2 - 0.2, width=W, height=H,
                  world_to_camera=look_at(eye, target))


def plane_maps(c, n_world, d_world, rng, noise, rgb):
    dirs = c.pixel_dirs_cam()
    n_cam = c.R_wc @ n_world
    d_cam = d_world - n_world @ c.center
    t = d_cam / (dirs @ n_cam)
    pw = (t[:, :, None] * dirs - c.t_wc) @ c.R_wc
    tex = 0.5 + 0.25 * np.sin(3.0 * pw[..., 0]) * np.cos(2.0 * pw[..., 1])
    img = np.stack([tex, 0.8 * tex + 0.1, 1.0 - tex], -1) if rgb else tex
    H, W = t.shape
    alpha = np.clip(0.9 + rng.normal(0, 0.03, (H, W)), 0, 1)
    normal = np.tile(-np.sign(d_cam) * n_cam, (H, W, 1)) * alpha[:, :, None]
    depth = t * alpha
    depth = depth + rng.normal(0, noise, depth.shape)
    normal = normal + rng.normal(0, noise, normal.shape)
    return {"depth": f32(depth), "alpha": f32(alpha), "normal": f32(normal), "image": f32(img)}


def main():
    rng = np.random.default_rng(2411)
    out = {}
    n_world = np.array([0.15, -0.1, 0.98])
    n_world /= np.linalg.norm(n_world)
    cases = (("p", True, False, (32, 28), (32, 28)),
             ("q", False, False, (32, 28), (32, 28)),
             ("x", True, True, (34, 30), (36, 30)))
    for tag, full, rgb, (W, H), (Wn, Hn) in cases:
        cr = cam([0.0, 0.0, 3.0], (0, 0, 0), W, H, 30.0)
        cn = cam([0.5, 0.3, 2.8], (0.05, 0, 0), Wn, Hn, 31.0)
        mr = plane_maps(cr, n_world, 0.0, rng, 0.01, rgb)
        mn = plane_maps(cn, n_world, 0.0, rng, 0.01, rgb)
        if tag == "x":
            mr["alpha"][5:8, 6:12] = 0.2          # below the alpha threshold
            mr["normal"][12, 14] = 0.0            # no normal
            mr["depth"][20, 9] = 0.0              # no depth
            mn["alpha"][10:14, 10:16] = 0.3       # neighbour samples rejected there
        cfg = mv.MultiviewConfig(full_chain=full)
        val, nv, up_r, up_n, stats = mv.multiview_loss(
            {k: v.astype(np.float64) for k, v in mr.items()}, cr,
            {k: v.astype(np.float64) for k, v in mn.items()}, cn, cfg)
        for side, m, c in (("r", mr, cr), ("n", mn, cn)):
            for k, v in m.items():
                out[f"{tag}_{side}_{k}"] = v
            out[f"{tag}_{side}_cam"] = np.array([c.fx, c.fy, c.cx, c.cy])
            out[f"{tag}_{side}_w2c"] = c.world_to_camera
        out[f"{tag}_full"] = np.int64(full)
        out[f"{tag}_value"], out[f"{tag}_n_valid"] = np.float64(val), np.int64(nv)
        out[f"{tag}_warp_px"], out[f"{tag}_ncc"] = np.float64(stats["warp_px"]), np.float64(stats["ncc"])
        for k in ("depth", "alpha", "normal"):
            out[f"{tag}_up_r_{k}"], out[f"{tag}_up_n_{k}"] = up_r[k], up_n[k]
        print(tag, "value", val, "n_valid", nv, stats)
    path = os.path.join(HERE, "multiview.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
