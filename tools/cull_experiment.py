"""Design experiment: how many in-box candidates survive a per-pixel bounding
ellipsoid test, against how many the reference's selection rule accepts.

    python tools/cull_experiment.py [--config c3] [--pixels 300]

For a sample of pixels of view 0: in-box primitives (reference pixel boxes),
those whose ray meets the bounding ellipsoid of the accepted patch (see
DESIGN.md section 4, "conic cull"), and those the selection rule
(intersect.py:58-115, alpha floor raster_kernels.py:58-60) accepts.  Ignores
early termination (it removes the same fraction from every count).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import scenes  # noqa: E402


def arc(a, rho):
    u = 2 * a * rho
    out = rho.copy()
    big = np.abs(u) >= 1e-3
    ub, ab = u[big], a[big]
    r = np.sqrt(ub * ub + 1)
    out[big] = (np.sign(ub) * np.log(np.abs(ub) + r) + ub * r) / (4 * ab)
    return out


def accept(vw, idx, d, t_clip=0.01):
    """vectorised selection rule for primitives idx and one camera ray d"""
    M, o = vw.M[idx], vw.ohat[idx]
    w1, w2, iw3 = vw.wv[idx].T
    s1, s2, s3 = vw.scales[idx].T
    pl = vw.planar[idx] == 1
    dh = M @ d
    A = w1 * dh[:, 0] ** 2 + w2 * dh[:, 1] ** 2
    B = 2 * (w1 * o[:, 0] * dh[:, 0] + w2 * o[:, 1] * dh[:, 1]) - iw3 * dh[:, 2]
    C = w1 * o[:, 0] ** 2 + w2 * o[:, 1] ** 2 - iw3 * o[:, 2]
    lin = np.abs(A) < 1e-6
    disc = B * B - 4 * A * C
    sq = np.sqrt(np.maximum(disc, 0))
    sa = np.where(A > 0, 1.0, -1.0)
    with np.errstate(all="ignore"):
        r0 = np.where(lin, -C / B, (-B - sa * sq) / (2 * A))
        r1 = np.where(lin, np.nan, (-B + sa * sq) / (2 * A))
        r0 = np.where(pl, -o[:, 2] / dh[:, 2], r0)
        r1 = np.where(pl, np.nan, r1)
    ok = np.where(pl, np.abs(dh[:, 2]) >= 1e-12, np.where(lin, np.abs(B) >= 1e-12, disc >= 0))
    acc = np.zeros(len(idx), bool)
    done = np.zeros(len(idx), bool)
    for r in (r0, r1):
        with np.errstate(all="ignore"):
            x = o[:, 0] + r * dh[:, 0]
            y = o[:, 1] + r * dh[:, 1]
            rho = np.sqrt(x * x + y * y)
            c = np.where(rho > 1e-12, x / np.where(rho > 0, rho, 1), 1.0)
            s = np.where(rho > 1e-12, y / np.where(rho > 0, rho, 1), 0.0)
            a = np.where(pl, 0.0, s3 * (w1 * c * c + w2 * s * s))
            l = np.where(pl, rho, arc(a, rho))
            sig = s1 * s2 / np.sqrt((s2 * c) ** 2 + (s1 * s) ** 2)
            sig = np.abs(sig)
            ell = (x / (3 * s1)) ** 2 + (y / (3 * s2)) ** 2 <= 1
            valid = ok & (r > t_clip) & (pl | ell) & (l <= 3 * sig) & ~done
            G = np.exp(-l * l / (2 * sig * sig))
        acc |= valid & (vw.alphas[idx] * G >= 1.0 / 255.0)
        done |= valid
    return acc


def ellipsoids(vw):
    """per primitive: two bounding ellipsoids (centre z, semi-axes) in the local frame"""
    s = np.abs(vw.scales)
    s1, s2, s3 = s.T
    smax = np.maximum(s1, s2)
    # (1) chord bound: rho^2 + z^2 <= l^2 <= 9 sigma^2  ->  semi-axes 3s1, 3s2, 3smax
    e1 = np.stack([np.zeros_like(s1), 3 * s1, 3 * s2, 3 * smax], 1)
    # (2) cylinder x slab: z = s3 (w1 x^2 + w2 y^2) in [zlo, zhi]; lambda-blend
    sg1 = np.sign(vw.wv[:, 0]) * np.sign(vw.scales[:, 2])
    sg2 = np.sign(vw.wv[:, 1]) * np.sign(vw.scales[:, 2])
    zmax = 9 * s3
    zhi = np.where((sg1 > 0) | (sg2 > 0), zmax, 0.0)
    zlo = np.where((sg1 < 0) | (sg2 < 0), -zmax, 0.0)
    zhi = np.minimum(zhi, 3 * smax)
    zlo = np.maximum(zlo, -3 * smax)
    h = np.maximum((zhi - zlo) / 2, 1e-9)
    lam = 0.8
    e2 = np.stack([(zhi + zlo) / 2, 3 * s1 / np.sqrt(lam), 3 * s2 / np.sqrt(lam),
                   h / np.sqrt(1 - lam)], 1)
    return e1, e2


def hits(vw, idx, d, e):
    M, o = vw.M[idx], vw.ohat[idx].copy()
    ee = e[idx]
    o[:, 2] -= ee[:, 0]
    dh = M @ d
    o2 = o / ee[:, 1:]
    d2 = dh / ee[:, 1:]
    dd = (d2 * d2).sum(1)
    oo = (o2 * o2).sum(1)
    od = (o2 * d2).sum(1)
    return oo * dd - od * od <= dd * 1.0001


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--pixels", type=int, default=300)
    a = ap.parse_args()
    sc = scenes.CONFIGS[a.config]()
    cam = sc.cams[0]
    prims64 = sc.prims.astype(np.float64)
    vw = qo.prepare(prims64, cam, tile_subset=[0])
    box = vw.pix_bbox
    e1, e2 = ellipsoids(vw)
    rng = np.random.default_rng(0)
    us = rng.integers(0, cam.width, a.pixels)
    vs = rng.integers(0, cam.height, a.pixels)
    dirs = cam.pixel_dirs() if hasattr(cam, "pixel_dirs") else qo.Cam(cam).pixel_dirs()
    tot = np.zeros(5)
    for u, v in zip(us, vs):
        idx = np.nonzero((box[:, 0] <= u) & (u <= box[:, 1]) & (box[:, 2] <= v) & (v <= box[:, 3]))[0]
        if len(idx) == 0:
            continue
        d = dirs[v, u]
        h1 = hits(vw, idx, d, e1)
        h2 = hits(vw, idx, d, e2)
        acc = accept(vw, idx, d)
        assert not np.any(acc & ~h1), "ellipsoid 1 not conservative"
        assert not np.any(acc & ~h2), "ellipsoid 2 not conservative"
        tot += [len(idx), h1.sum(), h2.sum(), (h1 & h2).sum(), acc.sum()]
    n = a.pixels
    print(f"per pixel: in-box {tot[0]/n:.1f}  chord-ellipsoid {tot[1]/n:.1f}  "
          f"slab-ellipsoid {tot[2]/n:.1f}  both {tot[3]/n:.1f}  accepted {tot[4]/n:.1f}")


if __name__ == "__main__":
    main()
