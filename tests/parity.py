"""Parity comparators: GPU outputs vs the float64 oracle.

Images: max-abs <= 1e-4 on colour / alpha / depth / normal.  Any pixel over
tolerance is classified: a COUNT FLIP when n_fragments differs (a
termination / alpha-floor / 3-sigma decision flipped between fp32 and fp64),
otherwise SAME-COUNT (an order swap of near-tied depths, a membership change,
or an unexplained continuous error).

Gradients: elementwise |g - o| <= 1e-5 + 1e-3 |o| (allclose semantics).
"""

import numpy as np

IMG_TOL = 1e-4
GRAD_RTOL = 1e-3
GRAD_ATOL = 1e-5
IMG_MAPS = ("color", "alpha", "depth", "normal")
GRAD_GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")


def image_report(gpu, ref):
    """gpu, ref: dicts of (H,W[,3]) maps incl. n_fragments."""
    flips = np.asarray(gpu["n_fragments"]) != np.asarray(ref["n_fragments"])
    out = {"count_flip_pixels": int(flips.sum())}
    bad_any = np.zeros(flips.shape, dtype=bool)
    for k in IMG_MAPS + ("depth_median", "transmittance", "curvature", "distortion"):
        d = np.abs(np.asarray(gpu[k], dtype=np.float64) - np.asarray(ref[k], dtype=np.float64))
        if d.ndim == 3:
            d = d.max(axis=2)
        bad = d > IMG_TOL
        if k in IMG_MAPS:
            bad_any |= bad
        r = np.abs(np.asarray(ref[k], dtype=np.float64))
        if r.ndim == 3:
            r = r.max(axis=2)
        rel = d / np.maximum(r, 1.0)            # relative where the map is large (curvature)
        out[k] = {"max_abs": float(d.max()) if d.size else 0.0,
                  "max_abs_same_count": float(d[~flips].max()) if (~flips).any() else 0.0,
                  "max_rel_same_count": float(rel[~flips].max()) if (~flips).any() else 0.0,
                  "rel_over_1e-4_same_count": int(((rel > 1e-4) & ~flips).sum()),
                  "rel_over_1e-3_same_count": int(((rel > 1e-3) & ~flips).sum()),
                  "over_tol": int(bad.sum()), "over_tol_count_flip": int((bad & flips).sum()),
                  "over_tol_same_count": int((bad & ~flips).sum())}
    out["pixels"] = int(flips.size)
    out["over_tol_pixels"] = int(bad_any.sum())
    out["over_tol_same_count"] = int((bad_any & ~flips).sum())
    return out


def grad_report(gpu, ref):
    out = {}
    tot_bad = tot = 0
    for k in GRAD_GROUPS + ("screen_center",):
        g = np.asarray(gpu[k], dtype=np.float64).ravel()
        o = np.asarray(ref[k], dtype=np.float64).ravel()
        err = np.abs(g - o)
        bad = err > GRAD_ATOL + GRAD_RTOL * np.abs(o)
        scale = np.abs(o).max() if o.size else 0.0
        out[k] = {"violations": int(bad.sum()), "n": int(g.size),
                  "max_err": float(err.max()) if err.size else 0.0,
                  "group_rel": float(err.max() / scale) if scale > 0 else 0.0}
        if k in GRAD_GROUPS:
            tot_bad += int(bad.sum())
            tot += int(g.size)
    out["violations"] = tot_bad
    out["n"] = tot
    return out
