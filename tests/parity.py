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


def over_tol_mask(gpu, ref):
    """pixels over IMG_TOL on any of colour / alpha / depth / normal"""
    bad = np.zeros(np.asarray(ref["alpha"]).shape, dtype=bool)
    for k in IMG_MAPS:
        d = np.abs(np.asarray(gpu[k], dtype=np.float64) - np.asarray(ref[k], dtype=np.float64))
        bad |= (d.max(axis=2) if d.ndim == 3 else d) > IMG_TOL
    return bad


def classify_stream(g_prims, o_prims):
    """SURVEY.md 8(c).3 class of one pixel from its two emitted streams
    (primitive ids in compositing order, GPU vs oracle)."""
    g, o = np.asarray(g_prims), np.asarray(o_prims)
    if len(g) != len(o):
        return "count_flip"
    if np.array_equal(g, o):
        return "continuous"            # same fragments, same order: unexplained
    if np.array_equal(np.sort(g), np.sort(o)):
        return "order_swap"
    return "membership"


def classify_pixels(prep, vw, gpu, ref, mask=None, limit=400):
    """Classify every pixel of `mask` (default: over tolerance) by comparing
    the GPU's emitted stream (PreparedView.trace_pixel: the same inline
    functions as the raster kernels) with the oracle's (qgs_oracle.trace_pixel:
    the C restatement of forward_kernel).  Returns counts per class plus the
    first few pixels of each class; pixels beyond `limit` count as
    'unclassified'."""
    from oracle import qgs_oracle as qo
    mask = over_tol_mask(gpu, ref) if mask is None else mask
    vs, us = np.nonzero(mask)
    out = {"count_flip": 0, "order_swap": 0, "membership": 0, "continuous": 0,
           "unclassified": 0, "examples": {}}
    for i, (v, u) in enumerate(zip(vs.tolist(), us.tolist())):
        if i >= limit:
            out["unclassified"] += 1
            continue
        if int(np.asarray(gpu["n_fragments"])[v, u]) != int(np.asarray(ref["n_fragments"])[v, u]):
            c = "count_flip"
        else:
            _, ge = prep.trace_pixel(u, v)
            _, oe = qo.trace_pixel(vw, u, v)
            c = classify_stream(ge["prim"], oe["prim"])
        out[c] += 1
        out["examples"].setdefault(c, [])
        if len(out["examples"][c]) < 4:
            out["examples"][c].append((u, v))
    return out


def median_flips(prep, vw, gpu, ref, tol=IMG_TOL, band=1e-5, limit=200):
    """depth_median is t of the last fragment composited while T > 0.5
    (raster_kernels.py:152): a discontinuous decision.  Same-count pixels
    whose median differs by more than `tol` must be T = 0.5 crossings within
    `band` in the oracle's own stream (or differ in their streams).  Returns
    (n_mismatch, n_unexplained)."""
    from oracle import qgs_oracle as qo
    same = np.asarray(gpu["n_fragments"]) == np.asarray(ref["n_fragments"])
    d = np.abs(np.asarray(gpu["depth_median"], np.float64) - np.asarray(ref["depth_median"], np.float64))
    vs, us = np.nonzero((d > tol) & same)
    bad = 0
    for i, (v, u) in enumerate(zip(vs.tolist(), us.tolist())):
        if i >= limit:
            bad += 1
            continue
        _, oe = qo.trace_pixel(vw, u, v)
        _, ge = prep.trace_pixel(u, v)
        if classify_stream(ge["prim"], oe["prim"]) != "continuous":
            continue                  # a different stream explains it
        T = np.asarray(oe["T"])       # T before each fragment
        if not np.any(np.abs(T - 0.5) <= band):
            bad += 1
    return len(vs), bad


def count_flip_prims(prep, vw, gpu, ref, limit=400):
    """Primitives composited (by either side) at pixels whose fragment count
    differs between the GPU and the oracle: their gradients legitimately
    differ by the flipped fragments' contributions."""
    from oracle import qgs_oracle as qo
    vs, us = np.nonzero(np.asarray(gpu["n_fragments"]) != np.asarray(ref["n_fragments"]))
    out = set()
    for v, u in list(zip(vs.tolist(), us.tolist()))[:limit]:
        _, ge = prep.trace_pixel(u, v)
        _, oe = qo.trace_pixel(vw, u, v)
        out.update(int(p) for p in ge["prim"])
        out.update(int(p) for p in oe["prim"])
    return out


def grad_conditioning(vw, gpu, ref, kg_abs, rel=1e-5, flip_prims=()):
    """Classify gradient elements over the 1e-3 rel / 1e-5 abs tolerance by
    their cancellation scale: bound_e = sum_j |d g_e / d slot_j| * A_j, with
    A_j = sum over the primitive's fragments of |contribution to slot j|
    (oracle kernel_grads(with_abs=True)) and the chain's exact Jacobian
    (qgs_oracle.chain_jacobian).  An fp32 gradient of fragments that each
    carry ~1e-7..1e-6 relative error cannot resolve an element below
    ~1e-6 * bound_e; a violation with |err| <= rel * bound_e is
    'cancellation-limited', otherwise 'unexplained'."""
    from oracle import qgs_oracle as qo
    viol = {}
    for k in GRAD_GROUPS + ("screen_center",):
        g = np.asarray(gpu[k], dtype=np.float64)
        o = np.asarray(ref[k], dtype=np.float64)
        P = o.shape[0]
        g, o = g.reshape(P, -1), o.reshape(P, -1)
        bad = np.abs(g - o) > GRAD_ATOL + GRAD_RTOL * np.abs(o)
        viol[k] = (np.nonzero(bad), g, o)
    prims = sorted({int(p) for (pi, _), _, _ in viol.values() for p in pi})
    out = {"violations": sum(len(v[0][0]) for v in viol.values()), "cancellation_limited": 0,
           "count_flip": 0, "unexplained": 0, "max_err_over_bound": 0.0, "examples": []}
    if not prims:
        return out
    J = qo.chain_jacobian(vw, prims)
    row = {p: i for i, p in enumerate(prims)}
    for k, ((pi, ci), g, o) in viol.items():
        for p, c in zip(pi.tolist(), ci.tolist()):
            b = float(np.abs(J[k][row[p], c]) @ kg_abs[p])
            err = abs(g[p, c] - o[p, c])
            ratio = err / b if b > 0 else np.inf
            out["max_err_over_bound"] = max(out["max_err_over_bound"], ratio)
            if ratio <= rel:
                out["cancellation_limited"] += 1
            elif p in flip_prims:
                out["count_flip"] += 1
            else:
                out["unexplained"] += 1
                if len(out["examples"]) < 8:
                    out["examples"].append({"group": k, "prim": p, "comp": c, "err": err,
                                            "ref": o[p, c], "bound": b})
    return out
