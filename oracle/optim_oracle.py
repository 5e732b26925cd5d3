"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU float64 numpy restatement of the reference's optimizer step and
densification (/root/reference/pkg/src/qgsplat/optim.py:14-64 and
train.py:239-335), the checker for csrc/optim.cu.  Parameter sets are dicts
of the six PrimitiveSet groups.  Pinned against fixtures produced by the
reference itself (tests/golden/optim.npz, tests/golden/make_optim_golden.py).

Only ``tests/`` may import this module; the product package never does.
"""

import numpy as np

GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")
S_MIN = 1e-4                     # model.py:16


def adam_step(p, g, m, v, t, lrs, freeze=None, beta1=0.9, beta2=0.999, eps=1e-15):
    """optim.py:23-47 (in place on p, m, v); returns the skipped count"""
    b1c, b2c = 1.0 - beta1 ** t, 1.0 - beta2 ** t
    n = len(p["centers"])
    bad = np.zeros(n, dtype=bool)
    for k in GROUPS:
        bad |= ~np.isfinite(np.asarray(g[k]).reshape(n, -1)).all(axis=1)
    for k in GROUPS:
        grad = np.array(g[k], dtype=np.float64)
        grad[bad] = 0.0
        if freeze and freeze.get(k) is not None:
            grad = np.where(freeze[k], 0.0, grad)
        m[k] = beta1 * m[k] + (1 - beta1) * grad
        v[k] = beta2 * v[k] + (1 - beta2) * grad * grad
        p[k] = p[k] - lrs[k] * (m[k] / b1c) / (np.sqrt(v[k] / b2c) + eps)
    p["quats"] = p["quats"] / np.linalg.norm(p["quats"], axis=1, keepdims=True)
    return int(bad.sum())


def accumulate_stats(stats, g_screen, g_centers):
    """train.py:239-244"""
    gn = np.linalg.norm(np.asarray(g_screen, dtype=np.float64), axis=1)
    seen = gn > 0
    stats["grad_accum"][seen] += gn[seen]
    stats["grad_count"][seen] += 1
    stats["center_accum"] += g_centers


def activate_scales(raw_scales, raw_signs):
    """model.py:29-45"""
    s = np.tanh(raw_signs) * np.exp(raw_scales)
    small = np.abs(s[..., :2]) < S_MIN
    s = s.copy()
    s[..., :2] = np.where(small, np.where(s[..., :2] < 0, -1.0, 1.0) * S_MIN, s[..., :2])
    return s


def quat_to_rot(q):
    """model.py:70-87"""
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((len(q), 3, 3))
    R[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
    R[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
    R[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
    return R


def densify_and_prune(p, m, v, stats, grad_threshold, percent_dense, extent, prune_opacity,
                      clone_nudge, max_primitives):
    """train.py:269-330; returns (p, m, v) of the new set"""
    n = len(p["centers"])
    cnt, acc = stats["grad_count"], stats["grad_accum"]
    mean = np.where(cnt > 0, acc / np.maximum(cnt, 1), 0.0)
    dens = mean > grad_threshold
    room = max_primitives - n
    if room <= 0:
        dens[:] = False
    elif dens.sum() > room:
        order = np.lexsort((np.arange(n), -mean))
        keep = np.zeros(n, dtype=bool)
        keep[order[:room]] = True
        dens &= keep
    sc = activate_scales(p["raw_scales"], p["raw_signs"])
    big = np.maximum(np.abs(sc[:, 0]), np.abs(sc[:, 1])) > percent_dense * extent
    split, clone = dens & big, dens & ~big
    sel = lambda d, mask: {k: d[k][mask] for k in GROUPS}  # noqa: E731
    parts, mparts, vparts = [sel(p, ~split)], [sel(m, ~split)], [sel(v, ~split)]
    zeros = lambda d: {k: np.zeros_like(d[k]) for k in GROUPS}  # noqa: E731
    if clone.any():
        c = sel(p, clone)
        g = stats["center_accum"][clone]
        nrm = np.linalg.norm(g, axis=1, keepdims=True)
        d = np.where(nrm > 1e-12, -g / np.maximum(nrm, 1e-12), 0.0)
        s = activate_scales(c["raw_scales"], c["raw_signs"])
        c["centers"] = c["centers"] + d * (clone_nudge * np.minimum(np.abs(s[:, 0]),
                                                                    np.abs(s[:, 1])))[:, None]
        parts.append(c)
        mparts.append(zeros(c))
        vparts.append(zeros(c))
    if split.any():
        par = sel(p, split)
        s = activate_scales(par["raw_scales"], par["raw_signs"])
        ax = (np.abs(s[:, 1]) > np.abs(s[:, 0])).astype(int)
        r = np.arange(len(ax))
        aw = quat_to_rot(par["quats"])[r, :, ax]
        off = 0.5 * np.abs(s[r, ax])[:, None] * aw
        for sign in (1.0, -1.0):
            ch = {k: par[k].copy() for k in GROUPS}
            ch["centers"] = ch["centers"] + sign * off
            ch["raw_scales"][r, ax] -= np.log(2.0)
            parts.append(ch)
            mparts.append(zeros(ch))
            vparts.append(zeros(ch))
    cat = lambda ps: {k: np.concatenate([q[k] for q in ps]) for k in GROUPS}  # noqa: E731
    p2, m2, v2 = cat(parts), cat(mparts), cat(vparts)
    keep = 1.0 / (1.0 + np.exp(-p2["raw_opacity"])) >= prune_opacity
    return sel(p2, keep), sel(m2, keep), sel(v2, keep)


def reset_opacity(raw_opacity, cap=0.01):
    """train.py:332-335"""
    a = np.minimum(1.0 / (1.0 + np.exp(-raw_opacity)), cap)
    return np.log(a / (1.0 - a))
