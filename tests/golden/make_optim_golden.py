"""Generate the optimizer / densification fixtures (tests/golden/optim.npz)
by running the REFERENCE qgsplat.optim.Adam and the reference trainer's
densify_and_prune / reset_opacity (train.py:269-335) on seeded state.

Run in the build container (where /root/reference exists):

    python tests/golden/make_optim_golden.py

Parameters, gradients and statistics are float32-representable (the device
path holds fp32 groups) and handed to the reference as float64.  The
trainer methods are called unbound on a minimal stand-in object carrying
exactly the attributes they read.  Nothing on the GPU box reads
/root/reference.
"""

import os
import sys
import tempfile
import types

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qgs_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from qgsplat import optim as ropt  # noqa: E402
from qgsplat.config import TrainConfig  # noqa: E402
from qgsplat.model import PrimitiveSet  # noqa: E402
from qgsplat.train import Trainer  # noqa: E402

FIELDS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def prims(rng, n, k=4):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return PrimitiveSet(
        f32(rng.normal(0, 1, (n, 3))), f32(q), f32(rng.normal(-3.5, 1.0, (n, 3))),
        f32(rng.normal(0, 1.5, (n, 3))), f32(rng.normal(0, 2.5, n)),
        f32(rng.normal(0, 0.5, (n, 3, k))))


def dump(out, tag, ps):
    for f in FIELDS:
        out[f"{tag}_{f}"] = getattr(ps, f).copy()


class Grads:
    pass


def main():
    rng = np.random.default_rng(16392)
    out = {}
    # ---- Adam: three steps, a non-finite gradient row in step 2, s3 frozen
    ps = prims(rng, 300)
    dump(out, "adam_in", ps)
    opt = ropt.Adam(ps)
    lrs = {"centers": 1.6e-4, "quats": 1e-3, "raw_scales": 5e-3, "raw_signs": 5e-3,
           "raw_opacity": 0.05, "sh": 2.5e-3}
    freeze = {"raw_scales": np.zeros((300, 3), bool), "raw_signs": np.zeros((300, 3), bool)}
    freeze["raw_scales"][:, 2] = True
    freeze["raw_signs"][:, 2] = True
    for s in range(3):
        g = Grads()
        for f in FIELDS:
            setattr(g, f, f32(rng.normal(0, 0.1, getattr(ps, f).shape)))
        if s == 1:
            g.sh[7, 1, 2] = np.nan
            g.centers[42, 0] = np.inf
        for f in FIELDS:
            out[f"adam_g{s}_{f}"] = getattr(g, f).copy()
        opt.step(ps, g, lrs, freeze=freeze if s > 0 else None)
        dump(out, f"adam_s{s}", ps)
    out["adam_skipped"] = np.int64(opt.skipped)
    for f in FIELDS:
        out[f"adam_m_{f}"], out[f"adam_v_{f}"] = opt.m[f].copy(), opt.v[f].copy()

    # ---- densify_and_prune: clones, splits, prunes; then a binding budget
    # with tied mean gradients; then no room at all
    for tag, n, max_prims in (("dp", 400, 5000), ("dr", 400, 400 + 23), ("dn", 200, 150)):
        ps = prims(rng, n)
        ps.raw_opacity[::9] = -8.0                      # prune these (alpha < 0.005)
        cnt = f32(rng.integers(0, 4, n))
        acc = f32(rng.uniform(0, 1.0, n) * cnt)
        if tag == "dr":
            acc[::5] = 0.75 * cnt[::5]                   # tied means at 0.75
        cacc = f32(rng.normal(0, 1e-3, (n, 3)))
        cacc[3] = 0.0                                    # clone without a direction
        opt = ropt.Adam(ps)
        for f in FIELDS:
            opt.m[f] = f32(rng.normal(0, 1e-3, opt.m[f].shape))
            opt.v[f] = f32(rng.uniform(0, 1e-6, opt.v[f].shape))
        cfg = TrainConfig(max_primitives=max_prims, densify_grad_threshold=0.3,
                          percent_dense=0.01, prune_opacity=0.005, clone_nudge=0.5)
        dump(out, f"{tag}_in", ps)
        for f in FIELDS:
            out[f"{tag}_in_m_{f}"], out[f"{tag}_in_v_{f}"] = opt.m[f].copy(), opt.v[f].copy()
        out[f"{tag}_grad_accum"], out[f"{tag}_grad_count"] = acc, cnt
        out[f"{tag}_center_accum"] = cacc
        me = types.SimpleNamespace(cfg=cfg, prims=ps, extent=3.0, opt=opt, grad_accum=acc.copy(),
                                   grad_count=cnt.copy(), center_accum=cacc.copy())
        me._reset_stats = types.MethodType(Trainer._reset_stats, me)
        Trainer.densify_and_prune(me)
        dump(out, f"{tag}_out", me.prims)
        for f in FIELDS:
            out[f"{tag}_out_m_{f}"], out[f"{tag}_out_v_{f}"] = me.opt.m[f].copy(), me.opt.v[f].copy()
        out[f"{tag}_cfg"] = np.array([cfg.densify_grad_threshold, cfg.percent_dense, 3.0,
                                      cfg.prune_opacity, cfg.clone_nudge, cfg.max_primitives])
        if tag == "dp":
            Trainer.reset_opacity(me)
            out["ro_raw_opacity"] = me.prims.raw_opacity.copy()
    path = os.path.join(HERE, "optim.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {t: len(out[f"{t}_out_centers"]) for t in ("dp", "dr", "dn")})


if __name__ == "__main__":
    main()
