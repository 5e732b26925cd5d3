"""Optimizer step and densification (reference
optim.py and train.py:239-335).

CPU tests pin the float64 oracle (oracle/optim_oracle.py) to fixtures the
reference produced (tests/golden/optim.npz).  GPU tests run the device path
(csrc/optim.cu through paper_2411_16392_b200.optim / .densify) on the same
fp32 inputs.  Structure (which primitives survive, clone, split, in which
order; skip counts) is exact; values are fp32 storage of fp64 arithmetic:
parameters within one fp32 ulp per step taken (rel 1.25e-7 each) plus 1e-9
absolute, Adam moments
rel 1e-6 of the group's scale.
"""

import os

import numpy as np
import pytest

from oracle import optim_oracle as oo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "optim.npz")
G = oo.GROUPS
LRS = {"centers": 1.6e-4, "quats": 1e-3, "raw_scales": 5e-3, "raw_signs": 5e-3,
       "raw_opacity": 0.05, "sh": 2.5e-3}


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def grp(gd, tag):
    return {k: gd[f"{tag}_{k}"].astype(np.float64) for k in G}


def close(a, b, rel=2.5e-7, abs_=1e-9):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    err = np.abs(a - b) - (rel * np.abs(b) + abs_)
    assert err.max() <= 0, f"worst excess {err.max():.3e}"


def close_scaled(a, b, rel=1e-6):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    assert np.abs(a - b).max() <= rel * max(np.abs(b).max(), 1e-30)


def freeze300():
    f = {"raw_scales": np.zeros((300, 3), bool), "raw_signs": np.zeros((300, 3), bool)}
    f["raw_scales"][:, 2] = True
    f["raw_signs"][:, 2] = True
    return f


def dcfg(gd, tag):
    c = gd[f"{tag}_cfg"]
    return dict(grad_threshold=c[0], percent_dense=c[1], extent=c[2], prune_opacity=c[3],
                clone_nudge=c[4], max_primitives=int(c[5]))


# ------------------------------------------------------------ oracle (CPU)

def test_oracle_adam_matches_reference(gold):
    p = grp(gold, "adam_in")
    m = {k: np.zeros_like(p[k]) for k in G}
    v = {k: np.zeros_like(p[k]) for k in G}
    skipped = 0
    for s in range(3):
        g = grp(gold, f"adam_g{s}")
        skipped += oo.adam_step(p, g, m, v, s + 1, LRS, freeze300() if s > 0 else None)
        for k in G:
            np.testing.assert_allclose(p[k], gold[f"adam_s{s}_{k}"], rtol=1e-14, atol=1e-15)
    assert skipped == int(gold["adam_skipped"]) == 2
    for k in G:
        np.testing.assert_allclose(m[k], gold[f"adam_m_{k}"], rtol=1e-13, atol=1e-18)
        np.testing.assert_allclose(v[k], gold[f"adam_v_{k}"], rtol=1e-13, atol=1e-20)


@pytest.mark.parametrize("tag", ["dp", "dr", "dn"])
def test_oracle_densify_matches_reference(gold, tag):
    c = dcfg(gold, tag)
    stats = {"grad_accum": gold[f"{tag}_grad_accum"], "grad_count": gold[f"{tag}_grad_count"],
             "center_accum": gold[f"{tag}_center_accum"]}
    p, m, v = oo.densify_and_prune(grp(gold, f"{tag}_in"), grp(gold, f"{tag}_in_m"),
                                   grp(gold, f"{tag}_in_v"), stats, c["grad_threshold"],
                                   c["percent_dense"], c["extent"], c["prune_opacity"],
                                   c["clone_nudge"], c["max_primitives"])
    for k in G:
        np.testing.assert_array_equal(p[k], gold[f"{tag}_out_{k}"])
        np.testing.assert_array_equal(m[k], gold[f"{tag}_out_m_{k}"])
        np.testing.assert_array_equal(v[k], gold[f"{tag}_out_v_{k}"])
    if tag == "dp":
        np.testing.assert_array_equal(oo.reset_opacity(p["raw_opacity"]), gold["ro_raw_opacity"])


# ---------------------------------------------------------------- device

def _dev_prims(d):
    import torch
    from paper_2411_16392_b200.rasterizer import DevicePrimitives
    return DevicePrimitives(**{k: torch.from_numpy(np.ascontiguousarray(d[k], dtype=np.float32))
                               .cuda() for k in G})


def _grads(d):
    import torch
    from paper_2411_16392_b200.rasterizer import GradientBuffer
    t = {k: torch.from_numpy(np.ascontiguousarray(d[k], dtype=np.float32)).cuda() for k in G}
    n = t["centers"].shape[0]
    return GradientBuffer(**t, screen_center=torch.zeros((n, 2), dtype=torch.float32,
                                                         device=t["centers"].device))


@pytest.mark.gpu
def test_adam_matches_reference(gold, cuda_device):
    from paper_2411_16392_b200 import optim
    p = _dev_prims(grp(gold, "adam_in"))
    opt = optim.Adam(p)
    for s in range(3):
        opt.step(p, _grads(grp(gold, f"adam_g{s}")), LRS, freeze=freeze300() if s > 0 else None)
        for k in G:
            # the reference keeps fp64 parameters; the device rounds to fp32
            # after every step: up to one more ulp per step
            close(getattr(p, k).cpu().numpy(), gold[f"adam_s{s}_{k}"].astype(np.float32),
                  rel=1.25e-7 * (s + 2))
    assert opt.skipped == int(gold["adam_skipped"])
    for k in G:
        close_scaled(opt.m[k].cpu().numpy(), gold[f"adam_m_{k}"])
        close_scaled(opt.v[k].cpu().numpy(), gold[f"adam_v_{k}"])


@pytest.mark.gpu
def test_adam_statistics_match_oracle(gold, cuda_device):
    import torch
    from paper_2411_16392_b200 import densify, optim
    rng = np.random.default_rng(3)
    d = grp(gold, "adam_in")
    p = _dev_prims(d)
    opt = optim.Adam(p)
    st = densify.DensifyStats(300)
    ref = {"grad_accum": np.zeros(300), "grad_count": np.zeros(300),
           "center_accum": np.zeros((300, 3))}
    for s in range(3):
        gb = _grads(grp(gold, f"adam_g{s}"))
        scr = rng.normal(0, 1, (300, 2)).astype(np.float32)
        scr[::7] = 0.0                                       # unseen this step
        gb.screen_center.copy_(torch.from_numpy(scr))
        opt.step(p, gb, LRS, stats=st)
        oo.accumulate_stats(ref, scr, gold[f"adam_g{s}_centers"].astype(np.float32))
    np.testing.assert_array_equal(st.grad_count.cpu().numpy(), ref["grad_count"])
    np.testing.assert_allclose(st.grad_accum.cpu().numpy(), ref["grad_accum"], rtol=1e-15)
    c = st.center_accum.cpu().numpy()
    fin = np.isfinite(ref["center_accum"])
    np.testing.assert_array_equal(fin, np.isfinite(c))
    np.testing.assert_allclose(c[fin], ref["center_accum"][fin], rtol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["dp", "dr", "dn"])
def test_densify_matches_reference(gold, tag, cuda_device):
    import torch
    from paper_2411_16392_b200 import densify, optim
    d = grp(gold, f"{tag}_in")
    p = _dev_prims(d)
    opt = optim.Adam(p)
    for k in G:
        opt.m[k] = torch.from_numpy(gold[f"{tag}_in_m_{k}"].astype(np.float32)).cuda()
        opt.v[k] = torch.from_numpy(gold[f"{tag}_in_v_{k}"].astype(np.float32)).cuda()
    n = len(d["centers"])
    st = densify.DensifyStats(n)
    st.grad_accum.copy_(torch.from_numpy(gold[f"{tag}_grad_accum"]))
    st.grad_count.copy_(torch.from_numpy(gold[f"{tag}_grad_count"]))
    st.center_accum.copy_(torch.from_numpy(gold[f"{tag}_center_accum"]))
    c = dcfg(gold, tag)
    cfg = densify.DensifyConfig(c["grad_threshold"], c["percent_dense"], c["prune_opacity"],
                                c["clone_nudge"], c["max_primitives"])
    p2 = densify.densify_and_prune(p, opt, st, cfg, c["extent"])
    n_out = len(gold[f"{tag}_out_centers"])
    assert len(p2) == n_out and st.grad_accum.shape[0] == n_out
    for k in G:
        close(getattr(p2, k).cpu().numpy(), gold[f"{tag}_out_{k}"].astype(np.float32))
        close(opt.m[k].cpu().numpy(), gold[f"{tag}_out_m_{k}"].astype(np.float32), abs_=0)
        close(opt.v[k].cpu().numpy(), gold[f"{tag}_out_v_{k}"].astype(np.float32), abs_=0)
    if tag == "dp":
        densify.reset_opacity(p2, opt)
        close(p2.raw_opacity.cpu().numpy(), gold["ro_raw_opacity"].astype(np.float32))
        assert not bool(opt.m["raw_opacity"].any()) and not bool(opt.v["raw_opacity"].any())


@pytest.mark.gpu
def test_densify_large_budget_selection(cuda_device):
    """top-`room` selection with many ties at C3-like size, against the oracle"""
    import torch
    from paper_2411_16392_b200 import densify, optim
    rng = np.random.default_rng(5)
    n, k = 200_000, 16
    q = rng.normal(size=(n, 4))
    d = {"centers": rng.normal(0, 1, (n, 3)), "quats": q / np.linalg.norm(q, axis=1, keepdims=True),
         "raw_scales": rng.normal(-4, 1, (n, 3)), "raw_signs": rng.normal(0, 1.5, (n, 3)),
         "raw_opacity": rng.normal(0, 2.5, n), "sh": rng.normal(0, 0.5, (n, 3, k))}
    d = {key: val.astype(np.float32).astype(np.float64) for key, val in d.items()}
    cnt = rng.integers(0, 3, n).astype(np.float64)
    acc = np.round(rng.uniform(0, 1, n) * 16) / 16 * cnt    # heavy ties
    cacc = rng.normal(0, 1e-3, (n, 3)).astype(np.float32).astype(np.float64)
    p = _dev_prims(d)
    opt = optim.Adam(p)
    st = densify.DensifyStats(n)
    st.grad_accum.copy_(torch.from_numpy(acc))
    st.grad_count.copy_(torch.from_numpy(cnt))
    st.center_accum.copy_(torch.from_numpy(cacc))
    cfg = densify.DensifyConfig(0.3, 0.005, 0.005, 0.5, n + 4321)
    p2 = densify.densify_and_prune(p, opt, st, cfg, 3.0)
    zero = {key: np.zeros_like(val) for key, val in d.items()}
    po, _, _ = oo.densify_and_prune(d, zero, zero, {"grad_accum": acc, "grad_count": cnt,
                                                    "center_accum": cacc},
                                    0.3, 0.005, 3.0, 0.005, 0.5, n + 4321)
    assert len(p2) == len(po["centers"])
    for key in G:
        close(getattr(p2, key).cpu().numpy(), po[key].astype(np.float32))
