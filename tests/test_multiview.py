"""Multi-view reprojection + NCC loss (reference
multiview.py:108-311).

CPU: the per-pixel float64 oracle (oracle/multiview_oracle.py) against the
fixtures the reference produced (tests/golden/multiview.npz).  GPU: the
device kernel (csrc/multiview.cu via paper_2411_16392_b200.multiview)
against the same fixtures and the oracle, plus the reference's own unit
cases.  Tolerances: the value and stats are fp64 on the device (rel 1e-9);
the upstream maps are fp32 (rel 1e-5 of the map's largest magnitude: fp64
sums in a different order, one fp32 rounding); n_valid exact.
"""

import os

import numpy as np
import pytest

from oracle import multiview_oracle as mo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "multiview.npz")
TAGS = ("p", "q", "x")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


class Cam:
    def __init__(self, intr, w2c, W, H):
        self.fx, self.fy, self.cx, self.cy = (float(v) for v in intr)
        self.width, self.height = W, H
        self.world_to_camera = np.asarray(w2c, dtype=np.float64)

    def as_dict(self):
        return {"fx": self.fx, "fy": self.fy, "cx": self.cx, "cy": self.cy,
                "R": self.world_to_camera[:3, :3], "t": self.world_to_camera[:3, 3]}


def case(g, tag):
    out = []
    for side in ("r", "n"):
        m = {k: g[f"{tag}_{side}_{k}"] for k in ("depth", "alpha", "normal", "image")}
        H, W = m["alpha"].shape
        out += [m, Cam(g[f"{tag}_{side}_cam"], g[f"{tag}_{side}_w2c"], W, H)]
    return out


def close_map(a, b, rel=1e-5, floor=1e-9):
    """max |a - b| within rel of b's largest magnitude (at least `floor`:
    some maps are pure cancellation noise, ~1e-18)"""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    err = np.abs(a - b).max() / max(np.abs(b).max(), floor)
    assert err <= rel, f"max rel err {err:.3e}"


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_matches_reference(gold, tag):
    mr, cr, mn, cn = case(gold, tag)
    v, nv, ur, un, st = mo.multiview_loss(mr, cr.as_dict(), mn, cn.as_dict(),
                                          full_chain=bool(gold[f"{tag}_full"]))
    assert nv == int(gold[f"{tag}_n_valid"])
    assert v == pytest.approx(float(gold[f"{tag}_value"]), rel=1e-11)
    assert st["warp_px"] == pytest.approx(float(gold[f"{tag}_warp_px"]), rel=1e-10)
    assert st["ncc"] == pytest.approx(float(gold[f"{tag}_ncc"]), rel=1e-12)
    for k in ("depth", "alpha", "normal"):
        close_map(ur[k], gold[f"{tag}_up_r_{k}"], rel=1e-9, floor=1e-7)
        close_map(un[k], gold[f"{tag}_up_n_{k}"], rel=1e-9, floor=1e-7)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_device_matches_reference(gold, tag, cuda_device):
    from paper_2411_16392_b200 import multiview as M
    mr, cr, mn, cn = case(gold, tag)
    cfg = M.MultiviewConfig(full_chain=bool(gold[f"{tag}_full"]))
    v, nv, ur, un, st = M.multiview_loss(mr, cr, mn, cn, cfg)
    assert nv == int(gold[f"{tag}_n_valid"])
    assert v == pytest.approx(float(gold[f"{tag}_value"]), rel=1e-9)
    assert st["warp_px"] == pytest.approx(float(gold[f"{tag}_warp_px"]), rel=1e-9)
    assert st["ncc"] == pytest.approx(float(gold[f"{tag}_ncc"]), rel=1e-12)
    for k in ("depth", "alpha", "normal"):
        close_map(ur[k].cpu().numpy(), gold[f"{tag}_up_r_{k}"])
        close_map(un[k].cpu().numpy(), gold[f"{tag}_up_n_{k}"])


@pytest.mark.gpu
def test_fused_accumulation(gold, cuda_device):
    import torch
    from paper_2411_16392_b200 import multiview as M
    mr, cr, mn, cn = case(gold, "x")
    dev = torch.device("cuda:0")
    up_r = {"depth": torch.full(mr["alpha"].shape, 0.5, device=dev),
            "alpha": torch.zeros(mr["alpha"].shape, device=dev),
            "normal": torch.zeros(mr["normal"].shape, device=dev)}
    up_n = {"depth": torch.zeros(mn["alpha"].shape, device=dev),
            "alpha": torch.zeros(mn["alpha"].shape, device=dev),
            "normal": torch.zeros(mn["normal"].shape, device=dev)}
    vals = M.accumulate_multiview(mr, cr, mn, cn, up_r, up_n, 0.05).cpu().numpy()
    assert vals[0] == pytest.approx(float(gold["x_value"]), rel=1e-9)
    assert int(vals[1]) == int(gold["x_n_valid"])
    got = up_r["depth"].cpu().numpy().astype(np.float64) - 0.5
    want = 0.05 * gold["x_up_r_depth"]
    assert np.abs(got - want).max() <= 0.5 * 2.0 ** -23 + 1e-5 * np.abs(want).max()
    close_map(up_n["normal"].cpu().numpy(), 0.05 * gold["x_up_n_normal"])


@pytest.mark.gpu
def test_reference_unit_cases(cuda_device):
    """qgsplat tests/test_multiview.py: identical views give zero loss; a
    plane seen by two cameras reprojects onto itself; nothing valid -> the
    reference's empty result"""
    from paper_2411_16392_b200 import multiview as M
    rng = np.random.default_rng(0)
    H = W = 24
    w2c = np.eye(4)
    w2c[2, 3] = 3.0
    cam = Cam([30.0, 30.0, 12.0, 12.0], w2c, W, H)
    dirs = mo.np.stack(np.meshgrid((np.arange(W) + 0.5 - 12) / 30, (np.arange(H) + 0.5 - 12) / 30),
                       -1)
    d = np.concatenate([dirs, np.ones((H, W, 1))], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    t = 3.0 / d[..., 2]
    img = 0.5 + 0.25 * np.sin(3 * t * d[..., 0]) * np.cos(2 * t * d[..., 1])
    maps = {"depth": t, "alpha": np.ones((H, W)), "image": img,
            "normal": np.tile([0.0, 0.0, -1.0], (H, W, 1))}
    v, nv, ur, un, st = M.multiview_loss(maps, cam, maps, cam)
    assert nv > 0 and v == pytest.approx(0.0, abs=1e-6)   # fp32 maps
    assert st["warp_px"] < 1e-5
    empty = dict(maps, alpha=np.zeros((H, W)))
    v, nv, ur, un, st = M.multiview_loss(empty, cam, maps, cam)
    assert (v, nv, st["ncc"]) == (0.0, 0, 1.0)
    assert not bool(ur["depth"].any()) and not bool(un["normal"].any())
    assert rng is not None
