"""Loss producers (reference losses.py / ssim.py).

CPU tests pin the float64 oracle (oracle/losses_oracle.py) to fixtures the
reference itself produced (tests/golden/losses.npz) and restate the
reference's own loss tests (tests/test_losses.py of qgsplat) against it.
GPU tests check the device kernels (csrc/losses.cu, through the C ABI via
paper_2411_16392_b200.losses / .ssim) against the fixtures and the oracle.

Tolerances: values are fp64 on the device (summation order differs from
numpy: rel 1e-10); gradient / normal maps are stored fp32 (rel 2e-6 of the
map's largest magnitude); masks are exact.
"""

import os

import numpy as np
import pytest

from oracle import losses_oracle as lo

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "losses.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def close_map(a, b, rel=2e-6):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape
    scale = max(np.abs(b).max(), 1e-30)
    err = np.abs(a - b).max() / scale
    assert err <= rel, f"max rel err {err:.3e}"


def f64(a):
    return np.asarray(a, dtype=np.float64)


def intr(g):
    return tuple(float(v) for v in g["nc_intr"])


class Cam:
    def __init__(self, fx, fy, cx, cy, W, H, w2c=None):
        self.fx, self.fy, self.cx, self.cy = fx, fy, cx, cy
        self.width, self.height = W, H
        self.world_to_camera = np.eye(4) if w2c is None else w2c

    def pixel_dirs_cam(self):
        return lo.pixel_dirs_cam(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


def gold_cam(g):
    W, H = (int(v) for v in g["nc_size"])
    return Cam(*intr(g), W, H, g["nc_w2c"])


def make_cam(res=24):
    """qgsplat tests/test_losses.py make_cam: fx = fy = 30, centred, 4 m away"""
    return Cam(30.0, 30.0, res / 2, res / 2, res, res)


def plane_depth(cam, n_cam, d0):
    dirs = cam.pixel_dirs_cam()
    return d0 / (dirs @ n_cam)


# ------------------------------------------------------------ oracle (CPU)

def test_oracle_photometric_matches_reference(gold):
    x, y = f64(gold["ph_x"]), f64(gold["ph_y"])
    for tag, m in (("m02", 0.2), ("m0", 0.0), ("m1", 1.0)):
        v, g = lo.photometric(x, y, m)
        assert v == pytest.approx(float(gold[f"ph_{tag}_value"]), rel=1e-13, abs=1e-15)
        close_map(g, gold[f"ph_{tag}_grad"], rel=1e-12)


def test_oracle_ssim_matches_reference(gold):
    s, g = lo.ssim(f64(gold["ss_x"]), f64(gold["ss_y"]), return_grad=True)
    assert s == pytest.approx(float(gold["ss_value"]), rel=1e-13)
    close_map(g, gold["ss_grad"], rel=1e-12)


def test_oracle_distortion_matches_reference(gold):
    v, g = lo.depth_distortion(f64(gold["di_map"]))
    assert v == pytest.approx(float(gold["di_value"]), rel=1e-13)
    close_map(g, gold["di_grad"], rel=1e-15)


def test_oracle_depth_normal_consistency_matches_reference(gold):
    N, mask = lo.depth_to_normal(gold["nc_depth"], gold["nc_alpha"], intr(gold))
    assert np.array_equal(mask, gold["nc_mask"])
    close_map(N, gold["nc_N"], rel=1e-12)
    for tag, guided in (("g", True), ("u", False)):
        v, da, dn, dk = lo.normal_consistency(gold["nc_alpha"], gold["nc_normal"], gold["nc_curv"],
                                              N, mask, 1e-6, guided)
        assert v == pytest.approx(float(gold[f"nc_{tag}_value"]), rel=1e-12)
        close_map(da, gold[f"nc_{tag}_da"], rel=1e-12)
        close_map(dn, gold[f"nc_{tag}_dn"], rel=1e-12)
        if guided:
            close_map(dk, gold[f"nc_{tag}_dk"], rel=1e-12)
        else:
            assert not np.any(dk) and not np.any(gold[f"nc_{tag}_dk"])


def test_oracle_reference_unit_cases():
    """the reference's own unit tests, restated against the oracle"""
    img = np.random.default_rng(0).uniform(0, 1, (32, 32, 3))
    assert lo.photometric(img, img, 0.2)[0] == pytest.approx(0.0, abs=1e-12)
    gt = np.random.default_rng(1).uniform(0.2, 0.8, (16, 16, 3))
    assert lo.photometric(gt + 0.1, gt, 0.0)[0] == pytest.approx(0.1, rel=1e-12)
    with pytest.raises(ValueError):
        lo.photometric(np.zeros((4, 4, 3)), np.zeros((5, 4, 3)))
    cam = make_cam()
    depth = plane_depth(cam, np.array([0.0, 0.0, 1.0]), 4.0)
    N, mask = lo.depth_to_normal(depth, np.ones_like(depth), (cam.fx, cam.fy, cam.cx, cam.cy))
    assert mask[1:-1, 1:-1].all() and not mask[0].any() and not mask[:, 0].any()
    assert np.linalg.norm(N[mask] - np.array([0, 0, -1.0]), axis=1).max() < 1e-9


# ---------------------------------------------------------------- device

@pytest.mark.gpu
def test_photometric_matches_reference(gold, cuda_device):
    from paper_2411_16392_b200 import losses as L
    for tag, m in (("m02", 0.2), ("m0", 0.0), ("m1", 1.0)):
        v, g = L.photometric(gold["ph_x"], gold["ph_y"], m)
        assert v == pytest.approx(float(gold[f"ph_{tag}_value"]), rel=1e-10, abs=1e-14)
        close_map(g.cpu().numpy(), gold[f"ph_{tag}_grad"])
    # tie pixel: sign(0) = 0 leaves only the SSIM term
    v, g = L.photometric(gold["ph_x"], gold["ph_y"], 0.0)
    assert float(g[3, 4].abs().max()) == 0.0


@pytest.mark.gpu
def test_ssim_matches_reference(gold, cuda_device):
    from paper_2411_16392_b200 import ssim as S
    s, g = S.ssim(gold["ss_x"], gold["ss_y"], return_grad=True)
    assert s == pytest.approx(float(gold["ss_value"]), rel=1e-10)
    close_map(g.cpu().numpy(), gold["ss_grad"])
    assert S.ssim(gold["ss_x"], gold["ss_y"]) == pytest.approx(s, rel=1e-15)


@pytest.mark.gpu
def test_distortion_matches_reference(gold, cuda_device):
    from paper_2411_16392_b200 import losses as L
    v, g = L.depth_distortion(gold["di_map"])
    assert v == pytest.approx(float(gold["di_value"]), rel=1e-10)
    close_map(g.cpu().numpy(), gold["di_grad"], rel=1e-7)


@pytest.mark.gpu
def test_depth_normal_consistency_matches_reference(gold, cuda_device):
    from paper_2411_16392_b200 import losses as L
    cam = gold_cam(gold)
    N, mask = L.depth_to_normal(gold["nc_depth"], gold["nc_alpha"], cam)
    assert np.array_equal(mask.cpu().numpy(), gold["nc_mask"])
    close_map(N.cpu().numpy(), gold["nc_N"], rel=1e-7)
    for tag, guided in (("g", True), ("u", False)):
        # N as the reference computed it (fp64 rounded to fp32 on the way in)
        v, da, dn, dk = L.curvature_guided_normal_consistency(
            gold["nc_alpha"], gold["nc_normal"], gold["nc_curv"], gold["nc_N"], gold["nc_mask"],
            1e-6, guided)
        assert v == pytest.approx(float(gold[f"nc_{tag}_value"]), rel=1e-6)
        close_map(da.cpu().numpy(), gold[f"nc_{tag}_da"])
        close_map(dn.cpu().numpy(), gold[f"nc_{tag}_dn"], rel=1e-6)
        if guided:
            close_map(dk.cpu().numpy(), gold[f"nc_{tag}_dk"], rel=1e-6)
        else:
            assert not bool(dk.any())


@pytest.mark.gpu
def test_fused_upstream_matches_reference(gold, cuda_device):
    """accumulate_upstream (depth -> normal fused into the consistency loss)
    against the reference's separate calls, at the train-step weights"""
    import torch
    from paper_2411_16392_b200 import losses as L
    cam = gold_cam(gold)
    H, W = gold["nc_depth"].shape
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(7)
    color = np.clip(rng.uniform(0, 1, (H, W, 3)), 0, 1).astype(np.float32)
    gt = np.clip(color + rng.normal(0, 0.05, color.shape), 0, 1).astype(np.float32)
    dist = rng.exponential(0.01, (H, W)).astype(np.float32)

    class T:
        pass
    t = T()
    t.color = torch.from_numpy(color).to(dev)
    t.distortion = torch.from_numpy(dist).to(dev)
    t.alpha = torch.from_numpy(gold["nc_alpha"]).to(dev)
    t.normal = torch.from_numpy(gold["nc_normal"]).to(dev)
    t.curvature = torch.from_numpy(gold["nc_curv"]).to(dev)
    t.depth_median = torch.from_numpy(gold["nc_depth"]).to(dev)
    up = {k: torch.full(s, 0.25, dtype=torch.float32, device=dev) for k, s in
          (("color", (H, W, 3)), ("alpha", (H, W)), ("depth", (H, W)), ("normal", (H, W, 3)),
           ("curvature", (H, W)), ("distortion", (H, W)))}
    w = L.LossWeights()
    parts = L.accumulate_upstream(t, gt, cam, up, w).cpu().numpy()
    l_c, g_c = lo.photometric(color, gt, w.lambda_photo_ssim)
    l_d, g_d = lo.depth_distortion(dist)
    v, da, dn, dk = lo.normal_consistency(gold["nc_alpha"], gold["nc_normal"], gold["nc_curv"],
                                          gold["nc_N"], gold["nc_mask"], w.eps_curvature, True)
    assert parts[0] == pytest.approx(l_c, rel=1e-10)
    assert parts[1] == pytest.approx(l_d, rel=1e-10)
    assert parts[2] == pytest.approx(v, rel=1e-10)
    def close_acc(got, want):
        # fp32 accumulation onto 0.25: one rounding at 0.25's ulp
        got = got.cpu().numpy().astype(np.float64)
        tol = 0.25 * 2.0 ** -23 + 2e-6 * np.abs(want).max()
        assert np.abs(got - (0.25 + want)).max() <= tol
    close_acc(up["color"], g_c)
    close_acc(up["distortion"], w.lambda_d * g_d)
    close_acc(up["alpha"], w.lambda_n * da)
    close_acc(up["normal"], w.lambda_n * dn)
    close_acc(up["curvature"], w.lambda_n * dk)
    assert float(up["depth"].sub(0.25).abs().max()) == 0.0


@pytest.mark.gpu
def test_reference_unit_cases_on_device(cuda_device):
    """qgsplat tests/test_losses.py, through the device drop-in"""
    import torch
    from paper_2411_16392_b200 import losses as L
    from paper_2411_16392_b200 import ssim as S
    img = np.random.default_rng(0).uniform(0, 1, (32, 32, 3)).astype(np.float32)
    v, g = L.photometric(img, img, 0.2)
    assert v == pytest.approx(0.0, abs=1e-12)
    gt = np.random.default_rng(1).uniform(0.2, 0.8, (16, 16, 3)).astype(np.float32)
    v, _ = L.photometric(gt + np.float32(0.1), gt, 0.0)
    assert v == pytest.approx(0.1, rel=1e-6)       # fp32 inputs: 0.1 is not exact
    with pytest.raises(ValueError):
        L.photometric(np.zeros((4, 4, 3)), np.zeros((5, 4, 3)))
    with pytest.raises(ValueError):
        S.ssim(np.zeros((10, 12)), np.zeros((10, 12)))
    d = np.zeros((8, 8), dtype=np.float32)
    v, g = L.depth_distortion(d)
    assert v == 0.0
    d[2, 3] = 0.25
    v, g = L.depth_distortion(d)
    assert v == pytest.approx(0.25 / 64) and float(g[0, 0]) == pytest.approx(1 / 64)

    cam = make_cam()
    depth = plane_depth(cam, np.array([0.0, 0.0, 1.0]), 4.0)
    N, mask = L.depth_to_normal(depth, np.ones_like(depth), cam)
    N, mask = N.cpu().numpy(), mask.cpu().numpy()
    assert mask[1:-1, 1:-1].all() and not mask[0].any() and not mask[:, 0].any()
    # the reference's bound is 1e-9 on float64 depth; the device reads fp32 maps
    assert np.linalg.norm(N[mask] - np.array([0, 0, -1.0]), axis=1).max() < 1e-5
    n_plane = np.array([0.3, -0.2, 0.93])
    n_plane /= np.linalg.norm(n_plane)
    depth = plane_depth(cam, n_plane, 3.0)
    N, mask = L.depth_to_normal(depth, np.ones_like(depth), cam)
    N, mask = N.cpu().numpy(), mask.cpu().numpy()
    assert np.linalg.norm(N[mask] - (-n_plane), axis=1).max() < 1e-3   # fp32 depth input
    depth = plane_depth(cam, np.array([0.0, 0, 1.0]), 4.0)
    alpha = np.ones_like(depth)
    alpha[10, 10] = 0.0
    _, mask = L.depth_to_normal(depth, alpha, cam)
    mask = mask.cpu().numpy()
    assert not mask[10, 10] and not mask[10, 11] and not mask[10, 9]
    assert not mask[11, 10] and not mask[9, 10]

    H = W = 8
    N = np.zeros((H, W, 3))
    N[:, :, 2] = -1.0
    m = np.ones((H, W), dtype=bool)
    alpha = np.full((H, W), 0.8)
    curv = np.random.default_rng(5).normal(size=(H, W))
    v, da, dn, dk = L.curvature_guided_normal_consistency(alpha, alpha[:, :, None] * N, curv, N, m)
    assert v == pytest.approx(0.0, abs=1e-7) and float(dk.abs().max()) < 1e-7
    H = W = 6
    N = np.zeros((H, W, 3))
    N[:, :, 2] = -1.0
    m = np.ones((H, W), dtype=bool)
    alpha = np.full((H, W), 0.9)
    v_flat, *_ = L.curvature_guided_normal_consistency(alpha, np.zeros((H, W, 3)),
                                                       np.zeros((H, W)), N, m)
    v_curved, *_ = L.curvature_guided_normal_consistency(alpha, np.zeros((H, W, 3)),
                                                         np.full((H, W), 1e9), N, m)
    assert v_curved < 1e-8 < v_flat
    assert L.lambda_curvature(0.0, 1e-6) == pytest.approx(0.999999, abs=1e-6)
    assert float(L.lambda_curvature(torch.tensor([1e9]), 1e-6)) < 1e-8


def test_loss_weights_and_total():
    from paper_2411_16392_b200 import losses as L
    w = L.LossWeights(lambda_d=2.0, lambda_n=0.5, lambda_mv=0.0)
    assert L.total_loss(1.0, 0.25, 0.5, 99.0, w) == pytest.approx(1.0 + 0.5 + 0.25)
    w0 = L.LossWeights(lambda_d=0, lambda_n=0, lambda_mv=0)
    assert L.total_loss(0.7, 1, 1, 1, w0) == pytest.approx(0.7)
    with pytest.raises(ValueError):
        L.LossWeights(lambda_d=-1)
    with pytest.raises(ValueError):
        L.LossWeights(lambda_photo_ssim=1.5)


@pytest.mark.gpu
def test_full_size_losses_against_oracle(cuda_device):
    """C3 image size (1600x1200): every device output against the oracle"""
    import torch
    from paper_2411_16392_b200 import losses as L
    rng = np.random.default_rng(11)
    H, W = 1200, 1600
    x = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    y = np.clip(x + rng.normal(0, 0.05, x.shape), 0, 1).astype(np.float32)
    v, g = L.photometric(x, y, 0.2)
    vo, go = lo.photometric(x, y, 0.2)
    assert v == pytest.approx(vo, rel=1e-10)
    close_map(g.cpu().numpy(), go)
    cam = Cam(1400.0, 1400.0, W / 2, H / 2, W, H)
    yy, xx = np.mgrid[0:H, 0:W]
    depth = (3.0 + 0.3 * np.sin(xx / 90.0) * np.cos(yy / 70.0)).astype(np.float32)
    alpha = rng.uniform(0.3, 1.0, (H, W)).astype(np.float32)
    depth[rng.random((H, W)) < 0.01] = 0.0
    N, mask = L.depth_to_normal(depth, alpha, cam)
    No, mo = lo.depth_to_normal(depth, alpha, (cam.fx, cam.fy, cam.cx, cam.cy))
    assert np.array_equal(mask.cpu().numpy(), mo)
    close_map(N.cpu().numpy(), No, rel=1e-6)
    normal = rng.normal(0, 0.5, (H, W, 3)).astype(np.float32)
    curv = rng.normal(0, 2, (H, W)).astype(np.float32)
    v, da, dn, dk = L.curvature_guided_normal_consistency(alpha, normal, curv, No, mo)
    vo, dao, dno, dko = lo.normal_consistency(alpha, normal, curv,
                                              No.astype(np.float32).astype(np.float64), mo)
    assert v == pytest.approx(vo, rel=1e-9)
    close_map(da.cpu().numpy(), dao)
    close_map(dn.cpu().numpy(), dno)
    close_map(dk.cpu().numpy(), dko)
    torch.cuda.synchronize()


def test_host_validation_without_device():
    """shape / window errors are raised on the host, before any transfer"""
    from paper_2411_16392_b200 import losses as L
    from paper_2411_16392_b200 import ssim as S
    with pytest.raises(ValueError):
        L.photometric(np.zeros((4, 4, 3)), np.zeros((5, 4, 3)))
    with pytest.raises(ValueError, match="SSIM window"):
        L.photometric(np.zeros((8, 40, 3)), np.zeros((8, 40, 3)), 0.2)
    with pytest.raises(ValueError):
        S.ssim(np.zeros((12, 12)), np.zeros((12, 13)))
    with pytest.raises(ValueError):
        S.ssim(np.zeros((10, 12)), np.zeros((10, 12)))
    with pytest.raises(ValueError):
        S.ssim(np.zeros((12,)), np.zeros((12,)))

