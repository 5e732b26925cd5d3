"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU float64 numpy restatement of the reference's loss producers
(/root/reference/pkg/src/qgsplat/losses.py and ssim.py), the checker for
csrc/losses.cu.  The 1-D Gaussian correlation with zero padding
(scipy.ndimage.correlate1d(mode="constant"), ssim.py:29-31) is restated as
eleven shifted, weighted adds over a zero-padded copy -- no scipy.  Pinned
against fixtures produced by the reference itself
(tests/golden/losses.npz, tests/golden/make_losses_golden.py).

Only ``tests/`` may import this module; the product package never does.
"""

import numpy as np

WINDOW = 11        # ssim.py:12
SIGMA = 1.5        # ssim.py:13
C1 = 0.01 ** 2     # ssim.py:14
C2 = 0.03 ** 2     # ssim.py:15


def gauss_taps():
    """ssim.py:19-23"""
    r = WINDOW // 2
    x = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-(x * x) / (2 * SIGMA * SIGMA))
    return k / k.sum()


_K = gauss_taps()


def _corr1d(img, axis):
    r = WINDOW // 2
    pad = [(0, 0)] * img.ndim
    pad[axis] = (r, r)
    p = np.pad(img, pad)
    n = img.shape[axis]
    out = np.zeros_like(img)
    for k in range(WINDOW):
        out += _K[k] * np.take(p, np.arange(k, k + n), axis=axis)
    return out


def blur(img):
    """ssim.py:29-31: axis 0 then axis 1"""
    return _corr1d(_corr1d(img, 0), 1)


def ssim(x, y, return_grad=False):
    """ssim.py:41-86"""
    xc = np.asarray(x, dtype=np.float64)
    yc = np.asarray(y, dtype=np.float64)
    two_d = xc.ndim == 2
    if two_d:
        xc, yc = xc[:, :, None], yc[:, :, None]
    if xc.shape != yc.shape:
        raise ValueError("image shapes differ")
    r = WINDOW // 2
    H, W, C = xc.shape
    if H < WINDOW or W < WINDOW:
        raise ValueError("image smaller than the SSIM window")
    crop = (slice(r, H - r), slice(r, W - r))
    n_valid = (H - 2 * r) * (W - 2 * r) * C
    total = 0.0
    grad = np.zeros_like(xc)
    for c in range(C):
        xi, yi = xc[:, :, c], yc[:, :, c]
        ux, uy = blur(xi), blur(yi)
        uxx, uyy, uxy = blur(xi * xi), blur(yi * yi), blur(xi * yi)
        vx, vy, vxy = uxx - ux * ux, uyy - uy * uy, uxy - ux * uy
        A1, A2 = 2 * ux * uy + C1, 2 * vxy + C2
        B1, B2 = ux * ux + uy * uy + C1, vx + vy + C2
        S = (A1 * A2) / (B1 * B2)
        total += S[crop].sum()
        if return_grad:
            M = np.zeros((H, W))
            M[crop] = 1.0 / n_valid
            d_ux = (2 * uy * B1 - A1 * 2 * ux) / (B1 * B1) * (A2 / B2) \
                + (A1 / B1) * (-2 * uy * B2 - A2 * (-2 * ux)) / (B2 * B2)
            d_uxx = (A1 / B1) * (-A2 / (B2 * B2))
            d_uxy = (A1 / B1) * (2 / B2)
            grad[:, :, c] = blur(M * d_ux) + 2 * xi * blur(M * d_uxx) + yi * blur(M * d_uxy)
    value = total / n_valid
    if return_grad:
        return value, (grad[:, :, 0] if two_d else grad)
    return value


def photometric(render, gt, lambda_photo_ssim=0.2):
    """losses.py:36-50"""
    render = np.asarray(render, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if render.shape != gt.shape:
        raise ValueError("image shapes differ")
    diff = render - gt
    l1 = np.abs(diff).mean()
    g = np.sign(diff) / diff.size * (1.0 - lambda_photo_ssim)
    if lambda_photo_ssim > 0:
        s, gs = ssim(render, gt, return_grad=True)
        return (1 - lambda_photo_ssim) * l1 + lambda_photo_ssim * (1.0 - s), g - lambda_photo_ssim * gs
    return l1, g


def depth_distortion(d):
    """losses.py:53-56"""
    d = np.asarray(d, dtype=np.float64)
    return d.mean(), np.full_like(d, 1.0 / d.size)


def pixel_dirs_cam(fx, fy, cx, cy, W, H):
    """cameras.py:53-59"""
    u = (np.arange(W) + 0.5 - cx) / fx
    v = (np.arange(H) + 0.5 - cy) / fy
    uu, vv = np.meshgrid(u, v)
    d = np.stack([uu, vv, np.ones_like(uu)], axis=-1)
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def depth_to_normal(depth, alpha, intr, alpha_thresh=0.5):
    """losses.py:59-89; intr = (fx, fy, cx, cy)"""
    depth = np.asarray(depth, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    H, W = depth.shape
    dirs = pixel_dirs_cam(*intr, W, H)
    P = depth[:, :, None] * dirs
    ok = (alpha > alpha_thresh) & (depth > 0)
    N = np.zeros((H, W, 3))
    mask = np.zeros((H, W), dtype=bool)
    du = P[1:-1, 2:] - P[1:-1, :-2]
    dv = P[2:, 1:-1] - P[:-2, 1:-1]
    n = np.cross(du, dv)
    nn = np.linalg.norm(n, axis=-1)
    valid = (ok[1:-1, 1:-1] & ok[1:-1, 2:] & ok[1:-1, :-2] & ok[2:, 1:-1] & ok[:-2, 1:-1]
             & (nn > 1e-12))
    n = np.where(valid[:, :, None], n / np.maximum(nn, 1e-12)[:, :, None], 0.0)
    flip = np.sum(n * dirs[1:-1, 1:-1], axis=-1) > 0
    n = np.where(flip[:, :, None], -n, n)
    N[1:-1, 1:-1] = n
    mask[1:-1, 1:-1] = valid
    return N, mask


def normal_consistency(alpha, normal_map, curv_map, N, mask, eps_curvature=1e-6, guided=True):
    """losses.py:97-113"""
    alpha = np.asarray(alpha, dtype=np.float64)
    normal_map = np.asarray(normal_map, dtype=np.float64)
    curv_map = np.asarray(curv_map, dtype=np.float64)
    m = np.asarray(mask).astype(np.float64)
    count = max(m.sum(), 1.0)
    ln = alpha - np.sum(normal_map * N, axis=-1)
    if guided:
        lam = 1.0 / (1.0 + np.abs(curv_map) + eps_curvature)
        dlam = -np.sign(curv_map) * lam * lam
    else:
        lam = np.ones_like(curv_map)
        dlam = np.zeros_like(curv_map)
    value = np.sum(m * lam * ln) / count
    return (value, m * lam / count, -(m * lam / count)[:, :, None] * N, m * dlam * ln / count)
