"""Training objectives on the device -- drop-in for ``qgsplat.losses``
(/root/reference/pkg/src/qgsplat/losses.py).

Same names, arguments and error behaviour as the reference module; maps are
torch tensors (any device / dtype is accepted and moved to the current CUDA
device as contiguous fp32), gradients come back as CUDA fp32 tensors and
loss values as Python floats.  The arithmetic runs in fp64 inside
libqgs_b200.so (csrc/losses.cu); there is no CPU path.

``accumulate_upstream`` is the fused form of the training step's loss block
(train.py:193-211): every term adds its weighted gradient straight into the
rasterizer's upstream maps and the loss values stay on the device.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rasterizer import _cam_struct, _ptr, _stream

_WS = {}


@dataclass
class LossWeights:
    """losses.py:20-34."""
    lambda_d: float = 1000.0
    lambda_n: float = 0.05
    lambda_mv: float = 0.05
    lambda_photo_ssim: float = 0.2
    eps_curvature: float = 1e-6

    def __post_init__(self):
        vals = (self.lambda_d, self.lambda_n, self.lambda_mv,
                self.lambda_photo_ssim, self.eps_curvature)
        if not all(np.isfinite(v) and v >= 0 for v in vals):
            raise ValueError("loss weights must be finite and non-negative")
        if not 0 <= self.lambda_photo_ssim <= 1:
            raise ValueError("lambda_photo_ssim must lie in [0, 1]")


def _dev(x, dtype=torch.float32):
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=dev).contiguous()


def _workspace(H, W, C):
    L = _lib.load()
    n = int(L.qgs_loss_workspace_bytes(H, W, C))
    key = torch.cuda.current_device()
    ws = _WS.get(key)
    if ws is None or ws.numel() < n:
        ws = torch.empty((n,), dtype=torch.uint8, device=torch.device("cuda", key))
        _WS[key] = ws
    return ws


def _photometric_dev(render, gt, lambda_photo_ssim, weight, d_render, values):
    if render.shape != gt.shape:
        raise ValueError(f"image shapes differ: {tuple(render.shape)} vs {tuple(gt.shape)}")
    H, W = int(render.shape[0]), int(render.shape[1])
    C = 1 if render.dim() == 2 else int(render.shape[2])
    if lambda_photo_ssim > 0 and (H < 11 or W < 11):
        raise ValueError("image smaller than the SSIM window")
    ws = _workspace(H, W, C)
    _lib.check(_lib.load().qgs_loss_photometric(
        _ptr(render), _ptr(gt), H, W, C, float(lambda_photo_ssim), float(weight), _ptr(d_render),
        _ptr(values), _ptr(ws), ws.numel(), _stream()), "qgs_loss_photometric")


def _check_images(render, gt, lambda_photo_ssim):
    """losses.py:40-41 and ssim.py:53-54, on the host before any transfer"""
    rs, gs = tuple(np.shape(render)), tuple(np.shape(gt))
    if rs != gs:
        raise ValueError(f"image shapes differ: {rs} vs {gs}")
    if lambda_photo_ssim > 0 and (rs[0] < 11 or rs[1] < 11):
        raise ValueError("image smaller than the SSIM window")


def photometric(render, gt, lambda_photo_ssim=0.2):
    """losses.py:36-50: (1-m) L1 + m (1 - SSIM); returns (value, d/d render)."""
    _check_images(render, gt, lambda_photo_ssim)
    render, gt = _dev(render), _dev(gt)
    g = torch.zeros_like(render)
    values = torch.zeros((3,), dtype=torch.float64, device=render.device)
    _photometric_dev(render, gt, lambda_photo_ssim, 1.0, g, values)
    return float(values[0].item()), g


def depth_distortion(distortion_map):
    """losses.py:53-56: mean per-pixel depth spread; the upstream is uniform."""
    d = _dev(distortion_map)
    H, W = int(d.shape[0]), int(d.shape[1])
    g = torch.zeros_like(d)
    values = torch.zeros((1,), dtype=torch.float64, device=d.device)
    ws = _workspace(H, W, 1)
    _lib.check(_lib.load().qgs_loss_distortion(_ptr(d), H, W, 1.0, _ptr(g), _ptr(values),
                                               _ptr(ws), ws.numel(), _stream()),
               "qgs_loss_distortion")
    return float(values[0].item()), g


def depth_to_normal(depth, alpha, cam, alpha_thresh=0.5):
    """losses.py:59-89: camera-frame normals from central differences of the
    back-projected depth (distance along the unit pixel ray).  Returns
    (N (H, W, 3) fp32, mask (H, W) bool)."""
    depth, alpha = _dev(depth), _dev(alpha)
    H, W = int(depth.shape[0]), int(depth.shape[1])
    if (int(cam.height), int(cam.width)) != (H, W):
        raise ValueError("depth map size does not match the camera")
    N = torch.empty((H, W, 3), dtype=torch.float32, device=depth.device)
    mask = torch.empty((H, W), dtype=torch.uint8, device=depth.device)
    _lib.check(_lib.load().qgs_depth_to_normal(_ptr(depth), _ptr(alpha), _cam_struct(cam),
                                               float(alpha_thresh), _ptr(N), _ptr(mask),
                                               _stream()), "qgs_depth_to_normal")
    return N, mask.bool()


def lambda_curvature(K, eps):
    """losses.py:92-94: 1 - sigmoid(ln(|K| + eps)) == 1 / (1 + |K| + eps)."""
    if isinstance(K, torch.Tensor):
        return 1.0 / (1.0 + K.abs() + eps)
    return 1.0 / (1.0 + np.abs(K) + eps)


class _MapCam:
    """intrinsics-free stand-in: the N / mask form of the consistency loss
    only needs the map size"""

    def __init__(self, H, W):
        self.fx = self.fy = 1.0
        self.cx = self.cy = 0.0
        self.width, self.height = W, H
        self.world_to_camera = np.eye(4)


def curvature_guided_normal_consistency(alpha, normal_map, curv_map, N, mask,
                                        eps_curvature=1e-6, guided=True):
    """losses.py:97-113: per-pixel lambda_K(K) (alpha - n . N) over the mask.
    Returns (value, d_alpha, d_normal, d_curvature); N and mask are constants."""
    alpha, normal_map = _dev(alpha), _dev(normal_map)
    curv_map, N = _dev(curv_map), _dev(N)
    mask = _dev(mask, torch.uint8)
    H, W = int(alpha.shape[0]), int(alpha.shape[1])
    da = torch.zeros_like(alpha)
    dn = torch.zeros_like(normal_map)
    dk = torch.zeros_like(curv_map)
    values = torch.zeros((2,), dtype=torch.float64, device=alpha.device)
    ws = _workspace(H, W, 1)
    _lib.check(_lib.load().qgs_loss_normal_consistency(
        _ptr(alpha), _ptr(normal_map), _ptr(curv_map), None, _ptr(N), _ptr(mask),
        _cam_struct(_MapCam(H, W)), 0.5, float(eps_curvature), int(bool(guided)), 1.0,
        _ptr(da), _ptr(dn), _ptr(dk), _ptr(values), _ptr(ws), ws.numel(), _stream()),
        "qgs_loss_normal_consistency")
    return float(values[0].item()), da, dn, dk


def total_loss(l_c, l_d, l_kn, l_mv, weights: LossWeights):
    """losses.py:116-118."""
    return (l_c + weights.lambda_d * l_d + weights.lambda_n * l_kn
            + weights.lambda_mv * l_mv)


def accumulate_upstream(targets, gt, cam, upstream, weights: LossWeights = None,
                        use_distortion=True, use_normal=True, guided=True, alpha_thresh=0.5):
    """The training step's loss block (train.py:193-211) fused on the device.

    Adds lambda-weighted gradients of the photometric, distortion and
    curvature-guided normal-consistency terms into ``upstream`` (the dict of
    ``rasterizer.zero_upstream``) and returns a device float64 tensor
    [l_c, l_d, l_kn] without synchronising.  The depth-derived normals are
    computed inside the consistency kernel (never written to HBM)."""
    w = weights or LossWeights()
    color = targets.color
    H, W = int(color.shape[0]), int(color.shape[1])
    gt = _dev(gt)
    parts = torch.zeros((3,), dtype=torch.float64, device=color.device)
    vals = torch.zeros((6,), dtype=torch.float64, device=color.device)
    _photometric_dev(color, gt, w.lambda_photo_ssim, 1.0, upstream["color"], vals[0:3])
    L = _lib.load()
    ws = _workspace(H, W, 3)
    if use_distortion and w.lambda_d > 0:
        _lib.check(L.qgs_loss_distortion(_ptr(targets.distortion), H, W, float(w.lambda_d),
                                         _ptr(upstream["distortion"]), _ptr(vals[3:4]), _ptr(ws),
                                         ws.numel(), _stream()), "qgs_loss_distortion")
    if use_normal and w.lambda_n > 0:
        _lib.check(L.qgs_loss_normal_consistency(
            _ptr(targets.alpha), _ptr(targets.normal), _ptr(targets.curvature),
            _ptr(targets.depth_median), None, None, _cam_struct(cam), float(alpha_thresh),
            float(w.eps_curvature), int(bool(guided)), float(w.lambda_n), _ptr(upstream["alpha"]),
            _ptr(upstream["normal"]), _ptr(upstream["curvature"]), _ptr(vals[4:6]), _ptr(ws),
            ws.numel(), _stream()), "qgs_loss_normal_consistency")
    parts[0] = vals[0]
    parts[1] = vals[3]
    parts[2] = vals[4]
    return parts
