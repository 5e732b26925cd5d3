"""Multi-view reprojection + NCC regulariser on the device -- drop-in for
``qgsplat.multiview`` (/root/reference/pkg/src/qgsplat/multiview.py).

``multiview_loss`` keeps the reference's signature and return tuple
(value, n_valid, upstream_ref, upstream_nbr, stats); maps may be numpy or
torch, the upstream maps come back as CUDA fp32 tensors.  The per-pixel
homography warp, NCC and the whole adjoint run in one fp64 kernel
(csrc/multiview.cu).  ``accumulate_multiview`` is the fused train-step form
(train.py:215-233): lambda-weighted gradients go straight into both views'
rasterizer upstream maps and the loss stays on the device.  The small host
helpers (gray, intrinsics, relative transform, plane homography) are the
reference's 3x3 algebra in numpy.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .losses import _dev
from .rasterizer import _cam_struct, _ptr, _stream

_WS = {}


@dataclass
class MultiviewConfig:
    """multiview.py:17-23."""
    patch_size: int = 7
    alpha_thresh: float = 0.5
    min_denom: float = 1e-6
    ncc_eps: float = 1e-8
    full_chain: bool = True

    def struct(self):
        c = _lib.MvConfig()
        c.patch_size = int(self.patch_size)
        c.alpha_thresh, c.min_denom = float(self.alpha_thresh), float(self.min_denom)
        c.ncc_eps, c.full_chain = float(self.ncc_eps), int(bool(self.full_chain))
        return c


def gray(img):
    """multiview.py:26-28 (host helper)."""
    img = np.asarray(img, dtype=np.float64)
    return img if img.ndim == 2 else img.mean(axis=2)


def intrinsic_matrix(cam):
    """multiview.py:31-32."""
    return np.array([[cam.fx, 0.0, cam.cx], [0.0, cam.fy, cam.cy], [0.0, 0.0, 1.0]])


def _R_t(cam):
    w2c = np.asarray(cam.world_to_camera, dtype=np.float64)
    return w2c[:3, :3], w2c[:3, 3]


def relative_transform(cam_a, cam_b):
    """multiview.py:35-39: (R, T) with X_b = R X_a + T."""
    Ra, ta = _R_t(cam_a)
    Rb, tb = _R_t(cam_b)
    R = Rb @ Ra.T
    return R, tb - R @ ta


def plane_homography(cam_a, cam_b, n_a, X_a):
    """multiview.py:42-48."""
    R, T = relative_transform(cam_a, cam_b)
    return intrinsic_matrix(cam_b) @ (R + np.outer(T, n_a) / (n_a @ X_a)) @ \
        np.linalg.inv(intrinsic_matrix(cam_a))


def _maps(m):
    depth, alpha = _dev(m["depth"]), _dev(m["alpha"])
    normal, image = _dev(m["normal"]), _dev(m["image"])
    s = _lib.MvMaps()
    s.depth, s.alpha, s.normal, s.image = _ptr(depth), _ptr(alpha), _ptr(normal), _ptr(image)
    s.height, s.width = int(alpha.shape[0]), int(alpha.shape[1])
    s.image_channels = 1 if image.dim() == 2 else int(image.shape[2])
    if tuple(depth.shape) != tuple(alpha.shape) or tuple(normal.shape[:2]) != tuple(alpha.shape) \
            or tuple(image.shape[:2]) != tuple(alpha.shape):
        raise ValueError("depth / alpha / normal / image sizes differ")
    return s, (depth, alpha, normal, image)


def _grads(up):
    g = _lib.MvGrads()
    if up is not None:
        g.depth, g.alpha, g.normal = _ptr(up.get("depth")), _ptr(up.get("alpha")), \
            _ptr(up.get("normal"))
    return g


def _run(ref_maps, cam_r, nbr_maps, cam_n, cfg, weight, up_ref, up_nbr, values):
    cfg = cfg or MultiviewConfig()
    sr, keep_r = _maps(ref_maps)
    sn, keep_n = _maps(nbr_maps)
    L = _lib.load()
    n = int(L.qgs_multiview_workspace_bytes(sr.height, sr.width, sn.height, sn.width))
    dev = keep_r[0].device
    ws = _WS.get(dev.index)
    if ws is None or ws.numel() < n:
        ws = torch.empty((n,), dtype=torch.uint8, device=dev)
        _WS[dev.index] = ws
    _lib.check(L.qgs_multiview_loss(sr, _cam_struct(cam_r), sn, _cam_struct(cam_n), cfg.struct(),
                                    float(weight), _grads(up_ref), _grads(up_nbr), _ptr(values),
                                    _ptr(ws), ws.numel(), _stream()), "qgs_multiview_loss")
    return keep_r, keep_n


def multiview_loss(ref_maps, cam_r, nbr_maps, cam_n, cfg: MultiviewConfig = None):
    """multiview.py:108-311.  Returns (value, n_valid, upstream_ref,
    upstream_nbr, stats) with upstream dicts of depth / alpha / normal."""
    dev = torch.device("cuda", torch.cuda.current_device())
    H, W = np.shape(ref_maps["alpha"])[:2]
    Hn, Wn = np.shape(nbr_maps["alpha"])[:2]
    z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)  # noqa: E731
    up_r = {"depth": z(H, W), "alpha": z(H, W), "normal": z(H, W, 3)}
    up_n = {"depth": z(Hn, Wn), "alpha": z(Hn, Wn), "normal": z(Hn, Wn, 3)}
    values = torch.zeros((4,), dtype=torch.float64, device=dev)
    _run(ref_maps, cam_r, nbr_maps, cam_n, cfg, 1.0, up_r, up_n, values)
    v = values.cpu().numpy()
    return float(v[0]), int(round(v[1])), up_r, up_n, {"warp_px": float(v[2]), "ncc": float(v[3])}


def accumulate_multiview(ref_maps, cam_r, nbr_maps, cam_n, up_ref, up_nbr, weight,
                         cfg: MultiviewConfig = None):
    """train.py:215-233 fused: adds weight * gradient into the two views'
    upstream dicts (rasterizer.zero_upstream layout) and returns the device
    float64 tensor [value, n_valid, warp_px, ncc] without synchronising."""
    values = torch.zeros((4,), dtype=torch.float64,
                         device=torch.device("cuda", torch.cuda.current_device()))
    _run(ref_maps, cam_r, nbr_maps, cam_n, cfg, weight, up_ref, up_nbr, values)
    return values
