"""SSIM (11x11 Gaussian window, sigma 1.5) and its input gradient on the
device -- drop-in for ``qgsplat.ssim`` (/root/reference/pkg/src/qgsplat/ssim.py).

The kernels are the photometric loss's (csrc/losses.cu) run with the SSIM
weight at 1, where the loss gradient is exactly -dSSIM/dx.
"""

import numpy as np
import torch

from .losses import _dev, _photometric_dev

WINDOW = 11
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def ssim(x, y, return_grad=False):
    """ssim.py:41-86: mean SSIM over the valid (crop) region, averaged over
    channels; with return_grad also dSSIM/dx (CUDA fp32, the shape of x)."""
    xs, ys = tuple(np.shape(x)), tuple(np.shape(y))
    if xs != ys:
        raise ValueError("image shapes differ")
    if len(xs) not in (2, 3):
        raise ValueError("images must be (H, W) or (H, W, C)")
    if xs[0] < WINDOW or xs[1] < WINDOW:
        raise ValueError("image smaller than the SSIM window")
    xd, yd = _dev(x), _dev(y)
    values = torch.zeros((3,), dtype=torch.float64, device=xd.device)
    g = torch.zeros_like(xd) if return_grad else None
    _photometric_dev(xd, yd, 1.0, 1.0, g, values)
    value = float(values[2].item())
    if return_grad:
        return value, -g
    return value
