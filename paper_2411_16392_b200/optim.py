"""Adam over the primitive parameter groups, on the device -- drop-in for
``qgsplat.optim`` (/root/reference/pkg/src/qgsplat/optim.py).

Parameters are a ``DevicePrimitives`` (fp32 groups in HBM); the moments are
fp32 tensors of the same shapes; the update runs in fp64 arithmetic inside
libqgs_b200.so (csrc/optim.cu, ``qgs_adam_step``).  ``step`` can fold the
densification statistics of train.py:239-244 into the same pass.
"""

import numpy as np
import torch

from . import _lib
from .rasterizer import DevicePrimitives, _ptr, _stream

GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")


def groups_struct(src, P=None, sh_coeffs=None):
    """qgs_groups over a DevicePrimitives or a dict of group tensors."""
    g = _lib.Groups()
    get = (lambda k: src[k]) if isinstance(src, dict) else (lambda k: getattr(src, k))
    for k in GROUPS:
        setattr(g, k, _ptr(get(k)))
    g.P = int(get("centers").shape[0]) if P is None else P
    g.sh_coeffs = int(get("sh").shape[2]) if sh_coeffs is None else sh_coeffs
    return g


def params_struct(src):
    p = _lib.Params()
    get = (lambda k: src[k]) if isinstance(src, dict) else (lambda k: getattr(src, k))
    for k in GROUPS:
        setattr(p, k, _ptr(get(k)))
    p.P = int(get("centers").shape[0])
    p.sh_coeffs = int(get("sh").shape[2])
    return p


class Adam:
    """optim.py:14-64."""

    def __init__(self, prims, beta1=0.9, beta2=0.999, eps=1e-15):
        prims = DevicePrimitives.from_host(prims)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.t = 0
        self.m = {g: torch.zeros_like(getattr(prims, g)) for g in GROUPS}
        self.v = {g: torch.zeros_like(getattr(prims, g)) for g in GROUPS}
        self._skipped = torch.zeros((1,), dtype=torch.int64, device=prims.centers.device)

    @property
    def skipped(self):
        """primitives whose step was skipped for non-finite gradients (syncs)"""
        return int(self._skipped.item())

    def step(self, prims, grads, lrs, freeze=None, stats=None):
        """lrs: group -> learning rate.  freeze: group -> bool mask (the
        group's shape) or None.  stats: a densify.DensifyStats to accumulate
        into before the update (train.py:239-244), or None."""
        if not isinstance(prims, DevicePrimitives):
            raise TypeError("Adam.step updates a DevicePrimitives in place")
        self.t += 1
        cfg = _lib.AdamConfig()
        cfg.lr[:] = [float(lrs[g]) for g in GROUPS]
        cfg.beta1, cfg.beta2, cfg.eps, cfg.t = self.beta1, self.beta2, self.eps, self.t
        keep_alive = []
        for i, g in enumerate(GROUPS):
            f = None if not freeze else freeze.get(g)
            if f is not None:
                f = torch.as_tensor(np.asarray(f) if not isinstance(f, torch.Tensor) else f)
                f = f.to(device=prims.centers.device, dtype=torch.uint8)
                f = f.expand_as(getattr(prims, g)).contiguous()
                keep_alive.append(f)
                cfg.freeze[i] = _ptr(f)
        st = None
        if stats is not None:
            st = stats.struct()
        _lib.check(_lib.load().qgs_adam_step(
            groups_struct(prims), grads.grads_struct(), groups_struct(self.m),
            groups_struct(self.v), cfg, st, _ptr(self._skipped), _stream()), "qgs_adam_step")
        return self

    def keep(self, mask):
        mask = torch.as_tensor(mask, device=self.m["centers"].device)
        for g in GROUPS:
            self.m[g] = self.m[g][mask].contiguous()
            self.v[g] = self.v[g][mask].contiguous()

    def extend(self, n_new):
        for g in GROUPS:
            pad = torch.zeros((n_new,) + tuple(self.m[g].shape[1:]), dtype=self.m[g].dtype,
                              device=self.m[g].device)
            self.m[g] = torch.cat([self.m[g], pad])
            self.v[g] = torch.cat([self.v[g], pad])

    def reset_group(self, group):
        self.m[group].zero_()
        self.v[group].zero_()


def center_lr(step, total, base, final_ratio, scene_extent):
    """optim.py:67-70: exponentially decayed centre learning rate."""
    frac = min(max(step / max(total, 1), 0.0), 1.0)
    return base * scene_extent * (final_ratio ** frac)
