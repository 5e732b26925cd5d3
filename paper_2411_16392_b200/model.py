"""Primitive container for the rasterizer boundary.

Mirrors qgsplat.model.PrimitiveSet (/root/reference/pkg/src/qgsplat/model.py:126-190):
struct-of-arrays raw parameters -- centers (N,3), quats (N,4) wxyz, raw_scales
(N,3), raw_signs (N,3), raw_opacity (N,), sh (N,3,(deg+1)^2).  Arrays may be
numpy (any float dtype) or torch tensors; the rasterizer uploads them as fp32.
"""

import numpy as np

S_MIN = 1e-4      # model.py:16
S3_FLAT = 1e-6    # model.py:17


class ParameterError(ValueError):
    """Raised when primitive parameters fail validation (model.py:20)."""


def _n(a):
    return a.shape[0]


class PrimitiveSet:
    FIELDS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")

    def __init__(self, centers, quats, raw_scales, raw_signs, raw_opacity, sh):
        self.centers, self.quats = centers, quats
        self.raw_scales, self.raw_signs = raw_scales, raw_signs
        self.raw_opacity, self.sh = raw_opacity, sh
        n = _n(centers)
        if not all(_n(getattr(self, f)) == n for f in self.FIELDS):
            raise ParameterError("inconsistent parameter array lengths")
        if len(sh.shape) != 3 or sh.shape[1] != 3:
            raise ParameterError("sh must have shape (N, 3, (deg+1)^2)")
        k = sh.shape[2]
        if int(round(np.sqrt(k))) ** 2 != k or k > 16:
            raise ParameterError("sh must hold (deg+1)^2 coefficients, deg <= 3")

    def __len__(self):
        return _n(self.centers)

    @property
    def sh_degree(self):
        return int(round(np.sqrt(self.sh.shape[2]))) - 1

    def astype(self, dtype):
        return PrimitiveSet(*(np.asarray(getattr(self, f), dtype=dtype) for f in self.FIELDS))

    def select(self, mask):
        return PrimitiveSet(*(getattr(self, f)[mask] for f in self.FIELDS))
