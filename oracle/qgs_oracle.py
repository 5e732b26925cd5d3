"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU float64 restatement of the reference QGS rasterizer path
(/root/reference/pkg/src/qgsplat/rasterizer.py:123-340 and the modules it
calls).  Vectorised per-primitive work (activations, rotations, spherical
harmonics, tight screen boxes, pair expansion, lexsort, the raw-parameter
chain) is numpy, written with the same numpy operations as the reference so
that the results are bit-identical; the per-pixel loops are the C
restatement in ``qgs_kernels.c`` (OpenMP over tiles).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product package never does.
"""

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "libqgs_oracle.so")

# model.py:16-17, bounds.py:19-23, intersect.py:22
S_MIN = 1e-4
S3_FLAT = 1e-6
TILE = 16
A_TIGHT_MIN = 1e-9
T_NEAR_CLIP = 0.01
NG = 33

# sh.py:9-15 (real SH constants, degrees 0..3)
_SH_C0 = 0.28209479177387814
_SH_C1 = 0.4886025119029199
_SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
          -1.0925484305920792, 0.5462742152960396)
_SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
          0.3731763325901154, -0.4570457994644658, 1.445305721320277,
          -0.5900435899266435)


# --------------------------------------------------------------- C library

def build(force=False):
    """Compile qgs_kernels.c into oracle/lib (gcc, OpenMP, no FP contraction)."""
    src = os.path.join(_HERE, "qgs_kernels.c")
    if not force and os.path.exists(_LIB_PATH) and \
            os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


_lib = None


class _Prims(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in
        ("ohat", "M", "wv", "sv", "lam", "alpha", "colors", "Nmat", "planar", "bbox")]


class _Settings(ctypes.Structure):
    _fields_ = [("resort", ctypes.c_int32), ("euclid", ctypes.c_int32),
                ("t_clip", ctypes.c_double), ("alpha_floor", ctypes.c_double),
                ("alpha_clamp", ctypes.c_double), ("t_term", ctypes.c_double)]


class _Hit(ctypes.Structure):
    _fields_ = [("valid", ctypes.c_int), ("branch", ctypes.c_int)] + [
        (n, ctypes.c_double) for n in
        ("t", "x", "y", "rho", "cth", "sth", "a", "l", "sig", "G")]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i64, vp = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        L.qo_arc_length.restype = d
        L.qo_arc_length.argtypes = [d, d]
        L.qo_arc_length_grad.argtypes = [d, d, vp]
        L.qo_sigma_dir.restype = d
        L.qo_sigma_dir.argtypes = [d, d, d, d]
        L.qo_sigma_dir_grad.argtypes = [d, d, d, d, vp]
        L.qo_fragment_geometry.argtypes = [d] * 12 + [ctypes.c_int, ctypes.c_int, d,
                                                       ctypes.POINTER(_Hit)]
        L.qo_forward.argtypes = [i64, i64, vp, vp, vp, i64, i64, ctypes.POINTER(_Prims),
                                 ctypes.POINTER(_Settings)] + [vp] * 11 + [vp, i64]
        L.qo_backward.restype = ctypes.c_int
        L.qo_backward.argtypes = [i64, i64, vp, vp, vp, i64, i64, ctypes.POINTER(_Prims),
                                  ctypes.POINTER(_Settings)] + [vp] * 14 + [vp, i64, vp]
        L.qo_tile_keys.argtypes = [i64, vp, vp, i64, ctypes.POINTER(_Prims), vp, vp, vp,
                                   d, d, d, d, i64, i64, ctypes.c_int, d, vp]
        L.qo_num_threads.restype = ctypes.c_int
        L.qo_set_diag_prim.argtypes = [i64, vp, i64]
        L.qo_diag_rows.restype = i64
        L.qo_trace_pixel.restype = ctypes.c_int
        L.qo_trace_pixel.argtypes = [i64, vp, vp, vp, i64, ctypes.POINTER(_Prims),
                                     ctypes.POINTER(_Settings), i64, i64, ctypes.c_int] + [vp] * 8
        _lib = L
    return _lib


def num_threads():
    return lib().qo_num_threads()


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------- scalar helpers

def arc_length(a, rho):
    return lib().qo_arc_length(float(a), float(rho))


def arc_length_grad(a, rho):
    out = np.zeros(3)
    lib().qo_arc_length_grad(float(a), float(rho), _p(out))
    return tuple(out)


def sigma_dir(s1, s2, c, s):
    return lib().qo_sigma_dir(float(s1), float(s2), float(c), float(s))


def sigma_dir_grad(s1, s2, c, s):
    out = np.zeros(5)
    lib().qo_sigma_dir_grad(float(s1), float(s2), float(c), float(s), _p(out))
    return tuple(out)


def fragment_geometry(w1, w2, iw3, s1, s2, s3, o, d, planar=False, euclid=False,
                      t_clip=T_NEAR_CLIP):
    """(valid, t, x, y, rho, cth, sth, a, l, sig, G, branch) of one local ray."""
    h = _Hit()
    lib().qo_fragment_geometry(*(float(v) for v in (w1, w2, iw3, s1, s2, s3, *o, *d)),
                               int(planar), int(euclid), float(t_clip), ctypes.byref(h))
    return (bool(h.valid), h.t, h.x, h.y, h.rho, h.cth, h.sth, h.a, h.l, h.sig, h.G,
            h.branch)


# ---------------------------------------------------- per-primitive numpy

def sign0(v):
    """model.py:24-26 -- sign with sign0(0) = +1."""
    return np.where(np.asarray(v) < 0, -1.0, 1.0)


def signed_scales(raw_scales, raw_signs):
    """model.py:29-45 -- tanh(sign) * exp(scale), |s1|,|s2| floored at S_MIN."""
    raw_scales = np.asarray(raw_scales, dtype=np.float64)
    raw_signs = np.asarray(raw_signs, dtype=np.float64)
    if not (np.isfinite(raw_scales).all() and np.isfinite(raw_signs).all()):
        raise ValueError("non-finite raw scale/sign")
    s = np.tanh(raw_signs) * np.exp(raw_scales)
    floor = np.zeros(s.shape, dtype=bool)
    floor[:, :2] = np.abs(s[:, :2]) < S_MIN
    s = s.copy()
    s[:, :2] = np.where(floor[:, :2], sign0(s[:, :2]) * S_MIN, s[:, :2])
    return s, floor


def rotations(q):
    """model.py:70-87 -- normalised (w,x,y,z) quaternions to (P,3,3)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((len(q), 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def rotation_vjp(q_raw, g_R):
    """model.py:90-110 -- dL/dR (P,3,3) to dL/dq_raw (P,4) through |q|."""
    q_raw = np.asarray(q_raw, dtype=np.float64)
    nq = np.linalg.norm(q_raw, axis=-1, keepdims=True)
    q = q_raw / nq
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    o = np.zeros_like(w)

    def m3(rows):
        return np.stack([np.stack(r, axis=-1) for r in rows], axis=-2)

    partials = (
        m3([[o, -2 * z, 2 * y], [2 * z, o, -2 * x], [-2 * y, 2 * x, o]]),
        m3([[o, 2 * y, 2 * z], [2 * y, -4 * x, -2 * w], [2 * z, 2 * w, -4 * x]]),
        m3([[-4 * y, 2 * x, 2 * w], [2 * x, o, 2 * z], [-2 * w, 2 * z, -4 * y]]),
        m3([[-4 * z, -2 * w, 2 * x], [2 * w, -4 * z, 2 * y], [2 * x, 2 * y, o]]),
    )
    gu = np.stack([np.sum(g_R * dR, axis=(-2, -1)) for dR in partials], axis=-1)
    return (gu - q * np.sum(gu * q, axis=-1, keepdims=True)) / nq


def _sh_basis(deg, d):
    """sh.py:22-46 -- real SH basis (P, (deg+1)^2) at unit directions."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    Y = np.empty((len(d), (deg + 1) ** 2))
    Y[:, 0] = _SH_C0
    if deg >= 1:
        Y[:, 1] = -_SH_C1 * y
        Y[:, 2] = _SH_C1 * z
        Y[:, 3] = -_SH_C1 * x
    if deg >= 2:
        c = _SH_C2
        Y[:, 4] = c[0] * x * y
        Y[:, 5] = c[1] * y * z
        Y[:, 6] = c[2] * (2 * z * z - x * x - y * y)
        Y[:, 7] = c[3] * x * z
        Y[:, 8] = c[4] * (x * x - y * y)
    if deg >= 3:
        c = _SH_C3
        Y[:, 9] = c[0] * y * (3 * x * x - y * y)
        Y[:, 10] = c[1] * x * y * z
        Y[:, 11] = c[2] * y * (4 * z * z - x * x - y * y)
        Y[:, 12] = c[3] * z * (2 * z * z - 3 * x * x - 3 * y * y)
        Y[:, 13] = c[4] * x * (4 * z * z - x * x - y * y)
        Y[:, 14] = c[5] * z * (x * x - y * y)
        Y[:, 15] = c[6] * x * (x * x - 3 * y * y)
    return Y


def _sh_basis_jac(deg, d):
    """sh.py:49-79 -- d(basis)/d(dir), (P, K, 3)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    o = np.zeros_like(x)
    J = np.zeros((len(d), (deg + 1) ** 2, 3))
    if deg >= 1:
        J[:, 1] = np.stack([o, -_SH_C1 + o, o], axis=-1)
        J[:, 2] = np.stack([o, o, _SH_C1 + o], axis=-1)
        J[:, 3] = np.stack([-_SH_C1 + o, o, o], axis=-1)
    if deg >= 2:
        c = _SH_C2
        J[:, 4] = np.stack([c[0] * y, c[0] * x, o], axis=-1)
        J[:, 5] = np.stack([o, c[1] * z, c[1] * y], axis=-1)
        J[:, 6] = np.stack([-2 * c[2] * x, -2 * c[2] * y, 4 * c[2] * z], axis=-1)
        J[:, 7] = np.stack([c[3] * z, o, c[3] * x], axis=-1)
        J[:, 8] = np.stack([2 * c[4] * x, -2 * c[4] * y, o], axis=-1)
    if deg >= 3:
        c = _SH_C3
        J[:, 9] = np.stack([6 * c[0] * x * y, c[0] * (3 * x * x - 3 * y * y), o], axis=-1)
        J[:, 10] = np.stack([c[1] * y * z, c[1] * x * z, c[1] * x * y], axis=-1)
        J[:, 11] = np.stack([-2 * c[2] * x * y, c[2] * (4 * z * z - x * x - 3 * y * y),
                             8 * c[2] * y * z], axis=-1)
        J[:, 12] = np.stack([-6 * c[3] * x * z, -6 * c[3] * y * z,
                             c[3] * (6 * z * z - 3 * x * x - 3 * y * y)], axis=-1)
        J[:, 13] = np.stack([c[4] * (4 * z * z - 3 * x * x - y * y), -2 * c[4] * x * y,
                             8 * c[4] * x * z], axis=-1)
        J[:, 14] = np.stack([2 * c[5] * x * z, -2 * c[5] * y * z, c[5] * (x * x - y * y)],
                            axis=-1)
        J[:, 15] = np.stack([c[6] * (3 * x * x - 3 * y * y), -6 * c[6] * x * y, o], axis=-1)
    return J


def _sh_degree(sh):
    return int(round(np.sqrt(sh.shape[2]))) - 1


def sh_colors(sh, d):
    """sh.py:82-88 -- colour = sum coeff*basis + 0.5, negative channels -> 0."""
    raw = np.einsum("nck,nk->nc", sh, _sh_basis(_sh_degree(sh), d)) + 0.5
    neg = raw < 0
    return np.where(neg, 0.0, raw), neg


def sh_colors_vjp(sh, d, neg, g_color):
    """sh.py:91-99 -- (g_sh, g_dir); clamped channels pass nothing."""
    deg = _sh_degree(sh)
    g = np.where(neg, 0.0, g_color)
    g_sh = np.einsum("nc,nk->nck", g, _sh_basis(deg, d))
    g_dir = np.einsum("nc,nck,nkd->nd", g, sh, _sh_basis_jac(deg, d))
    return g_sh, g_dir


# ------------------------------------------------------------ screen boxes

def _radius(a, sig):
    # geodesic.py:80-91 inlined as in bounds.py:177-178
    return 14.0 * sig / (6.0 + np.sqrt(36.0 + 112.0 * a * sig))


def _axis_curvatures(sc):
    a0 = sc[:, 2] * sign0(sc[:, 0]) / sc[:, 0] ** 2
    a1 = sc[:, 2] * sign0(sc[:, 1]) / sc[:, 1] ** 2
    return a0, a1


def _support_box(sc):
    """bounds.py:167-195 -- local 3-sigma support box corners (P,8,3)."""
    m1, m2, m3 = np.abs(sc[:, 0]), np.abs(sc[:, 1]), np.abs(sc[:, 2])
    a0, a1 = _axis_curvatures(sc)
    flat = m3 < S3_FLAT
    amin = np.where(a0 * a1 < 0, 0.0, np.minimum(np.abs(a0), np.abs(a1)))
    amax = np.maximum(np.abs(a0), np.abs(a1))
    r1 = np.where(flat, 3.0 * m1, _radius(amin, 3.0 * m1))
    r2 = np.where(flat, 3.0 * m2, _radius(amin, 3.0 * m2))
    big, small = np.maximum(m1, m2), np.minimum(m1, m2)
    zb = np.maximum(0.0, (21.0 * big - 6.0 * _radius(amax, 3.0 * small)) / 4.0)
    zlo = np.where(flat, 0.0, np.where((a0 < 0) | (a1 < 0), -zb, 0.0))
    zhi = np.where(flat, 0.0, np.where((a0 > 0) | (a1 > 0), zb, 0.0))
    out = np.empty((len(sc), 8, 3))
    k = 0
    for ex in (-1, 1):
        for ey in (-1, 1):
            for ez in (zlo, zhi):
                out[:, k, 0] = ex * r1
                out[:, k, 1] = ey * r2
                out[:, k, 2] = ez
                k += 1
    return out


def _tangent_frustum(sc):
    """bounds.py:198-231 -- elliptic tangent-plane frustum corners + mask."""
    m1, m2, m3 = np.abs(sc[:, 0]), np.abs(sc[:, 1]), np.abs(sc[:, 2])
    c0, c1 = _axis_curvatures(sc)
    ok = (m3 >= S3_FLAT) & (c0 * c1 > 0) & \
        (np.minimum(np.abs(c0), np.abs(c1)) >= A_TIGHT_MIN)
    zs = np.where(c0 > 0, 1.0, -1.0)
    a0 = np.where(ok, np.abs(c0), 1.0)
    a1 = np.where(ok, np.abs(c1), 1.0)
    q1 = _radius(a0, 3.0 * m1)
    q2 = _radius(a1, 3.0 * m2)
    big, small = np.maximum(m1, m2), np.minimum(m1, m2)
    zb = np.maximum(0.0, (21.0 * big - 6.0 * _radius(np.maximum(a0, a1), 3.0 * small)) / 4.0)
    h = np.maximum(zb, np.maximum(a0 * q1 ** 2, a1 * q2 ** 2))
    e1 = (h / a0 + q1 * q1) / (2.0 * q1)
    e2 = (h / a1 + q2 * q2) / (2.0 * q2)
    out = np.empty((len(sc), 8, 3))
    k = 0
    for ex in (-1, 1):
        for ey in (-1, 1):
            out[:, k, 0] = ex * q1 / 2
            out[:, k, 1] = ey * q2 / 2
            out[:, k, 2] = 0.0
            out[:, k + 4, 0] = ex * e1
            out[:, k + 4, 1] = ey * e2
            out[:, k + 4, 2] = zs * h
            k += 1
    return out, ok


def _pixel_box(world, cam, z_eps=1e-6):
    """bounds.py:234-269 -- inclusive pixel AABB of projected corners."""
    pc = world @ cam.R_wc.T + cam.t_wc
    z = pc[:, :, 2]
    front = z > z_eps
    every, some = front.all(axis=1), front.any(axis=1)
    zz = np.where(front, z, 1.0)
    u = cam.fx * pc[:, :, 0] / zz + cam.cx
    v = cam.fy * pc[:, :, 1] / zz + cam.cy
    inf = 1e18
    umin = np.floor(np.where(front, u, inf).min(axis=1) - 0.5)
    vmin = np.floor(np.where(front, v, inf).min(axis=1) - 0.5)
    umax = np.ceil(np.where(front, u, -inf).max(axis=1) - 0.5)
    vmax = np.ceil(np.where(front, v, -inf).max(axis=1) - 0.5)
    box = np.empty((len(world), 4), dtype=np.int64)
    box[:, 0] = np.clip(umin, 0, cam.width - 1)
    box[:, 1] = np.clip(umax, 0, cam.width - 1)
    box[:, 2] = np.clip(vmin, 0, cam.height - 1)
    box[:, 3] = np.clip(vmax, 0, cam.height - 1)
    box[some & ~every] = (0, cam.width - 1, 0, cam.height - 1)
    gone = ~some | (box[:, 0] > box[:, 1]) | (box[:, 2] > box[:, 3])
    box[gone] = (0, -1, 0, -1)
    return box


def screen_boxes(sc, centers, R, cam):
    """bounds.py:272-292 -- loose box intersected with the frustum box."""
    loose = _pixel_box(np.einsum("pij,pkj->pki", R, _support_box(sc))
                       + centers[:, None, :], cam)
    fc, ok = _tangent_frustum(sc)
    fr = _pixel_box(np.einsum("pij,pkj->pki", R, fc) + centers[:, None, :], cam)
    box = loose.copy()
    live_l = loose[:, 0] <= loose[:, 1]
    both = ok & live_l & (fr[:, 0] <= fr[:, 1])
    box[both, 0] = np.maximum(loose[both, 0], fr[both, 0])
    box[both, 1] = np.minimum(loose[both, 1], fr[both, 1])
    box[both, 2] = np.maximum(loose[both, 2], fr[both, 2])
    box[both, 3] = np.minimum(loose[both, 3], fr[both, 3])
    box[ok & ((fr[:, 0] > fr[:, 1]) | (fr[:, 2] > fr[:, 3])) & live_l] = (0, -1, 0, -1)
    box[(box[:, 0] > box[:, 1]) | (box[:, 2] > box[:, 3])] = (0, -1, 0, -1)
    return box


# ------------------------------------------------------------------ camera

class Cam:
    """Pinhole camera view used by the oracle (cameras.py:15-94 semantics)."""

    def __init__(self, cam):
        self.fx, self.fy = float(cam.fx), float(cam.fy)
        self.cx, self.cy = float(cam.cx), float(cam.cy)
        self.width, self.height = int(cam.width), int(cam.height)
        self.w2c = np.asarray(cam.world_to_camera, dtype=np.float64)
        self.R_wc = self.w2c[:3, :3]
        self.t_wc = self.w2c[:3, 3]
        self.R_cw = self.R_wc.T
        self.center = -self.R_wc.T @ self.t_wc

    def to_cam(self, pts):
        return np.asarray(pts, dtype=np.float64) @ self.R_wc.T + self.t_wc

    def project(self, pts):
        pc = self.to_cam(pts)
        return (self.fx * pc[..., 0] / pc[..., 2] + self.cx,
                self.fy * pc[..., 1] / pc[..., 2] + self.cy)

    def pixel_dirs(self):
        u = (np.arange(self.width) + 0.5 - self.cx) / self.fx
        v = (np.arange(self.height) + 0.5 - self.cy) / self.fy
        uu, vv = np.meshgrid(u, v)
        d = np.stack([uu, vv, np.ones_like(uu)], axis=-1)
        return np.ascontiguousarray(d / np.linalg.norm(d, axis=-1, keepdims=True))


# ----------------------------------------------------------------- prepare

@dataclass
class Settings:
    """rasterizer.py:22-30 defaults."""
    background: tuple = (0.0, 0.0, 0.0)
    t_near_clip: float = T_NEAR_CLIP
    alpha_floor: float = 1.0 / 255.0
    alpha_clamp: float = 0.999
    t_term: float = 1e-4
    resort: bool = True
    euclidean_density: bool = False


def _settings(st):
    st = st or Settings()
    return _Settings(int(bool(st.resort)), int(bool(st.euclidean_density)),
                     float(st.t_near_clip), float(st.alpha_floor),
                     float(st.alpha_clamp), float(st.t_term))


class View:
    """Everything rasterizer.prepare puts in a PreparedView, as numpy arrays."""

    def _cstruct(self):
        keep = [np.ascontiguousarray(a) for a in (
            self.ohat, self.M, self.wv, self.scales, self.lam, self.alphas,
            self.colors, self.Nmat, self.planar, self.pix_bbox)]
        self._keep = keep
        return _Prims(len(self.alphas), *(_p(a) for a in keep))


def _as64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _tile_list_args(vw):
    tl = getattr(vw, "tile_list", None)
    if tl is None:
        return (None, 0)
    vw._tl = np.ascontiguousarray(tl, dtype=np.int64)
    return (_p(vw._tl), len(vw._tl))


def prepare(prims, cam, settings=None, tile_subset=None):
    """rasterizer.py:123-195.  `tile_subset` restricts the pairs (and the later
    forward/backward) to those tiles -- used only to time a bounded sample."""
    t_start = time.perf_counter()
    st = settings or Settings()
    cam = cam if isinstance(cam, Cam) else Cam(cam)
    centers, quats = _as64(prims.centers), _as64(prims.quats)
    raw_opacity, sh = _as64(prims.raw_opacity), _as64(prims.sh)
    P = len(centers)
    vw = View()
    vw.cam, vw.settings, vw.prims = cam, st, prims
    sc, vw.clamped = signed_scales(prims.raw_scales, prims.raw_signs)
    vw.scales = sc
    vw.alphas = 1.0 / (1.0 + np.exp(-raw_opacity))
    R = rotations(quats).reshape(P, 3, 3)
    vw.R = R
    s1, s2, s3 = sc[:, 0], sc[:, 1], sc[:, 2]
    vw.planar = (np.abs(s3) < S3_FLAT).astype(np.uint8)
    w1 = sign0(s1) / s1 ** 2
    w2 = sign0(s2) / s2 ** 2
    iw3 = np.where(vw.planar == 1, 0.0, 1.0 / np.where(vw.planar == 1, 1.0, s3))
    vw.wv = np.ascontiguousarray(np.stack([w1, w2, iw3], axis=1))
    vw.lam = np.ascontiguousarray(np.stack([s3 * w1, s3 * w2], axis=1))
    eye = cam.center
    vw.ohat = np.ascontiguousarray(np.einsum("pji,pj->pi", R, eye - centers))
    vw.M = np.ascontiguousarray(np.einsum("pji,jk->pik", R, cam.R_cw))
    vw.Nmat = np.ascontiguousarray(np.einsum("ij,pjk->pik", cam.R_wc, R))
    rel = centers - eye
    dist = np.maximum(np.linalg.norm(rel, axis=1), 1e-12)
    vw.view_dist = dist
    vw.view_dirs = rel / dist[:, None]
    colors, vw.color_clamped = sh_colors(sh, vw.view_dirs)
    vw.colors = np.ascontiguousarray(colors)

    tx_n = (cam.width + TILE - 1) // TILE
    ty_n = (cam.height + TILE - 1) // TILE
    vw.tiles_x, vw.tiles_y = tx_n, ty_n
    box = screen_boxes(sc, centers, R, cam)
    tm = vw.timing = {"per_primitive": time.perf_counter() - t_start}
    vw.pix_bbox = box
    live = box[:, 0] <= box[:, 1]
    bx0, bx1, by0, by1 = box[:, 0] // TILE, box[:, 1] // TILE, box[:, 2] // TILE, box[:, 3] // TILE
    vw.tile_list = None
    per = np.where(live, (bx1 - bx0 + 1) * (by1 - by0 + 1), 0)
    vw.n_pairs_full = int(per.sum())

    def expand(per):
        n_pairs = int(per.sum())
        owner = np.repeat(np.arange(P, dtype=np.int64), per)
        tiles = np.zeros(n_pairs, dtype=np.int64)
        if n_pairs:
            first = np.concatenate([[0], np.cumsum(per)[:-1]])
            k = np.arange(n_pairs, dtype=np.int64) - first[owner]
            cols = (bx1 - bx0 + 1)[owner]
            tiles = (by0[owner] + k // cols) * tx_n + bx0[owner] + k % cols
        return n_pairs, owner, tiles

    t_mark = time.perf_counter()
    if tile_subset is None:
        n_pairs, owner, tiles = expand(per)
        tm["pair_expand"] = time.perf_counter() - t_mark
    else:
        # CPU-baseline sampling: only the pairs that fall in the given tiles,
        # in the same (primitive, row-major tile) order
        S = np.unique(np.asarray(tile_subset, dtype=np.int64))
        vw.tile_list = S
        sx, sy = S % tx_n, S // tx_n
        own, til = [], []
        for c0 in range(0, P, 65536):
            sl = slice(c0, min(P, c0 + 65536))
            m = (live[sl, None] & (bx0[sl, None] <= sx[None]) & (sx[None] <= bx1[sl, None])
                 & (by0[sl, None] <= sy[None]) & (sy[None] <= by1[sl, None]))
            pi, si = np.nonzero(m)
            own.append(pi + c0)
            til.append(S[si])
        owner = np.concatenate(own).astype(np.int64)
        tiles = np.concatenate(til).astype(np.int64)
        n_pairs = len(owner)
        # the same vectorised expansion on the sampled pair count stands in
        # for the full expansion's cost (its own result is not used)
        t_mark = time.perf_counter()
        expand(np.bincount(owner, minlength=P))
        tm["pair_expand"] = time.perf_counter() - t_mark
    vw.n_pairs_sampled = n_pairs
    t_mark = time.perf_counter()
    vu, vv = cam.project(centers)
    keys = np.empty(n_pairs)
    cs = vw._cstruct()
    lib().qo_tile_keys(n_pairs, _p(tiles), _p(owner), tx_n, ctypes.byref(cs),
                       _p(_as64(vu)), _p(_as64(vv)), _p(dist), cam.cx, cam.cy,
                       cam.fx, cam.fy, cam.width, cam.height,
                       int(bool(st.euclidean_density)), float(st.t_near_clip), _p(keys))
    vw.pair_tiles_unsorted, vw.pair_prims_unsorted, vw.keys_unsorted = tiles, owner, keys
    tm["keys"] = time.perf_counter() - t_mark
    t_mark = time.perf_counter()
    order = np.lexsort((owner, keys, tiles))
    vw.keys = keys[order]
    vw.tile_prims = owner[order]
    counts = np.bincount(tiles[order], minlength=tx_n * ty_n)
    vw.tile_offsets = np.zeros(tx_n * ty_n + 1, dtype=np.int64)
    np.cumsum(counts, out=vw.tile_offsets[1:])
    tm["sort"] = time.perf_counter() - t_mark
    t_mark = time.perf_counter()
    vw.dirs = cam.pixel_dirs()
    tm["dirs"] = time.perf_counter() - t_mark
    return vw


# ----------------------------------------------------------------- forward

def forward(vw):
    """rasterizer.py:198-227; returns a dict of (H, W[, 3]) float64 maps."""
    cam, st = vw.cam, vw.settings
    H, W = cam.height, cam.width
    o = {k: np.zeros((H, W, 3)) for k in ("color_raw", "normal")}
    for k in ("alpha", "depth", "depth_sq", "depth_median", "curvature", "distortion"):
        o[k] = np.zeros((H, W))
    o["transmittance"] = np.ones((H, W))
    o["n_fragments"] = np.zeros((H, W), dtype=np.int64)
    viol = np.zeros(vw.tiles_x * vw.tiles_y, dtype=np.int64)
    cs, cst = vw._cstruct(), _settings(st)
    lib().qo_forward(H, W, _p(vw.dirs), _p(vw.tile_offsets), _p(vw.tile_prims),
                     vw.tiles_x, vw.tiles_y, ctypes.byref(cs), ctypes.byref(cst),
                     _p(o["color_raw"]), _p(o["alpha"]), _p(o["depth"]), _p(o["depth_sq"]),
                     _p(o["depth_median"]), _p(o["normal"]), _p(o["curvature"]),
                     _p(o["distortion"]), _p(o["transmittance"]), _p(o["n_fragments"]),
                     _p(viol), *_tile_list_args(vw))
    bg = np.asarray(st.background, dtype=np.float64)
    o["color"] = o["color_raw"] + o["transmittance"][:, :, None] * bg
    o["order_violations"] = int(viol.sum())
    o["violations_per_tile"] = viol
    return o


# ---------------------------------------------------------------- backward

def kernel_grads(vw, targets, upstream, with_abs=False):
    """rasterizer.py:237-266 -- the per-primitive 33-slot kernel gradients.
    with_abs: also return the per-slot sums of |each fragment's contribution|
    (diagnostics: the cancellation scale of every slot)."""
    cam, st = vw.cam, vw.settings
    H, W = cam.height, cam.width

    def up(key, shape):
        a = upstream.get(key)
        return np.zeros(shape) if a is None else _as64(a)

    u_color = up("color", (H, W, 3))
    u_alpha = np.array(up("alpha", (H, W)))
    bg = np.asarray(st.background, dtype=np.float64)
    u_alpha = np.ascontiguousarray(u_alpha - u_color @ bg)
    u_depth, u_normal = up("depth", (H, W)), up("normal", (H, W, 3))
    u_curv, u_dist = up("curvature", (H, W)), up("distortion", (H, W))
    kg = np.zeros((len(vw.alphas), NG))
    kg_abs = np.zeros((len(vw.alphas), NG)) if with_abs else None
    cs, cst = vw._cstruct(), _settings(st)
    f = {k: _as64(targets[k]) for k in ("color_raw", "alpha", "depth", "depth_sq",
                                        "normal", "curvature", "distortion")}
    rc = lib().qo_backward(H, W, _p(vw.dirs), _p(vw.tile_offsets), _p(vw.tile_prims),
                           vw.tiles_x, vw.tiles_y, ctypes.byref(cs), ctypes.byref(cst),
                           _p(f["color_raw"]), _p(f["alpha"]), _p(f["depth"]),
                           _p(f["depth_sq"]), _p(f["normal"]), _p(f["curvature"]),
                           _p(f["distortion"]), _p(u_color), _p(u_alpha), _p(u_depth),
                           _p(u_normal), _p(u_curv), _p(u_dist), _p(kg),
                           *_tile_list_args(vw), _p(kg_abs))
    if rc != 0:
        raise MemoryError("oracle backward: allocation failed")
    return (kg, kg_abs) if with_abs else kg


def fragment_contributions(vw, targets, upstream, prim, max_rows=1 << 16):
    """diagnostics: every composited fragment of primitive `prim` with its 33
    slot contributions -> (pixel index, t, (n, 33) slots)"""
    buf = np.zeros((max_rows, NG + 2))
    lib().qo_set_diag_prim(int(prim), _p(buf), max_rows)
    try:
        kernel_grads(vw, targets, upstream)
        n = min(lib().qo_diag_rows(), max_rows)
    finally:
        lib().qo_set_diag_prim(-1, None, 0)
    rows = buf[:n]
    order = np.lexsort((rows[:, 1], rows[:, 0]))
    rows = rows[order]
    return rows[:, 0].astype(np.int64), rows[:, 1], rows[:, 2:]


def chain_jacobian(vw, idx):
    """d(raw gradients) / d(kernel slots) of primitives `idx`: the chain is
    linear in the slots and per-primitive, so column j is chain() of the
    unit slot j.  Returns {group: (len(idx), group size, NG)}."""
    from types import SimpleNamespace
    idx = np.asarray(idx, dtype=np.int64)
    pr = vw.prims
    sub_prims = SimpleNamespace(**{f: np.asarray(getattr(pr, f))[idx] for f in
                                   ("centers", "quats", "raw_scales", "raw_signs",
                                    "raw_opacity", "sh")})
    sub = SimpleNamespace(prims=sub_prims, cam=vw.cam, alphas=vw.alphas[idx],
                          scales=vw.scales[idx], wv=vw.wv[idx], planar=vw.planar[idx],
                          clamped=vw.clamped[idx], R=vw.R[idx], view_dirs=vw.view_dirs[idx],
                          view_dist=vw.view_dist[idx], color_clamped=vw.color_clamped[idx])
    cols = []
    for j in range(NG):
        e = np.zeros((len(idx), NG))
        e[:, j] = 1.0
        out = chain(sub, e)
        cols.append({k: np.asarray(v).reshape(len(idx), -1) for k, v in out.items()})
    return {k: np.stack([c[k] for c in cols], axis=2) for k in cols[0]}


def chain(vw, kg):
    """rasterizer.py:270-334 -- kernel slots to raw-parameter gradients."""
    prims, cam = vw.prims, vw.cam
    P = len(vw.alphas)
    centers, quats = _as64(prims.centers), _as64(prims.quats)
    g_ohat = kg[:, 0:3]
    g_M = kg[:, 3:12].reshape(P, 3, 3)
    g_w = kg[:, 12:15].copy()
    g_s = kg[:, 15:18].copy()
    g_alpha = kg[:, 18]
    g_col = kg[:, 19:22]
    g_N = kg[:, 22:31].reshape(P, 3, 3)
    g_lam = kg[:, 31:33]
    sc, wv = vw.scales, vw.wv
    s1, s2, s3 = sc[:, 0], sc[:, 1], sc[:, 2]
    curved = vw.planar == 0
    g_s[:, 2] += g_lam[:, 0] * wv[:, 0] + g_lam[:, 1] * wv[:, 1]
    g_w[:, 0] += g_lam[:, 0] * s3
    g_w[:, 1] += g_lam[:, 1] * s3
    g_s[:, 0] += g_w[:, 0] * (-2.0 * wv[:, 0] / s1)
    g_s[:, 1] += g_w[:, 1] * (-2.0 * wv[:, 1] / s2)
    g_s[:, 2] += np.where(curved, g_w[:, 2] * (-1.0 / np.where(curved, s3, 1.0) ** 2), 0.0)
    th = np.tanh(_as64(prims.raw_signs))
    ex = np.exp(_as64(prims.raw_scales))
    free = ~vw.clamped
    out = {}
    out["raw_scales"] = np.where(free, g_s * (th * ex), 0.0)
    out["raw_signs"] = np.where(free, g_s * ((1.0 - th * th) * ex), 0.0)
    out["raw_opacity"] = g_alpha * vw.alphas * (1.0 - vw.alphas)
    g_R = np.einsum("jk,pik->pji", cam.R_cw, g_M)
    eye = cam.center
    g_R += np.einsum("pj,pi->pji", eye - centers, g_ohat)
    g_R += np.einsum("ji,pjk->pik", cam.R_wc, g_N)
    out["quats"] = rotation_vjp(quats, g_R)
    g_c = -np.einsum("pij,pj->pi", vw.R, g_ohat)
    out["sh"], g_dir = sh_colors_vjp(_as64(prims.sh), vw.view_dirs, vw.color_clamped, g_col)
    d = vw.view_dirs
    g_c += (g_dir - d * np.sum(g_dir * d, axis=1, keepdims=True)) / vw.view_dist[:, None]
    out["centers"] = g_c
    pc = cam.to_cam(centers)
    X, Y, Z = pc[:, 0], pc[:, 1], pc[:, 2]
    Zs = np.where(np.abs(Z) < 1e-9, 1e-9, Z)
    Ju = cam.fx * (cam.R_wc[0][None, :] / Zs[:, None]
                   - X[:, None] * cam.R_wc[2][None, :] / Zs[:, None] ** 2)
    Jv = cam.fy * (cam.R_wc[1][None, :] / Zs[:, None]
                   - Y[:, None] * cam.R_wc[2][None, :] / Zs[:, None] ** 2)
    gu = np.sum(Ju * g_c, axis=1) * (2.0 / cam.width)
    gv = np.sum(Jv * g_c, axis=1) * (2.0 / cam.height)
    out["screen_center"] = np.stack([gu, gv], axis=1)
    return out


def backward(vw, targets, upstream):
    """rasterizer.py:230-267."""
    return chain(vw, kernel_grads(vw, targets, upstream))


def trace_pixel(vw, u, v, max_frags=4096):
    """Accepted candidates and emitted fragments of one pixel (diagnostics)."""
    ap, at, aa = np.zeros(max_frags, np.int64), np.zeros(max_frags), np.zeros(max_frags)
    ep, et, ea, eT = (np.zeros(max_frags, np.int64), np.zeros(max_frags), np.zeros(max_frags),
                      np.zeros(max_frags))
    na = ctypes.c_int(0)
    cs, cst = vw._cstruct(), _settings(vw.settings)
    ne = lib().qo_trace_pixel(vw.cam.width, _p(vw.dirs), _p(vw.tile_offsets), _p(vw.tile_prims),
                              vw.tiles_x, ctypes.byref(cs), ctypes.byref(cst), int(u), int(v),
                              max_frags, _p(ap), _p(at), _p(aa), ctypes.byref(na), _p(ep), _p(et),
                              _p(ea), _p(eT))
    na, ne = min(na.value, max_frags), min(ne, max_frags)
    return ({"prim": ap[:na], "t": at[:na], "abar": aa[:na]},
            {"prim": ep[:ne], "t": et[:ne], "abar": ea[:ne], "T": eT[:ne]})


def time_sampled_view(prims, cam, upstream, n_sample=128, seed=0, settings=None):
    """Time prepare + forward + backward of one view on a random sample of
    its tiles and extrapolate to the whole view (CPU baseline, bench.py).

    Per-primitive work (activations, SH, screen boxes, chain) is timed in
    full; per-tile work (pair expansion, keys, sort, forward, backward) is
    timed on `n_sample` random tiles and scaled by n_tiles / n_sample."""
    cam = cam if isinstance(cam, Cam) else Cam(cam)
    n_tiles = ((cam.width + TILE - 1) // TILE) * ((cam.height + TILE - 1) // TILE)
    n = min(n_sample, n_tiles)
    # systematic sample: every (n_tiles / n)-th tile from a seeded offset,
    # which tracks the image's density profile far better than a random pick
    stride = n_tiles / n
    off = np.random.default_rng(seed).uniform(0, stride)
    S = np.unique((off + stride * np.arange(n)).astype(np.int64).clip(0, n_tiles - 1))
    n = len(S)
    vw = prepare(prims, cam, settings, tile_subset=S)
    t0 = time.perf_counter()
    fw = forward(vw)
    t1 = time.perf_counter()
    kg = kernel_grads(vw, fw, upstream)
    t2 = time.perf_counter()
    chain(vw, kg)
    t3 = time.perf_counter()
    tm = vw.timing
    pair_scale = vw.n_pairs_full / max(vw.n_pairs_sampled, 1)
    tile_scale = n_tiles / n
    est = (tm["per_primitive"] + tm["dirs"] + (t3 - t2)
           + (tm["pair_expand"] + tm["keys"] + tm["sort"]) * pair_scale
           + ((t1 - t0) + (t2 - t1)) * tile_scale)
    return {"seconds_per_view_est": est, "tiles_sampled": int(n), "tiles": int(n_tiles),
            "pairs_sampled": int(vw.n_pairs_sampled), "pairs": int(vw.n_pairs_full),
            "threads": num_threads(),
            "phases": {**{k: round(v, 4) for k, v in tm.items()}, "forward": t1 - t0,
                       "backward": t2 - t1, "chain": t3 - t2}}


def time_full_view(prims, cam, upstream, settings=None):
    """Time prepare + forward + backward (kernel gradients + chain) of one
    whole view (CPU baseline and the reference arm of bench.py): nothing
    sampled, nothing extrapolated."""
    t0 = time.perf_counter()
    vw = prepare(prims, cam, settings)
    t1 = time.perf_counter()
    fw = forward(vw)
    t2 = time.perf_counter()
    kg = kernel_grads(vw, fw, upstream)
    t3 = time.perf_counter()
    chain(vw, kg)
    t4 = time.perf_counter()
    return {"seconds": t4 - t0, "pairs": int(len(vw.tile_prims)), "threads": num_threads(),
            "phases": {**{k: round(v, 3) for k, v in vw.timing.items()},
                       "prepare": round(t1 - t0, 3), "forward": round(t2 - t1, 3),
                       "backward": round(t3 - t2, 3), "chain": round(t4 - t3, 3)}}


def cpu_model():
    """CPU model string and logical core count of this host."""
    name = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    name = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": name, "logical_cores": os.cpu_count()}


def render(prims, cam, settings=None):
    vw = prepare(prims, cam, settings)
    return forward(vw), vw
