"""Seeded synthetic workloads for the BASELINE.json configs.

No public dataset is named for this path, so every config is a seeded
synthetic scene with the shapes, sizes and value distributions BASELINE.json
states.  All primitive parameters and upstream gradients are drawn and
stored in float32; the oracle receives the same values upcast exactly to
float64.  Draw order per scene: centres, quaternions, log-scales,
curvatures, opacity logits, SH DC, SH rest, camera eyes, then upstream.

The parameterisation follows the reference's own init convention
(train.py:50-55): raw_sign = 3*sign(k) and raw_scale = log(s) - log(tanh 3)
for the two in-plane axes, so s_i = sign(k_i) * exp(l_i); the height scale
s3 = 0.5*sqrt(|k1| s1^2 |k2| s2^2) (vertex curvature kappa_i = 2 s3 / s_i^2,
surface.py:3-6) with raw_sign 3, or raw_sign 0 for an exactly planar disk.
"""

from dataclasses import dataclass

import numpy as np

from .cameras import Camera, look_at
from .model import PrimitiveSet

_LOG_TANH3 = float(np.log(np.tanh(3.0)))
_SH_C0 = 0.28209479177387814


@dataclass
class Scene:
    name: str
    prims: PrimitiveSet          # float32 arrays
    cams: list
    upstream: list               # per view dict of float32 (H,W[,3]) arrays, or None
    meta: dict


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def pinhole(width, height, eye, fov_x_deg=60.0):
    f = (width / 2.0) / np.tan(np.radians(fov_x_deg) / 2.0)
    return Camera(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width,
                  height=height, world_to_camera=look_at(eye, np.zeros(3)))


def _unit(rng, n):
    v = rng.standard_normal((n, 3), dtype=np.float32).astype(np.float64)
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _quats(rng, n):
    q = rng.standard_normal((n, 4), dtype=np.float32).astype(np.float64)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _scales_from(log_s1, log_s2, k1s, k2s, planar_mask=None):
    """Raw scale/sign arrays from log in-plane scales and curvature*scale draws
    (k_i * s_i, dimensionless)."""
    s1, s2 = np.exp(log_s1), np.exp(log_s2)
    k1, k2 = k1s / s1, k2s / s2
    s3 = 0.5 * np.sqrt(np.abs(k1) * s1 ** 2 * np.abs(k2) * s2 ** 2)
    s3 = np.maximum(s3, 1e-30)
    raw_scales = np.stack([log_s1 - _LOG_TANH3, log_s2 - _LOG_TANH3,
                           np.log(s3) - _LOG_TANH3], axis=1)
    sg = lambda k: np.where(k < 0, -3.0, 3.0)  # noqa: E731
    raw_signs = np.stack([sg(k1), sg(k2), np.full_like(k1, 3.0)], axis=1)
    if planar_mask is not None:
        raw_signs[planar_mask, 2] = 0.0
    return raw_scales, raw_signs


def _sh(rng, n, deg):
    K = (deg + 1) ** 2
    sh = np.zeros((n, 3, K))
    sh[:, :, 0] = (rng.random((n, 3), dtype=np.float32).astype(np.float64) - 0.5) / _SH_C0
    if K > 1:
        sh[:, :, 1:] = 0.1 * rng.standard_normal((n, 3, K - 1), dtype=np.float32)
    return sh


def _upstream(rng, cams, keys=("color", "depth", "normal", "alpha"), all_six=False):
    ups = []
    for c in cams:
        H, W = c.height, c.width
        u = {}
        for k in ("color", "depth", "normal", "alpha", "curvature", "distortion"):
            if k in keys or all_six:
                shape = (H, W, 3) if k in ("color", "normal") else (H, W)
                u[k] = rng.standard_normal(shape, dtype=np.float32)
        ups.append(u)
    return ups


def _pack(name, centers, quats, raw_scales, raw_signs, logit, sh, cams, ups, meta):
    prims = PrimitiveSet(_f32(centers), _f32(quats), _f32(raw_scales), _f32(raw_signs),
                         _f32(logit), _f32(sh))
    return Scene(name, prims, cams, ups, meta)


def config1(seed=1, n=2048, res=128, with_upstream=True):
    """C1: forward-only N=2048 at 128^2, SH0 (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    quats = _quats(rng, n)
    ls = -3.0 + 0.3 * rng.standard_normal((n, 2), dtype=np.float32)
    ks = 0.5 * rng.standard_normal((n, 2), dtype=np.float32)
    raw_scales, raw_signs = _scales_from(ls[:, 0], ls[:, 1], ks[:, 0], ks[:, 1])
    logit = rng.standard_normal(n, dtype=np.float32)
    sh = _sh(rng, n, 0)
    eye = 3.0 * _unit(rng, 1)[0]
    cams = [pinhole(res, res, eye)]
    ups = _upstream(rng, cams) if with_upstream else None
    return _pack("c1", centers, quats, raw_scales, raw_signs, logit, sh, cams, ups,
                 {"N": n, "res": [res, res], "sh_deg": 0, "views": 1})


def config2(seed=2, n=100_000, res=800, views=4):
    """C2: N=100K at 800^2, SH3, 4 views, forward+backward."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    quats = _quats(rng, n)
    ls = -3.0 + 0.3 * rng.standard_normal((n, 2), dtype=np.float32)
    ks = 0.5 * rng.standard_normal((n, 2), dtype=np.float32)
    raw_scales, raw_signs = _scales_from(ls[:, 0], ls[:, 1], ks[:, 0], ks[:, 1])
    logit = rng.standard_normal(n, dtype=np.float32)
    sh = _sh(rng, n, 3)
    cams = [pinhole(res, res, 3.0 * e) for e in _unit(rng, views)]
    ups = _upstream(rng, cams)
    return _pack("c2", centers, quats, raw_scales, raw_signs, logit, sh, cams, ups,
                 {"N": n, "res": [res, res], "sh_deg": 3, "views": views})


def config3(seed=3, n=500_000, width=1600, height=1200, views=8, sigma_n=0.02):
    """C3 (headline): N=500K at 1600x1200, SH3, 8 views; 80% of centres on a
    noisy unit sphere (radial noise sigma_n, unspecified upstream -> 0.02),
    20% uniform clutter in [-1,1]^3; k ~ N(0,1)/s; logit N(1,1)."""
    rng = np.random.default_rng(seed)
    n_s = int(round(0.8 * n))
    dirs = _unit(rng, n_s)
    rad = 1.0 + sigma_n * rng.standard_normal(n_s, dtype=np.float32)
    clutter = rng.uniform(-1, 1, (n - n_s, 3)).astype(np.float32)
    centers = np.concatenate([dirs * rad[:, None], clutter])
    quats = _quats(rng, n)
    ls = -3.0 + 0.3 * rng.standard_normal((n, 2), dtype=np.float32)
    ks = 1.0 * rng.standard_normal((n, 2), dtype=np.float32)
    raw_scales, raw_signs = _scales_from(ls[:, 0], ls[:, 1], ks[:, 0], ks[:, 1])
    logit = 1.0 + rng.standard_normal(n, dtype=np.float32)
    sh = _sh(rng, n, 3)
    cams = [pinhole(width, height, 3.0 * e) for e in _unit(rng, views)]
    ups = _upstream(rng, cams)
    return _pack("c3", centers, quats, raw_scales, raw_signs, logit, sh, cams, ups,
                 {"N": n, "res": [width, height], "sh_deg": 3, "views": views,
                  "sigma_n": sigma_n})


def config4(seed=4, n=2_000_000, width=1920, height=1080, views=64, r_min=0.05,
            with_upstream=True):
    """C4: N=2M, 1920x1080, 64 views on the radius-5 upper hemisphere; centres
    log-radial out to 20 (r_min unspecified upstream -> 0.05); l ~ N(-4, 0.5^2)."""
    rng = np.random.default_rng(seed)
    d = _unit(rng, n)
    r = np.exp(rng.uniform(np.log(r_min), np.log(20.0), n).astype(np.float32))
    centers = d * r[:, None]
    quats = _quats(rng, n)
    ls = -4.0 + 0.5 * rng.standard_normal((n, 2), dtype=np.float32)
    ks = 0.5 * rng.standard_normal((n, 2), dtype=np.float32)
    raw_scales, raw_signs = _scales_from(ls[:, 0], ls[:, 1], ks[:, 0], ks[:, 1])
    logit = rng.standard_normal(n, dtype=np.float32)
    sh = _sh(rng, n, 3)
    e = _unit(rng, views)
    e[:, 2] = np.abs(e[:, 2])
    cams = [pinhole(width, height, 5.0 * v) for v in e]
    ups = _upstream(rng, cams) if with_upstream else None
    return _pack("c4", centers, quats, raw_scales, raw_signs, logit, sh, cams, ups,
                 {"N": n, "res": [width, height], "sh_deg": 3, "views": views,
                  "r_min": r_min})


def config5(seed=5, n=300_000, res=1024, views=4):
    """C5 degenerate stress: curvature |k| s in [0,5] (10% exactly planar),
    footprints 1..512 px, opacity ~ sigmoid(N(4,0.5^2)), 5% edge-on to view 0."""
    rng = np.random.default_rng(seed)
    centers = 0.3 * rng.standard_normal((n, 3), dtype=np.float32).astype(np.float64)
    quats = _quats(rng, n)
    f = (res / 2.0) / np.tan(np.radians(30.0))
    d_px = np.exp(rng.uniform(0.0, np.log(512.0), n).astype(np.float32))
    l1 = np.log(d_px * 3.0 / (6.0 * f))
    l2 = l1 + 0.2 * rng.standard_normal(n, dtype=np.float32)
    mag = rng.uniform(0, 5, (n, 2)).astype(np.float32)
    sgn = np.where(rng.random((n, 2)) < 0.5, -1.0, 1.0)
    ks = mag * sgn
    planar = rng.random(n) < 0.1
    ks[planar] = 1.0
    raw_scales, raw_signs = _scales_from(l1, l2, ks[:, 0], ks[:, 1], planar_mask=planar)
    logit = 4.0 + 0.5 * rng.standard_normal(n, dtype=np.float32)
    sh = _sh(rng, n, 3)
    eyes = 3.0 * _unit(rng, views)
    cams = [pinhole(res, res, e) for e in eyes]
    # 5% edge-on w.r.t. view 0: rotate so the local z axis is perpendicular
    # to the ray from eye 0 to the centre
    edge = np.nonzero(rng.random(n) < 0.05)[0]
    for i in edge:
        ray = centers[i] - eyes[0]
        ray /= np.linalg.norm(ray)
        zax = np.cross(ray, _unit(rng, 1)[0])
        zax /= np.linalg.norm(zax)
        xax = ray
        yax = np.cross(zax, xax)
        Rm = np.stack([xax, yax, zax], axis=1)
        quats[i] = _rot_to_quat(Rm)
    ups = _upstream(rng, cams)
    return _pack("c5", centers, quats, raw_scales, raw_signs, logit, sh, cams, ups,
                 {"N": n, "res": [res, res], "sh_deg": 3, "views": views,
                  "planar": int(planar.sum()), "edge_on": int(len(edge))})


def _rot_to_quat(Rm):
    w = np.sqrt(max(0.0, 1.0 + Rm[0, 0] + Rm[1, 1] + Rm[2, 2])) / 2.0
    x = np.sqrt(max(0.0, 1.0 + Rm[0, 0] - Rm[1, 1] - Rm[2, 2])) / 2.0
    y = np.sqrt(max(0.0, 1.0 - Rm[0, 0] + Rm[1, 1] - Rm[2, 2])) / 2.0
    z = np.sqrt(max(0.0, 1.0 - Rm[0, 0] - Rm[1, 1] + Rm[2, 2])) / 2.0
    x = np.copysign(x, Rm[2, 1] - Rm[1, 2])
    y = np.copysign(y, Rm[0, 2] - Rm[2, 0])
    z = np.copysign(z, Rm[1, 0] - Rm[0, 1])
    return np.array([w, x, y, z])


def small_scene(seed, n=12, res=32, sh_deg=1, spread=0.6, z_span=1.5, curved=True,
                opacity=(0.3, 0.9), eye=(0.0, 0.0, 5.0), focal=None, width=None, height=None):
    """Small stacked-primitives scene in the style of the reference's unit
    tests (primitives spread in x/y, stacked in z, camera on +z)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-spread, spread, (n, 3))
    c[:, 2] = np.linspace(-z_span / 2, z_span / 2, n)
    q = 0.15 * rng.standard_normal((n, 4))
    q[:, 0] += 1.0
    rs = np.column_stack([rng.uniform(-0.6, 0.2, n), rng.uniform(-0.6, 0.2, n),
                          rng.uniform(-1.5, -0.7, n)])
    sg = np.column_stack([np.full(n, 3.0), np.full(n, 3.0),
                          rng.uniform(0.5, 1.5, n) * np.where(rng.random(n) < 0.5, -1.0, 1.0)])
    if not curved:
        sg[:, 2] = 0.0
    sh = rng.uniform(-0.1, 0.1, (n, 3, (sh_deg + 1) ** 2))
    sh[:, :, 0] = rng.uniform(0.5, 1.5, (n, 3))
    op = rng.uniform(*opacity, n)
    logit = np.log(op / (1 - op))
    focal = focal or res * 1.2
    W, H = width or res, height or res             # ragged sizes: partial tiles and blocks
    cam = Camera(fx=focal, fy=focal, cx=W / 2, cy=H / 2, width=W, height=H,
                 world_to_camera=look_at(eye, np.zeros(3)))
    ups = _upstream(rng, [cam], all_six=True)
    return _pack(f"small{seed}", c, q, rs, sg, logit, sh, [cam], ups,
                 {"N": n, "res": [W, H], "sh_deg": sh_deg, "views": 1})


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}
