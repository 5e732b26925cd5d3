"""Drop-in for qgsplat.rasterizer on B200 (sm_100a).

Same module-level API as /root/reference/pkg/src/qgsplat/rasterizer.py:
``RenderSettings`` (:22), ``PreparedView`` (:33), ``RenderTargets`` (:61),
``GradientBuffer`` (:77, with zeros / iadd / finite), ``zero_upstream``
(:111), ``prepare`` (:123), ``forward`` (:198), ``backward`` (:230) and
``render`` (:337), with the same argument and return signatures.  Inputs may
be the reference's own numpy PrimitiveSet / Camera objects; outputs are
CUDA tensors (fp32 maps, int32 counts) with ``to_numpy()`` helpers.

Every stage runs in libqgs_b200.so (include/qgs_b200.h) on the current torch
CUDA stream; the only host synchronisation per view is the read of the
(tile, primitive) pair count that sizes the sort buffers.
"""

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .model import ParameterError, PrimitiveSet

T_NEAR_CLIP = 0.01   # intersect.py:22
TILE = 16            # bounds.py:19
# Fragment log kept by the forward for the backward: 20 B per logged
# fragment (prim, fp64 depth, fp32 local hit point) in a pool of pages (16
# slots x the 32 pixels of a raster warp) that warps take as their deepest
# pixel grows (include/qgs_b200.h, qgs_targets).  The pool is sized from the
# pages the previous forward of the same image size used (x FRAG_POOL_SLACK),
# starting from FRAG_POOL_SLOTS_PER_PX; a block that finds the pool empty is
# replayed by the backward with the full candidate test instead.
FRAG_PAGE = 16
FRAG_MAX_PAGES = 32
FRAG_POOL_SLOTS_PER_PX = 96
FRAG_POOL_SLACK = 1.15
_pool_hint = {}          # (device, H, W) -> (pinned int32 of pages used, event)
_FORCE_POOL_PAGES = None


@dataclass
class RenderSettings:
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    t_near_clip: float = T_NEAR_CLIP
    alpha_floor: float = 1.0 / 255.0
    alpha_clamp: float = 0.999
    t_term: float = 1e-4
    resort: bool = True
    euclidean_density: bool = False
    # extension (not in the reference): False disables the forward's
    # screen-space conic cull; outputs are identical either way
    conic_cull: bool = True
    # extension: True (the default) re-makes in float64 every selection /
    # alpha-floor decision whose fp32 margin lies in its rounding band, so the
    # accepted set is the reference's float64 one at full scale; False keeps
    # the fp32 decisions (faster, a few acceptance flips per million pixels)
    exact_decisions: bool = True
    # extension: True makes the backward bitwise repeatable like the
    # reference's serial merge (raster_kernels.py:673-681): fragments' slots
    # go to rows fixed by the forward and are summed per primitive in row
    # order in fp64 (qgs_backward_deterministic) instead of fp32 atomics
    deterministic: bool = False


# ----------------------------------------------------------------- helpers

def _stream():
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def ctypes_ptr(x):
    import ctypes
    return ctypes.c_void_p(x)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _cam_struct(cam):
    w2c = np.asarray(cam.world_to_camera, dtype=np.float64)
    R, t = w2c[:3, :3], w2c[:3, 3]
    center = -R.T @ t            # cameras.py:48-51
    c = _lib.Camera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    c.R_wc[:] = [float(v) for v in R.ravel()]
    c.t_wc[:] = [float(v) for v in t]
    c.center[:] = [float(v) for v in center]
    return c


def _settings_struct(st):
    s = _lib.Settings()
    s.background[:] = [float(v) for v in np.asarray(st.background, dtype=np.float64).ravel()[:3]]
    s.t_near_clip, s.alpha_floor = float(st.t_near_clip), float(st.alpha_floor)
    s.alpha_clamp, s.t_term = float(st.alpha_clamp), float(st.t_term)
    s.resort, s.euclidean_density = int(bool(st.resort)), int(bool(st.euclidean_density))
    s.no_cull = int(not getattr(st, "conic_cull", True))
    s.exact_decisions = int(bool(getattr(st, "exact_decisions", True)))
    return s


class DevicePrimitives:
    """Raw primitive parameters resident on the GPU as contiguous fp32."""

    FIELDS = PrimitiveSet.FIELDS

    def __init__(self, centers, quats, raw_scales, raw_signs, raw_opacity, sh, sh_ready=None):
        self.centers, self.quats = centers, quats
        self.raw_scales, self.raw_signs = raw_scales, raw_signs
        self.raw_opacity, self.sh = raw_opacity, sh
        # event after the SH coefficients' upload on a copy stream (from_host
        # with sh_stream), or None: prepare() bins a view before it is done
        self.sh_ready = sh_ready

    @staticmethod
    def from_host(prims, device=None, non_blocking=False, sh_stream=None):
        """Upload to the device.  sh_stream (with pinned host tensors and
        non_blocking): the SH coefficients go over on that stream instead,
        and prepare() runs the view's geometry and binning while they are on
        their way (qgs_preprocess_geometry / qgs_preprocess_color)."""
        if isinstance(prims, DevicePrimitives):
            return prims
        device = device or torch.device("cuda", torch.cuda.current_device())

        def up(a):
            if isinstance(a, torch.Tensor):
                t = a.to(device=device, dtype=torch.float32, non_blocking=non_blocking)
            else:
                t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))
                t = t.to(device=device, non_blocking=non_blocking)
            return t.contiguous()

        split = sh_stream is not None and non_blocking
        out = [up(getattr(prims, f)) for f in PrimitiveSet.FIELDS if not (split and f == "sh")]
        ev = None
        if split:
            main = torch.cuda.current_stream(device)
            sh_stream.wait_stream(main)          # the previous user of the buffers is done
            with torch.cuda.stream(sh_stream):
                sh = up(prims.sh)
                ev = torch.cuda.Event()
                ev.record(sh_stream)
            sh.record_stream(main)
            out.append(sh)
        return DevicePrimitives(*out, sh_ready=ev)

    def __len__(self):
        return self.centers.shape[0]

    @property
    def sh_coeffs(self):
        return self.sh.shape[2]

    def params_struct(self):
        p = _lib.Params()
        p.centers, p.quats = _ptr(self.centers), _ptr(self.quats)
        p.raw_scales, p.raw_signs = _ptr(self.raw_scales), _ptr(self.raw_signs)
        p.raw_opacity, p.sh = _ptr(self.raw_opacity), _ptr(self.sh)
        p.P, p.sh_coeffs = len(self), self.sh_coeffs
        return p


def _validate_host(prims):
    """model.py:37-38 for host (numpy) inputs: non-finite raw scales / signs
    raise ParameterError before anything is uploaded.  Device inputs are
    checked by the preprocess kernel (a negative pair count, no extra sync)."""
    for f in ("raw_scales", "raw_signs"):
        a = getattr(prims, f)
        if not isinstance(a, torch.Tensor) and not np.isfinite(np.asarray(a)).all():
            raise ParameterError("non-finite raw scale/sign")


# ------------------------------------------------------------------- types

@dataclass
class PreparedView:
    cam: object
    settings: RenderSettings
    prims: object                 # the caller's PrimitiveSet (reference kept, not copied)
    dev: DevicePrimitives
    prep: torch.Tensor            # opaque per-primitive device state (qgs_prep_bytes)
    n_pairs: int
    tile_offsets: torch.Tensor    # int32 (tiles_x*tiles_y + 1,)
    tile_prims: torch.Tensor      # int32 (n_pairs,)
    tiles_x: int
    tiles_y: int
    _cam_c: object = None
    _st_c: object = None

    def _export(self):
        P = len(self.dev)
        dev = self.prep.device
        sc = torch.empty((P, 3), dtype=torch.float64, device=dev)
        al = torch.empty((P,), dtype=torch.float64, device=dev)
        co = torch.empty((P, 3), dtype=torch.float64, device=dev)
        bb = torch.empty((P, 4), dtype=torch.int32, device=dev)
        pl = torch.empty((P,), dtype=torch.uint8, device=dev)
        _lib.check(_lib.load().qgs_export_prep(_ptr(self.prep), P, _ptr(sc), _ptr(al), _ptr(co),
                                               _ptr(bb), _ptr(pl), _stream()), "export_prep")
        return sc, al, co, bb, pl

    @property
    def scales(self):
        return self._export()[0]

    @property
    def alphas(self):
        return self._export()[1]

    @property
    def colors(self):
        return self._export()[2]

    @property
    def pix_bbox(self):
        return self._export()[3]

    @property
    def planar(self):
        return self._export()[4]

    # the rest of the reference's PreparedView (rasterizer.py:33-58), each
    # exported on demand from the device state (qgs_export_prep_geometry)
    _GEOM = {"R": ((3, 3), torch.float64), "ohat": ((3,), torch.float64),
             "M": ((3, 3), torch.float64), "Nmat": ((3, 3), torch.float64),
             "wv": ((3,), torch.float64), "lam": ((2,), torch.float64),
             "view_dirs": ((3,), torch.float64), "view_dist": ((), torch.float64),
             "clamped": ((3,), torch.bool), "color_clamped": ((3,), torch.bool)}

    def _geometry(self, name):
        shape, dt = self._GEOM[name]
        P = len(self.dev)
        t = torch.empty((P,) + shape, dtype=torch.uint8 if dt == torch.bool else dt,
                        device=self.prep.device)
        ex = _lib.PrepExport()
        setattr(ex, name, _ptr(t))
        _lib.check(_lib.load().qgs_export_prep_geometry(self.dev.params_struct(), _ptr(self.prep),
                                                        self._cam_c, ex, _stream()),
                   "export_prep_geometry")
        return t.bool() if dt == torch.bool else t

    R = property(lambda self: self._geometry("R"))
    ohat = property(lambda self: self._geometry("ohat"))
    M = property(lambda self: self._geometry("M"))
    Nmat = property(lambda self: self._geometry("Nmat"))
    wv = property(lambda self: self._geometry("wv"))
    lam = property(lambda self: self._geometry("lam"))
    view_dirs = property(lambda self: self._geometry("view_dirs"))
    view_dist = property(lambda self: self._geometry("view_dist"))
    clamped = property(lambda self: self._geometry("clamped"))
    color_clamped = property(lambda self: self._geometry("color_clamped"))

    @property
    def dirs(self):
        """(H, W, 3) float64 unit camera-frame pixel rays (cameras.py:53-59)"""
        H, W = int(self.cam.height), int(self.cam.width)
        t = torch.empty((H, W, 3), dtype=torch.float64, device=self.prep.device)
        _lib.check(_lib.load().qgs_pixel_dirs(self._cam_c, _ptr(t), _stream()), "pixel_dirs")
        return t

    def trace_pixel(self, u, v, max_frags=4096):
        """Replay pixel (u, v): accepted candidates and emitted fragments."""
        dev = self.prep.device
        i = lambda: torch.zeros((max_frags,), dtype=torch.int32, device=dev)  # noqa: E731
        f = lambda: torch.zeros((max_frags,), dtype=torch.float32, device=dev)  # noqa: E731
        ap, at, aa, ep, et, ea = i(), f(), f(), i(), f(), f()
        eT = torch.zeros((max_frags,), dtype=torch.float64, device=dev)
        cnt = torch.zeros((2,), dtype=torch.int32, device=dev)
        _lib.check(_lib.load().qgs_trace_pixel(
            _ptr(self.prep), len(self.dev), self._cam_c, self._st_c, _ptr(self.tile_offsets),
            _ptr(self.tile_prims), int(u), int(v), max_frags, *(_ptr(x) for x in
                                                                (ap, at, aa, ep, et, ea, eT, cnt)),
            _stream()), "trace_pixel")
        na, ne = (int(x) for x in cnt.cpu())
        na, ne = min(na, max_frags), min(ne, max_frags)
        return ({"prim": ap[:na].cpu().numpy(), "t": at[:na].cpu().numpy(),
                 "abar": aa[:na].cpu().numpy()},
                {"prim": ep[:ne].cpu().numpy(), "t": et[:ne].cpu().numpy(),
                 "abar": ea[:ne].cpu().numpy(), "T": eT[:ne].cpu().numpy()})

    def sorted_keys(self):
        """float64 sort key of every entry of tile_prims (parity/debug)."""
        keys = torch.empty((max(self.n_pairs, 1),), dtype=torch.float64, device=self.prep.device)
        _lib.check(_lib.load().qgs_sorted_keys(
            _ptr(self.prep), len(self.dev), self._cam_c, self._st_c, _ptr(self.tile_offsets),
            _ptr(self.tile_prims), self.n_pairs, _ptr(keys), _stream()), "sorted_keys")
        return keys[: self.n_pairs]


_MAPS = ("color", "color_raw", "alpha", "depth", "depth_sq", "depth_median", "normal",
         "curvature", "distortion", "transmittance", "n_fragments")


@dataclass
class RenderTargets:
    color: torch.Tensor           # blended colour + background, (H, W, 3)
    color_raw: torch.Tensor
    alpha: torch.Tensor
    depth: torch.Tensor           # sum omega_i t_i
    depth_sq: torch.Tensor
    depth_median: torch.Tensor
    normal: torch.Tensor          # camera-frame blended normal
    curvature: torch.Tensor
    distortion: torch.Tensor
    transmittance: torch.Tensor
    n_fragments: torch.Tensor
    violations: torch.Tensor      # per tile (int32)
    aux: torch.Tensor             # (12, H, W) float64 blend sums for the backward
    frag_prim: torch.Tensor = None     # fragment log pool (pages, 16, 32) int32 primitive ids
    frag_t: torch.Tensor = None        # ... float64 depths
    frag_xy: torch.Tensor = None       # ... (pages, 16, 32, 2) fp32 local hit points
    frag_page_table: torch.Tensor = None   # (raster warps, 32) int32 page ids
    frag_page_count: torch.Tensor = None   # (raster warps,) int32, -1 = not logged
    frag_pool_next: torch.Tensor = None    # (1,) int32 pages handed out
    tile_order: torch.Tensor = None    # tiles by descending pair count (raster schedule)

    @property
    def order_violations(self):
        return int(self.violations.sum().item())

    def to_numpy(self):
        d = {k: getattr(self, k).cpu().numpy() for k in _MAPS}
        d["order_violations"] = self.order_violations
        return d


@dataclass
class GradientBuffer:
    centers: torch.Tensor
    quats: torch.Tensor
    raw_scales: torch.Tensor
    raw_signs: torch.Tensor
    raw_opacity: torch.Tensor
    sh: torch.Tensor
    screen_center: torch.Tensor   # ndc-scale projected centre gradient, (P, 2)

    GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")

    @staticmethod
    def zeros(prims, device=None):
        if isinstance(prims, DevicePrimitives):
            device = prims.centers.device
            shp = {f: tuple(getattr(prims, f).shape) for f in DevicePrimitives.FIELDS}
        else:
            device = device or torch.device("cuda", torch.cuda.current_device())
            shp = {f: tuple(np.shape(getattr(prims, f))) for f in PrimitiveSet.FIELDS}
        z = {f: torch.zeros(s, dtype=torch.float32, device=device) for f, s in shp.items()}
        return GradientBuffer(**z, screen_center=torch.zeros((shp["centers"][0], 2),
                                                             dtype=torch.float32, device=device))

    @staticmethod
    def zeros_flat(prims: "DevicePrimitives"):
        """Like zeros(), but the six raw groups are views of ONE flat fp32
        buffer (``.buffer``) so a multi-GPU step all-reduces it in place."""
        device = prims.centers.device
        shp = [tuple(getattr(prims, f).shape) for f in DevicePrimitives.FIELDS]
        sizes = [int(np.prod(s)) for s in shp]
        buf = torch.zeros((sum(sizes),), dtype=torch.float32, device=device)
        views, o = [], 0
        for s, n in zip(shp, sizes):
            views.append(buf[o:o + n].view(s))
            o += n
        gb = GradientBuffer(*views, screen_center=torch.zeros((shp[0][0], 2), dtype=torch.float32,
                                                              device=device))
        gb.buffer = buf
        return gb

    def zero_(self):
        for f in self.GROUPS + ("screen_center",):
            getattr(self, f).zero_()
        return self

    def iadd(self, other):
        for f in self.GROUPS + ("screen_center",):
            getattr(self, f).add_(getattr(other, f))
        return self

    def finite(self):
        return all(bool(torch.isfinite(getattr(self, f)).all()) for f in self.GROUPS)

    def grads_struct(self):
        g = _lib.Grads()
        for f in self.GROUPS + ("screen_center",):
            setattr(g, f, _ptr(getattr(self, f)))
        return g

    def flat(self):
        """The six raw groups packed into one fp32 vector (all-reduce layout)."""
        return torch.cat([getattr(self, f).reshape(-1) for f in self.GROUPS])

    def to_numpy(self):
        return {f: getattr(self, f).cpu().numpy() for f in self.GROUPS + ("screen_center",)}


def zero_upstream(cam, device=None):
    device = device or torch.device("cuda", torch.cuda.current_device())
    H, W = int(cam.height), int(cam.width)
    z = lambda *s: torch.zeros(s, dtype=torch.float32, device=device)  # noqa: E731
    return {"color": z(H, W, 3), "alpha": z(H, W), "depth": z(H, W), "normal": z(H, W, 3),
            "curvature": z(H, W), "distortion": z(H, W)}


# ------------------------------------------------------------------ stages

def prepare(prims, cam, settings: RenderSettings = None, validate=True) -> PreparedView:
    """rasterizer.py:123-195: preprocessing, key duplication and tile sort."""
    settings = settings or RenderSettings()
    L = _lib.load()
    if validate:
        _validate_host(prims)
    dev = DevicePrimitives.from_host(prims)
    device = dev.centers.device
    P = len(dev)
    cam_c, st_c = _cam_struct(cam), _settings_struct(settings)
    tiles_x = (int(cam.width) + TILE - 1) // TILE
    tiles_y = (int(cam.height) + TILE - 1) // TILE
    prep = torch.empty((L.qgs_prep_bytes(P),), dtype=torch.uint8, device=device)
    n_dev = torch.empty((1,), dtype=torch.int64, device=device)
    pp = dev.params_struct()
    # SH coefficients still on their way (DevicePrimitives.from_host with
    # sh_stream): geometry and binning first, the colour after them
    defer = dev.sh_ready is not None and not dev.sh_ready.query()
    if defer:
        _lib.check(L.qgs_preprocess_geometry(pp, cam_c, st_c, _ptr(prep), _ptr(n_dev), _stream()),
                   "qgs_preprocess_geometry")
    else:
        _lib.check(L.qgs_preprocess(pp, cam_c, st_c, _ptr(prep), _ptr(n_dev), _stream()),
                   "qgs_preprocess")
    n_pairs = int(n_dev.item())              # the one host sync per view
    if n_pairs < 0:                          # -k: k primitives with non-finite raw scales/signs
        raise ParameterError(f"non-finite raw scale/sign ({-n_pairs} primitives)")
    n_tiles = tiles_x * tiles_y
    ws_bytes = L.qgs_bin_workspace_bytes(P, n_pairs, n_tiles)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=device)
    tile_offsets = torch.empty((n_tiles + 1,), dtype=torch.int32, device=device)
    tile_prims = torch.empty((max(n_pairs, 1),), dtype=torch.int32, device=device)
    _lib.check(L.qgs_bin(_ptr(prep), P, cam_c, st_c, n_pairs, _ptr(ws), ws_bytes,
                         _ptr(tile_offsets), _ptr(tile_prims), _stream()), "qgs_bin")
    if defer:
        torch.cuda.current_stream(device).wait_event(dev.sh_ready)
        _lib.check(L.qgs_preprocess_color(pp, cam_c, _ptr(prep), _stream()), "qgs_preprocess_color")
    return PreparedView(cam=cam, settings=settings, prims=prims, dev=dev, prep=prep,
                        n_pairs=n_pairs, tile_offsets=tile_offsets,
                        tile_prims=tile_prims[:n_pairs], tiles_x=tiles_x, tiles_y=tiles_y,
                        _cam_c=cam_c, _st_c=st_c)


def _pool_pages(device, H, W, warps):
    """pages for this forward's fragment log: what the last forward of this
    image size used (read from pinned memory, no sync) with some slack, or a
    first guess from the pixel count"""
    if _FORCE_POOL_PAGES is not None:            # tests: force pool exhaustion
        return _FORCE_POOL_PAGES
    guess = (H * W * FRAG_POOL_SLOTS_PER_PX) // (FRAG_PAGE * 32) + warps
    h = _pool_hint.get((device, H, W))
    if h is not None and h[1].query():
        used = int(h[0][0])
        if used > 0:
            return max(int(used * FRAG_POOL_SLACK) + 64, warps)
    return guess


def _alloc_frag_log(tg, t, prep, H, W, device):
    warps = prep.tiles_x * prep.tiles_y * 8
    pages = _pool_pages(device, H, W, warps)
    slots = pages * FRAG_PAGE * 32
    tg.frag_prim = torch.empty((slots,), dtype=torch.int32, device=device)
    tg.frag_t = torch.empty((slots,), dtype=torch.float64, device=device)
    tg.frag_page_table = torch.empty((warps, FRAG_MAX_PAGES), dtype=torch.int32, device=device)
    tg.frag_page_count = torch.empty((warps,), dtype=torch.int32, device=device)
    tg.frag_pool_next = torch.empty((1,), dtype=torch.int32, device=device)   # zeroed by qgs_forward
    t.frag_prim, t.frag_t = _ptr(tg.frag_prim), _ptr(tg.frag_t)
    t.frag_page_table, t.frag_page_count = _ptr(tg.frag_page_table), _ptr(tg.frag_page_count)
    t.frag_pool_next, t.frag_pool_pages = _ptr(tg.frag_pool_next), pages
    if not os.environ.get("QGS_NO_FRAG_XY"):   # diagnostic: float64 re-shading
        tg.frag_xy = torch.empty((slots, 2), dtype=torch.float32, device=device)
        t.frag_xy = _ptr(tg.frag_xy)


def _note_pool_use(tg, device, H, W):
    """copy the pages used to pinned memory (async) for the next forward's sizing"""
    key = (device, H, W)
    h = _pool_hint.get(key)
    if h is None or h[1].query():
        buf = h[0] if h is not None else torch.zeros((1,), dtype=torch.int32).pin_memory()
        buf.copy_(tg.frag_pool_next, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        _pool_hint[key] = (buf, ev)


def forward(prep: PreparedView, keep_aux=True, counters=None, frag_log=True) -> RenderTargets:
    """rasterizer.py:198-227.  `counters` (optional uint64/int64 CUDA tensor of
    5) accumulates [in-box candidates, accepted fragments, composited,
    candidates after the conic cull, candidates passing the coarse test]."""
    cam = prep.cam
    H, W = int(cam.height), int(cam.width)
    device = prep.prep.device
    f32 = lambda *s: torch.empty(s, dtype=torch.float32, device=device)  # noqa: E731
    tg = RenderTargets(
        color=f32(H, W, 3), color_raw=f32(H, W, 3), alpha=f32(H, W), depth=f32(H, W),
        depth_sq=f32(H, W), depth_median=f32(H, W), normal=f32(H, W, 3), curvature=f32(H, W),
        distortion=f32(H, W), transmittance=f32(H, W),
        n_fragments=torch.empty((H, W), dtype=torch.int32, device=device),
        violations=torch.empty((prep.tiles_x * prep.tiles_y,), dtype=torch.int32, device=device),
        aux=torch.empty((_lib.AUX_PLANES, H, W) if keep_aux else (1,), dtype=torch.float64,
                        device=device))
    t = _lib.Targets()
    for k in _MAPS + ("violations",):
        setattr(t, k, _ptr(getattr(tg, k)))
    t.aux = _ptr(tg.aux) if keep_aux else None
    if keep_aux and frag_log:
        _alloc_frag_log(tg, t, prep, H, W, device)
    tg.tile_order = torch.empty((prep.tiles_x * prep.tiles_y,), dtype=torch.int32, device=device)
    t.tile_order = _ptr(tg.tile_order)
    t.counters = _ptr(counters)
    _lib.check(_lib.load().qgs_forward(_ptr(prep.prep), len(prep.dev), prep._cam_c, prep._st_c,
                                       _ptr(prep.tile_offsets), _ptr(prep.tile_prims), t,
                                       _stream()), "qgs_forward")
    if tg.frag_pool_next is not None:
        _note_pool_use(tg, device, H, W)
    return tg


def _up_tensor(a, shape, device):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        t = a.to(device=device, dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(device)
    if tuple(t.shape) != shape:
        raise ValueError(f"upstream shape {tuple(t.shape)} != {shape}")
    return t.contiguous()


def kernel_grads(prep: PreparedView, targets: RenderTargets, upstream, kg=None) -> torch.Tensor:
    """backward_kernel + merge (raster_kernels.py:505-681): (P, 24) fp32 slots,
    accumulated into `kg` when given (it must then be zeroed by the caller)."""
    cam = prep.cam
    H, W = int(cam.height), int(cam.width)
    device = prep.prep.device
    shapes = {"color": (H, W, 3), "alpha": (H, W), "depth": (H, W), "normal": (H, W, 3),
              "curvature": (H, W), "distortion": (H, W)}
    ups = {k: _up_tensor(upstream.get(k), s, device) for k, s in shapes.items()}
    u = _lib.Upstream()
    for k, v in ups.items():
        setattr(u, k, _ptr(v))
    t = _lib.Targets()
    for k in _MAPS + ("violations",):
        setattr(t, k, _ptr(getattr(targets, k)))
    if targets.aux.dim() != 3:
        raise ValueError("backward needs forward(prep, keep_aux=True)")
    t.aux = _ptr(targets.aux)
    t.tile_order = _ptr(targets.tile_order)
    if targets.frag_prim is not None:
        t.frag_prim, t.frag_t = _ptr(targets.frag_prim), _ptr(targets.frag_t)
        t.frag_xy = _ptr(targets.frag_xy)
        t.frag_page_table = _ptr(targets.frag_page_table)
        t.frag_page_count = _ptr(targets.frag_page_count)
    if kg is None:
        kg = torch.zeros((len(prep.dev), _lib.KG_STRIDE), dtype=torch.float32, device=device)
    L = _lib.load()
    if getattr(prep.settings, "deterministic", False):
        n_frags = int(targets.n_fragments.sum().item())      # sizes the row buffer
        nb = L.qgs_backward_det_workspace_bytes(len(prep.dev), n_frags, prep._cam_c)
        ws = torch.empty((nb,), dtype=torch.uint8, device=device)
        _lib.check(L.qgs_backward_deterministic(
            _ptr(prep.prep), len(prep.dev), prep._cam_c, prep._st_c, _ptr(prep.tile_offsets),
            _ptr(prep.tile_prims), t, u, _ptr(kg), n_frags, _ptr(ws), nb, _stream()),
            "qgs_backward_deterministic")
        return kg
    _lib.check(L.qgs_backward(_ptr(prep.prep), len(prep.dev), prep._cam_c, prep._st_c,
                              _ptr(prep.tile_offsets), _ptr(prep.tile_prims), t, u,
                              _ptr(kg), _stream()), "qgs_backward")
    return kg


def chain(prep: PreparedView, kg: torch.Tensor, out: GradientBuffer = None) -> GradientBuffer:
    """_chain_to_raw (rasterizer.py:270-334); accumulates into `out`."""
    out = out if out is not None else GradientBuffer.zeros(prep.dev)
    _lib.check(_lib.load().qgs_chain(prep.dev.params_struct(), _ptr(prep.prep), _ptr(kg),
                                     prep._cam_c, out.grads_struct(), _stream()), "qgs_chain")
    return out


def backward(prep: PreparedView, targets: RenderTargets, upstream,
             out: GradientBuffer = None) -> GradientBuffer:
    """rasterizer.py:230-267.  With `out`, gradients are accumulated into it
    (several views on one device sum before a single all-reduce)."""
    return chain(prep, kernel_grads(prep, targets, upstream), out)


def render(prims, cam, settings=None):
    """Convenience one-shot forward (rasterizer.py:337-340)."""
    prep = prepare(prims, cam, settings)
    return forward(prep), prep
