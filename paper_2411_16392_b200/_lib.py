"""ctypes binding of libqgs_b200.so (include/qgs_b200.h).

The library is built in-tree by paper_2411_16392_b200/build.py.  There is no
CPU fallback: if the shared object is missing or fails to load, importing
the rasterizer raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# QGS_LIB_VARIANT=debug: the bounds-checking build (tests/test_debug_checks.py)
LIB_PATH = os.path.join(_HERE, "lib", "libqgs_b200_debug.so"
                        if os.environ.get("QGS_LIB_VARIANT") == "debug" else "libqgs_b200.so")

KG_STRIDE = 16
AUX_PLANES = 12
TILE = 16

vp = ctypes.c_void_p
f64 = ctypes.c_double
i32 = ctypes.c_int32
i64 = ctypes.c_int64


class Camera(ctypes.Structure):
    _fields_ = [("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64),
                ("width", i32), ("height", i32),
                ("R_wc", f64 * 9), ("t_wc", f64 * 3), ("center", f64 * 3)]


class Settings(ctypes.Structure):
    _fields_ = [("background", f64 * 3), ("t_near_clip", f64), ("alpha_floor", f64),
                ("alpha_clamp", f64), ("t_term", f64), ("resort", i32),
                ("euclidean_density", i32), ("no_cull", i32), ("exact_decisions", i32)]


class Params(ctypes.Structure):
    _fields_ = [("centers", vp), ("quats", vp), ("raw_scales", vp), ("raw_signs", vp),
                ("raw_opacity", vp), ("sh", vp), ("P", i32), ("sh_coeffs", i32)]


class Targets(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("color", "color_raw", "alpha", "depth", "depth_sq",
                                  "depth_median", "normal", "curvature", "distortion",
                                  "transmittance", "n_fragments", "violations", "aux",
                                  "counters", "frag_prim", "frag_t", "frag_xy", "frag_page_table",
                                  "frag_page_count", "frag_pool_next")] + \
        [("frag_pool_pages", i32), ("tile_order", vp)]


class Upstream(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("color", "alpha", "depth", "normal", "curvature",
                                  "distortion")]


class Grads(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("centers", "quats", "raw_scales", "raw_signs",
                                  "raw_opacity", "sh", "screen_center")]


class Groups(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity",
                                  "sh")] + [("P", i32), ("sh_coeffs", i32)]


class AdamConfig(ctypes.Structure):
    _fields_ = [("lr", f64 * 6), ("beta1", f64), ("beta2", f64), ("eps", f64), ("t", i64),
                ("freeze", vp * 6)]


class DensifyStats(ctypes.Structure):
    _fields_ = [("grad_accum", vp), ("grad_count", vp), ("center_accum", vp)]


class DensifyConfig(ctypes.Structure):
    _fields_ = [("grad_threshold", f64), ("percent_dense", f64), ("scene_extent", f64),
                ("prune_opacity", f64), ("clone_nudge", f64), ("max_primitives", i64)]


class MvMaps(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("depth", "alpha", "normal", "image")] + \
        [("height", i32), ("width", i32), ("image_channels", i32)]


class MvConfig(ctypes.Structure):
    _fields_ = [("patch_size", i32), ("alpha_thresh", f64), ("min_denom", f64),
                ("ncc_eps", f64), ("full_chain", i32)]


class MvGrads(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("depth", "alpha", "normal")]


class PrepExport(ctypes.Structure):
    _fields_ = [(n, vp) for n in ("R", "ohat", "M", "Nmat", "wv", "lam", "view_dirs",
                                  "view_dist", "clamped", "color_clamped")]


class QGSError(RuntimeError):
    pass


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2411_16392_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    sigs = {
        "qgs_prep_bytes": (ctypes.c_size_t, [i32]),
        "qgs_preprocess": (ctypes.c_int, [P(Params), P(Camera), P(Settings), vp, vp, vp]),
        "qgs_preprocess_geometry": (ctypes.c_int, [P(Params), P(Camera), P(Settings), vp, vp, vp]),
        "qgs_preprocess_color": (ctypes.c_int, [P(Params), P(Camera), vp, vp]),
        "qgs_bin_workspace_bytes": (ctypes.c_size_t, [i32, i64, i32]),
        "qgs_bin": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), i64, vp, ctypes.c_size_t,
                                   vp, vp, vp]),
        "qgs_sorted_keys": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), vp, vp, i64, vp, vp]),
        "qgs_tile_keys_f64": (ctypes.c_int, [i64, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                             P(Camera), P(Settings), vp, vp]),
        "qgs_forward": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), vp, vp, P(Targets), vp]),
        "qgs_backward": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), vp, vp, P(Targets),
                                        P(Upstream), vp, vp]),
        "qgs_backward_det_workspace_bytes": (ctypes.c_size_t, [i32, i64, P(Camera)]),
        "qgs_backward_deterministic": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), vp, vp,
                                                      P(Targets), P(Upstream), vp, i64, vp,
                                                      ctypes.c_size_t, vp]),
        "qgs_chain": (ctypes.c_int, [P(Params), vp, vp, P(Camera), P(Grads), vp]),
        "qgs_export_prep": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, vp, vp]),
        "qgs_export_prep_geometry": (ctypes.c_int, [P(Params), vp, P(Camera), P(PrepExport), vp]),
        "qgs_pixel_dirs": (ctypes.c_int, [P(Camera), vp, vp]),
        "qgs_trace_pixel": (ctypes.c_int, [vp, i32, P(Camera), P(Settings), vp, vp, i32, i32,
                                           i32] + [vp] * 9),
        "qgs_loss_workspace_bytes": (ctypes.c_size_t, [i32, i32, i32]),
        "qgs_loss_photometric": (ctypes.c_int, [vp, vp, i32, i32, i32, f64, f64, vp, vp, vp,
                                                ctypes.c_size_t, vp]),
        "qgs_loss_distortion": (ctypes.c_int, [vp, i32, i32, f64, vp, vp, vp, ctypes.c_size_t,
                                               vp]),
        "qgs_depth_to_normal": (ctypes.c_int, [vp, vp, P(Camera), f64, vp, vp, vp]),
        "qgs_loss_normal_consistency": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, P(Camera), f64, f64,
                                                       i32, f64, vp, vp, vp, vp, vp,
                                                       ctypes.c_size_t, vp]),
        "qgs_adam_step": (ctypes.c_int, [P(Groups), P(Grads), P(Groups), P(Groups),
                                         P(AdamConfig), P(DensifyStats), vp, vp]),
        "qgs_densify_workspace_bytes": (ctypes.c_size_t, [i32]),
        "qgs_densify_plan": (ctypes.c_int, [P(Params), P(DensifyStats), P(DensifyConfig), vp,
                                            ctypes.c_size_t, vp, vp]),
        "qgs_densify_apply": (ctypes.c_int, [P(Params), P(Params), P(Params), P(DensifyStats),
                                             P(DensifyConfig), vp, P(Groups), P(Groups),
                                             P(Groups), vp]),
        "qgs_reset_opacity": (ctypes.c_int, [P(Groups), P(Groups), P(Groups), f64, vp]),
        "qgs_multiview_workspace_bytes": (ctypes.c_size_t, [i32, i32, i32, i32]),
        "qgs_multiview_loss": (ctypes.c_int, [P(MvMaps), P(Camera), P(MvMaps), P(Camera),
                                              P(MvConfig), f64, P(MvGrads), P(MvGrads), vp, vp,
                                              ctypes.c_size_t, vp]),
        "qgs_diag_counters": (ctypes.c_int, [vp, i32]),
        "qgs_last_error": (ctypes.c_char_p, []),
        "qgs_version": (ctypes.c_int, []),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTS = ("qgs_prep_bytes", "qgs_preprocess", "qgs_preprocess_geometry", "qgs_preprocess_color",
           "qgs_bin_workspace_bytes", "qgs_bin",
           "qgs_sorted_keys", "qgs_tile_keys_f64", "qgs_forward", "qgs_backward", "qgs_backward_det_workspace_bytes",
           "qgs_backward_deterministic", "qgs_chain",
           "qgs_export_prep", "qgs_export_prep_geometry", "qgs_pixel_dirs", "qgs_trace_pixel", "qgs_loss_workspace_bytes",
           "qgs_loss_photometric", "qgs_loss_distortion", "qgs_depth_to_normal",
           "qgs_loss_normal_consistency", "qgs_adam_step", "qgs_densify_workspace_bytes",
           "qgs_densify_plan", "qgs_densify_apply", "qgs_reset_opacity",
           "qgs_multiview_workspace_bytes", "qgs_multiview_loss", "qgs_diag_counters", "qgs_last_error",
           "qgs_version")


def check(rc, what):
    if rc != 0:
        msg = load().qgs_last_error().decode(errors="replace")
        raise QGSError(f"{what} failed ({rc}): {msg}")
