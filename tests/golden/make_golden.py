"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports qgsplat from /root/reference/pkg/src (numba cache and bytecode
redirected away from the read-only tree), renders a set of seeded scenes
through qgsplat.rasterizer.prepare/forward/backward, and writes one
compressed .npz per scene next to this script.  The fixtures pin the oracle
(tests/test_oracle_golden.py) and, through it, the GPU path.  Nothing at run
time on the GPU box reads /root/reference.
"""

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qgs_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from qgsplat import raster_kernels as rk  # noqa: E402
from qgsplat import rasterizer as rz  # noqa: E402
from qgsplat.cameras import Camera as RefCamera  # noqa: E402
from qgsplat.model import PrimitiveSet as RefPrims  # noqa: E402

from paper_2411_16392_b200 import scenes  # noqa: E402

_captured = {}
_orig_keys = rk.tile_sort_depths
_orig_merge = rk.merge_pair_grads


def _keys_hook(*a):
    out = _orig_keys(*a)
    _captured["keys_unsorted"] = out.copy()
    _captured["pair_tiles_unsorted"] = np.asarray(a[0]).copy()
    _captured["pair_prims_unsorted"] = np.asarray(a[1]).copy()
    _captured["vert_u"] = np.asarray(a[8]).copy()
    _captured["vert_v"] = np.asarray(a[9]).copy()
    return out


def _merge_hook(tile_prims, pair_grad, out):
    _orig_merge(tile_prims, pair_grad, out)
    _captured["kg"] = out.copy()


rk.tile_sort_depths = _keys_hook
rk.merge_pair_grads = _merge_hook


def run(name, prims32, cam, upstream, settings_kw):
    prims = RefPrims(*(np.asarray(getattr(prims32, f), dtype=np.float64)
                       for f in ("centers", "quats", "raw_scales", "raw_signs",
                                 "raw_opacity", "sh")))
    rcam = RefCamera(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                     height=cam.height, world_to_camera=cam.world_to_camera)
    bg = np.asarray(settings_kw.get("background", (0.0, 0.0, 0.0)), dtype=np.float64)
    st = rz.RenderSettings(background=bg, resort=settings_kw.get("resort", True),
                           euclidean_density=settings_kw.get("euclidean_density", False))
    _captured.clear()
    prep = rz.prepare(prims, rcam, st)
    tg = rz.forward(prep)
    up = {k: np.asarray(v, dtype=np.float64) for k, v in (upstream or {}).items()}
    gr = rz.backward(prep, tg, up)
    rec = {
        # inputs
        "centers": prims.centers, "quats": prims.quats, "raw_scales": prims.raw_scales,
        "raw_signs": prims.raw_signs, "raw_opacity": prims.raw_opacity, "sh": prims.sh,
        "cam_intr": np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
        "cam_size": np.array([cam.width, cam.height]),
        "w2c": np.asarray(cam.world_to_camera, dtype=np.float64),
        "background": bg, "resort": np.array(int(st.resort)),
        "euclid": np.array(int(st.euclidean_density)),
        # prepare
        "scales": prep.scales, "alphas": prep.alphas, "colors": prep.colors,
        "pix_bbox": prep.pix_bbox, "tile_offsets": prep.tile_offsets,
        "tile_prims": prep.tile_prims, "planar": prep.planar,
        # forward
        **{f"map_{k}": getattr(tg, k) for k in
           ("color", "color_raw", "alpha", "depth", "depth_sq", "depth_median", "normal",
            "curvature", "distortion", "transmittance", "n_fragments")},
        "order_violations": np.array(tg.order_violations),
        # backward
        **{f"grad_{k}": getattr(gr, k) for k in
           ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh",
            "screen_center")},
    }
    for k, v in _captured.items():
        if k != "kg" or len(prims) <= 64:
            rec[k] = v
    for k, v in up.items():
        rec[f"up_{k}"] = v
    # inputs and upstream are exact float32 values: store them compactly
    for k in ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh",
              *(f"up_{k}" for k in up)):
        v32 = rec[k].astype(np.float32)
        assert np.array_equal(v32.astype(np.float64), rec[k]), k
        rec[k] = v32
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"{name}: P={len(prims)} pairs={len(prep.tile_prims)} "
          f"viol={tg.order_violations} -> {os.path.getsize(path) / 1e3:.0f} kB")


VARIANTS = [
    ("s_default", dict(seed=0), {}),
    ("s_background", dict(seed=1), {"background": (0.1, 0.2, 0.3)}),
    ("s_resort_off", dict(seed=2), {"resort": False}),
    ("s_euclid", dict(seed=3), {"euclidean_density": True}),
    ("s_planar", dict(seed=4, curved=False), {}),
    ("s_overflow", dict(seed=5, n=40, spread=0.4, z_span=0.5, opacity=(0.2, 0.5)), {}),
    ("s_sh3", dict(seed=6, sh_deg=3, n=20), {"background": (0.25, 0.25, 0.25)}),
    ("s_sh2", dict(seed=7, sh_deg=2, n=16, res=24), {}),
    # ragged image: partial tiles and partial 8x4 raster blocks on both axes
    ("s_ragged", dict(seed=8, n=30, res=32, width=37, height=29), {}),
]


def main():
    only = set(sys.argv[1:])           # optional: regenerate just these fixtures
    if only:
        for name, kw, st in VARIANTS:
            if name in only:
                sc = scenes.small_scene(**kw)
                run(name, sc.prims, sc.cams[0], sc.upstream[0], st)
        return
    sc = scenes.config1()
    run("c1", sc.prims, sc.cams[0], sc.upstream[0], {})
    # reduced C2 / C5 shapes (SH3, heavy overlap, buffer overflow, degenerate)
    sc = scenes.config2(seed=12, n=4000, res=128, views=1)
    run("c2_small", sc.prims, sc.cams[0], sc.upstream[0], {})
    sc = scenes.config5(seed=15, n=2500, res=112, views=1)
    run("c5_small", sc.prims, sc.cams[0], sc.upstream[0], {})
    sc = scenes.config3(seed=13, n=5000, width=128, height=96, views=1)
    run("c3_small", sc.prims, sc.cams[0], sc.upstream[0], {})
    # unit-test style scenes with every setting variant
    for name, kw, st in VARIANTS:
        sc = scenes.small_scene(**kw)
        run(name, sc.prims, sc.cams[0], sc.upstream[0], st)


if __name__ == "__main__":
    main()
