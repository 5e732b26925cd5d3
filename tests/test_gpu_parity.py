"""GPU parity: the sm_100a path vs the reference (golden fixtures made by the
reference itself) and vs the float64 oracle on the same seeded inputs.

Integer outputs (screen boxes, tile ranges, sorted primitive lists) are
compared bit-exactly; sort keys are bit-exact at unit level (the key kernel
fed the oracle's float64 prepared arrays).  Images and gradients use the
BASELINE tolerances (max-abs 1e-4; 1e-3 rel / 1e-5 abs), see tests/parity.py.
"""

import numpy as np
import pytest
import torch

from tests import golden_io, parity

pytestmark = pytest.mark.gpu

SMALL = [n for n in golden_io.names() if n.startswith("s_")]
SCENES = golden_io.names()


@pytest.fixture(scope="module")
def rz(cuda_device):
    from paper_2411_16392_b200 import rasterizer
    return rasterizer


def _settings(rz, gc):
    s = gc.settings
    return rz.RenderSettings(background=np.asarray(s.background), resort=s.resort,
                             euclidean_density=s.euclidean_density)


def _run(rz, gc):
    st = _settings(rz, gc)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    gr = rz.backward(prep, tg, gc.upstream)
    torch.cuda.synchronize()
    return prep, tg, gr


@pytest.mark.parametrize("name", SCENES)
def test_binning_bit_exact(rz, name):
    gc = golden_io.load(name)
    g = gc.g
    prep = rz.prepare(gc.prims, gc.cam, _settings(rz, gc))
    assert np.array_equal(prep.pix_bbox.cpu().numpy().astype(np.int64), g["pix_bbox"])
    assert np.array_equal(prep.tile_offsets.cpu().numpy().astype(np.int64), g["tile_offsets"])
    assert np.array_equal(prep.tile_prims.cpu().numpy().astype(np.int64), g["tile_prims"])
    assert np.array_equal(prep.planar.cpu().numpy(), g["planar"])


@pytest.mark.parametrize("name", SCENES)
def test_sort_keys_unit_bit_exact(rz, name):
    """qgs_tile_keys_f64 fed the oracle's float64 prepared arrays reproduces
    tile_sort_depths bit for bit."""
    from oracle import qgs_oracle as qo
    from paper_2411_16392_b200 import _lib
    gc = golden_io.load(name)
    vw = qo.prepare(gc.prims, gc.cam, gc.settings)
    dev = torch.device("cuda")
    T = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    tiles, prims = T(vw.pair_tiles_unsorted, torch.int64), T(vw.pair_prims_unsorted, torch.int64)
    args = [T(vw.ohat), T(vw.M), T(vw.wv), T(vw.scales), T(vw.planar, torch.uint8),
            T(gc.g["vert_u"]), T(gc.g["vert_v"]), T(vw.view_dist)]
    n = len(vw.keys_unsorted)
    keys = torch.empty((max(n, 1),), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().qgs_tile_keys_f64(
        n, tiles.data_ptr(), prims.data_ptr(), vw.tiles_x, *(a.data_ptr() for a in args),
        rz._cam_struct(gc.cam), rz._settings_struct(_settings(rz, gc)), keys.data_ptr(),
        rz._stream()), "tile_keys_f64")
    got = keys[:n].cpu().numpy()
    assert np.array_equal(got, vw.keys_unsorted), \
        f"{int((got != vw.keys_unsorted).sum())} of {n} keys differ"


@pytest.mark.parametrize("name", SCENES)
def test_sorted_keys_end_to_end(rz, name):
    """End-to-end keys (GPU fp64 preprocessing) vs the reference's: the
    transcendental activations may differ in the last bit, so report ULPs and
    require that the ORDER (tile_prims, checked above) is unaffected."""
    gc = golden_io.load(name)
    from oracle import qgs_oracle as qo
    vw = qo.prepare(gc.prims, gc.cam, gc.settings)
    prep = rz.prepare(gc.prims, gc.cam, _settings(rz, gc))
    got = prep.sorted_keys().cpu().numpy()
    ulp = np.abs(got.view(np.int64) - vw.keys.view(np.int64))
    rel = np.abs(got - vw.keys) / np.abs(vw.keys)
    exact = float((ulp == 0).mean())
    assert rel.max() <= 1e-9, (f"max key rel diff {rel.max():.2e} ({ulp.max()} ulp), "
                               f"{exact:.1%} bit-identical")


@pytest.mark.parametrize("name", SCENES)
def test_forward_within_tolerance(rz, name):
    gc = golden_io.load(name)
    g = gc.g
    _, tg, _ = _run(rz, gc)
    ref = {k: g[f"map_{k}"] for k in ("color", "alpha", "depth", "normal", "depth_median",
                                       "transmittance", "curvature", "distortion",
                                       "n_fragments")}
    rep = parity.image_report(tg.to_numpy(), ref)
    # the golden scenes have no fp32-vs-fp64 decision flip at all
    assert rep["over_tol_pixels"] == 0, rep
    assert rep["count_flip_pixels"] == 0, rep


@pytest.mark.parametrize("name", SMALL + ["c1"])
def test_backward_within_tolerance(rz, name):
    gc = golden_io.load(name)
    g = gc.g
    _, _, gr = _run(rz, gc)
    ref = {k: g[f"grad_{k}"] for k in parity.GRAD_GROUPS + ("screen_center",)}
    rep = parity.grad_report(gr.to_numpy(), ref)
    assert rep["violations"] == 0 and rep["screen_center"]["violations"] == 0, rep


@pytest.mark.parametrize("name", ["c1", "c2_small", "s_default", "s_resort_off", "s_background"])
def test_backward_deterministic_mode(rz, name):
    """RenderSettings(deterministic=True): bitwise-repeatable gradients
    (pkg/tests/test_rasterizer_gradients.py:217-229) within the reference
    tolerances, through the log and the replay paths alike"""
    import dataclasses
    gc = golden_io.load(name)
    st = dataclasses.replace(_settings(rz, gc), deterministic=True)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    g1 = rz.backward(prep, tg, gc.upstream).to_numpy()
    g2 = rz.backward(prep, tg, gc.upstream).to_numpy()
    tg.frag_prim = tg.frag_t = None                     # replay path
    g3 = rz.backward(prep, tg, gc.upstream).to_numpy()
    for k in parity.GRAD_GROUPS + ("screen_center",):
        assert np.array_equal(g1[k], g2[k]), k
    ref = {k: gc.g[f"grad_{k}"] for k in parity.GRAD_GROUPS + ("screen_center",)}
    for g in (g1, g3):
        rep = parity.grad_report(g, ref)
        assert rep["violations"] == 0 and rep["screen_center"]["violations"] == 0, rep


def test_forward_deterministic(rz):
    gc = golden_io.load("c2_small")
    st = _settings(rz, gc)
    a = rz.forward(rz.prepare(gc.prims, gc.cam, st)).to_numpy()
    b = rz.forward(rz.prepare(gc.prims, gc.cam, st)).to_numpy()
    for k in ("color", "alpha", "depth", "normal", "n_fragments"):
        assert np.array_equal(a[k], b[k]), k


def test_empty_scene(rz):
    gc = golden_io.load("s_default")
    far = gc.prims.select(np.zeros(len(gc.prims), dtype=bool))
    prep = rz.prepare(far, gc.cam)
    assert prep.n_pairs == 0
    tg = rz.forward(prep)
    assert float(tg.alpha.abs().max()) == 0.0
    assert float(tg.transmittance.min()) == 1.0
    gr = rz.backward(prep, tg, gc.upstream)
    assert gr.centers.numel() == 0


@pytest.mark.parametrize("name", ["s_default", "s_resort_off", "c2_small"])
@pytest.mark.parametrize("mode", ["no_log", "pool_exhausted"])
def test_backward_replay_fallback(rz, name, mode):
    """The backward's two paths -- the forward's paged fragment log and the
    replay of the block's candidate stream (taken without a log, or for the
    blocks that found the log's page pool empty) -- give the same kernel
    gradients."""
    gc = golden_io.load(name)
    st = _settings(rz, gc)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    assert tg.frag_prim is not None
    assert int(tg.frag_page_count.min()) >= 0          # every block logged
    kg_log = rz.kernel_grads(prep, tg, gc.upstream)
    if mode == "no_log":
        tg.frag_prim = tg.frag_t = None
    else:
        used = int(tg.frag_pool_next.item())
        if used < 2:
            pytest.skip("scene too shallow")
        try:
            rz._FORCE_POOL_PAGES = used // 2           # about half the blocks overflow
            tg = rz.forward(prep)
        finally:
            rz._FORCE_POOL_PAGES = None
        cnt = tg.frag_page_count.cpu().numpy()
        assert (cnt < 0).any() and (cnt >= 0).any()
    kg_rep = rz.kernel_grads(prep, tg, gc.upstream)
    a, b = kg_log.cpu().numpy().astype(np.float64), kg_rep.cpu().numpy().astype(np.float64)
    scale = np.abs(a).max(axis=0, keepdims=True) + 1e-30
    # the log path re-shades in fp32 from the logged hit point, the replay in
    # float64: they agree to ~1e-5 of each slot's scale (both are within the
    # reference tolerance, see test_backward_within_tolerance)
    assert np.all(np.abs(a - b) <= 1e-4 * scale + 1e-6 * np.abs(a)), \
        float((np.abs(a - b) / scale).max())


def test_fragment_log_pool_is_compact(rz):
    """the log's pages scale with the fragments composited: every logged
    fragment has a slot, and the pages handed out hold at most 2x the
    fragments (a warp's pages follow its deepest pixel)"""
    from paper_2411_16392_b200 import scenes
    sc = scenes.config2(views=1)
    prep = rz.prepare(sc.prims, sc.cams[0])
    tg = rz.forward(prep)
    used = int(tg.frag_pool_next.item())
    nfr = int(tg.n_fragments.sum().item())
    assert int(tg.frag_page_count.min()) >= 0
    assert int(tg.frag_page_count.sum().item()) == used
    warps = tg.frag_page_count.numel()
    assert nfr <= used * 16 * 32 <= 3 * nfr + 16 * 32 * warps


@pytest.mark.parametrize("copies", [5, 40, 300, 700, 8500])
def test_sort_ties_duplicates(rz, copies):
    """Duplicated primitives give identical (f32 and fp64) keys: the sort must
    still equal lexsort((prim, key, tile)), i.e. break ties by primitive id,
    through every path of the tile sort (shared-memory tile, bucket groups of
    a large tile, one bucket larger than shared memory)."""
    from oracle import qgs_oracle as qo
    from paper_2411_16392_b200 import scenes
    from paper_2411_16392_b200.model import PrimitiveSet
    sc = scenes.small_scene(seed=11, n=16, res=48, sh_deg=1)
    p = sc.prims
    idx = np.concatenate([np.arange(len(p)), np.full(copies, 3), np.full(copies // 2, 7)])
    rng = np.random.default_rng(copies)
    idx = idx[rng.permutation(len(idx))]
    dup = PrimitiveSet(*(np.ascontiguousarray(getattr(p, f)[idx]) for f in PrimitiveSet.FIELDS))
    prep = rz.prepare(dup, sc.cams[0])
    vw = qo.prepare(dup.astype(np.float64), sc.cams[0])
    assert np.array_equal(prep.tile_offsets.cpu().numpy().astype(np.int64), vw.tile_offsets)
    assert np.array_equal(prep.tile_prims.cpu().numpy().astype(np.int64), vw.tile_prims)


def _cull_pair(rz, prims, cam, base):
    import dataclasses
    on = dataclasses.replace(base, conic_cull=True)
    off = dataclasses.replace(base, conic_cull=False)
    a = rz.forward(rz.prepare(prims, cam, on)).to_numpy()
    b = rz.forward(rz.prepare(prims, cam, off)).to_numpy()
    for k in ("color", "alpha", "depth", "depth_sq", "depth_median", "normal", "curvature",
              "distortion", "transmittance", "n_fragments"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", SCENES)
def test_conic_cull_is_exact(rz, name):
    """The screen-space conic cull only removes candidates the selection rule
    rejects: every output map is bit-identical with the cull off."""
    gc = golden_io.load(name)
    _cull_pair(rz, gc.prims, gc.cam, _settings(rz, gc))


@pytest.mark.parametrize("cfg", ["c2", "c5"])
def test_conic_cull_is_exact_full_view(rz, cfg):
    from paper_2411_16392_b200 import scenes
    sc = scenes.CONFIGS[cfg]()
    _cull_pair(rz, sc.prims, sc.cams[0], rz.RenderSettings())
    _cull_pair(rz, sc.prims, sc.cams[1], rz.RenderSettings(euclidean_density=True))


@pytest.mark.gpu
def test_tile_schedule_is_a_permutation(cuda_device):
    """raster schedule (tile_order_kernel): every tile exactly once, pair
    counts non-increasing up to the quarter-octave binning"""
    from paper_2411_16392_b200 import rasterizer as rz, scenes
    sc = scenes.CONFIGS["c2"]()
    prep = rz.prepare(rz.DevicePrimitives.from_host(sc.prims), sc.cams[0])
    tg = rz.forward(prep)
    order = tg.tile_order.cpu().numpy()
    n_tiles = prep.tile_offsets.numel() - 1
    assert np.array_equal(np.sort(order), np.arange(n_tiles))
    cnt = np.diff(prep.tile_offsets.cpu().numpy())[order]
    key = np.floor(4 * np.log2(cnt.astype(np.float64) + 1))
    assert np.all(np.diff(key) <= 1)           # the kernel bins with an fp32 log2
    assert key[0] >= key.max() - 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c3_small", "s_overflow", "s_planar", "s_euclid"])
def test_fp32_decisions_mode(rz, name):
    """settings.exact_decisions=False (selection decisions in fp32 only): the
    same binning and, within the tolerances, the same images and gradients"""
    gc = golden_io.load(name)
    st = rz.RenderSettings(background=np.asarray(gc.settings.background),
                           resort=gc.settings.resort,
                           euclidean_density=gc.settings.euclidean_density, exact_decisions=False)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    gr = rz.backward(prep, tg, gc.upstream)
    g = gc.g
    ref = {k: g[f"map_{k}"] for k in ("color", "alpha", "depth", "normal", "depth_median",
                                       "transmittance", "curvature", "distortion",
                                       "n_fragments")}
    rep = parity.image_report(tg.to_numpy(), ref)
    assert rep["over_tol_same_count"] == 0, rep
    assert rep["count_flip_pixels"] <= max(2, rep["pixels"] // 2000), rep
    ref_g = {k: g[f"grad_{k}"] for k in parity.GRAD_GROUPS + ("screen_center",)}
    gq = parity.grad_report(gr.to_numpy(), ref_g)
    assert gq["violations"] <= max(2, gq["n"] // 10000), gq
    assert np.array_equal(prep.tile_prims.cpu().numpy(), g["tile_prims"])


@pytest.mark.gpu
@pytest.mark.parametrize("size", [(1, 1), (3, 5), (17, 2), (9, 33)])
def test_tiny_and_ragged_images(rz, size):
    """images smaller than a raster block / a tile, against the oracle"""
    from oracle import qgs_oracle as qo
    from paper_2411_16392_b200 import scenes
    W, H = size
    sc = scenes.small_scene(seed=11, n=16, res=8, width=W, height=H)
    cam = sc.cams[0]
    prims64 = sc.prims.astype(np.float64)
    vw = qo.prepare(prims64, cam)
    ref = qo.forward(vw)
    up = {k: np.asarray(v, np.float64) for k, v in sc.upstream[0].items()}
    ref_g = qo.backward(vw, ref, up)
    prep = rz.prepare(sc.prims, cam)
    assert np.array_equal(prep.tile_prims.cpu().numpy(), vw.tile_prims)
    tg = rz.forward(prep)
    rep = parity.image_report(tg.to_numpy(), ref)
    assert rep["over_tol_same_count"] == 0, rep
    gr = rz.backward(prep, tg, sc.upstream[0])
    gq = parity.grad_report(gr.to_numpy(), {k: ref_g[k] for k in parity.GRAD_GROUPS + ("screen_center",)})
    assert gq["violations"] <= 1, gq


@pytest.mark.gpu
def test_sort_order_at_scale(rz):
    """size-independent sort properties at 4.2M primitives on a small image
    (tiles of ~260K pairs: the staged, two-level path with 23 id bits): every
    tile's list is non-decreasing in its exact float64 key with ties by
    primitive id, and each primitive appears in exactly its box's tiles"""
    from paper_2411_16392_b200 import scenes
    n = (1 << 22) + 12345
    sc = scenes.small_scene(seed=21, n=n, res=64, spread=0.9, z_span=2.0)
    prep = rz.prepare(sc.prims, sc.cams[0])
    keys = prep.sorted_keys().cpu().numpy()
    off = prep.tile_offsets.cpu().numpy().astype(np.int64)
    tp = prep.tile_prims.cpu().numpy().astype(np.int64)
    assert off[-1] == prep.n_pairs == len(tp)
    tile = np.repeat(np.arange(len(off) - 1), np.diff(off))
    # lexsort order: (tile, key, prim) strictly increasing along the list
    same_tile = tile[1:] == tile[:-1]
    dk = keys[1:] - keys[:-1]
    ok = ~same_tile | (dk > 0) | ((dk == 0) & (tp[1:] > tp[:-1]))
    assert ok.all(), int((~ok).sum())
    # membership: each primitive's pair count equals its tile-box area
    counts = np.bincount(tp, minlength=n)
    bb = prep.pix_bbox.cpu().numpy().astype(np.int64)
    live = bb[:, 0] <= bb[:, 1]
    area = np.where(live, (bb[:, 1] // 16 - bb[:, 0] // 16 + 1) * (bb[:, 3] // 16 - bb[:, 2] // 16 + 1), 0)
    assert np.array_equal(counts, area)
    assert np.diff(off).max() > 100_000


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2_small", "s_planar", "s_sh3", "s_euclid"])
def test_prepared_view_fields(rz, name):
    """Every PreparedView field of the reference (rasterizer.py:33-58) is
    exported by the drop-in; float fields agree with the float64 oracle's
    (numpy ops of the reference) to 1e-12, flags and pixel rays exactly."""
    from oracle import qgs_oracle as qo
    gc = golden_io.load(name)
    prep = rz.prepare(gc.prims, gc.cam, _settings(rz, gc))
    vw = qo.prepare(gc.prims, gc.cam, gc.settings)
    P = len(gc.prims)
    for f in ("R", "ohat", "M", "Nmat", "wv", "lam", "view_dirs", "view_dist", "scales",
              "alphas", "colors"):
        got = getattr(prep, f).cpu().numpy()
        ref = np.asarray(getattr(vw, f), np.float64).reshape(got.shape)
        assert got.shape[0] == P, f
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-14), (f, float(np.abs(got - ref).max()))
    assert np.array_equal(prep.clamped.cpu().numpy(), np.asarray(vw.clamped, bool))
    assert np.array_equal(prep.color_clamped.cpu().numpy(), np.asarray(vw.color_clamped, bool))
    assert np.array_equal(prep.dirs.cpu().numpy(), vw.dirs)
    assert np.array_equal(prep.planar.cpu().numpy(), g_planar(vw))
    assert prep.tiles_x == vw.tiles_x and prep.tiles_y == vw.tiles_y


def g_planar(vw):
    return np.asarray(vw.planar, np.uint8)
