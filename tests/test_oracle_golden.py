"""Pin the oracle (oracle/qgs_oracle.py + qgs_kernels.c) to the reference.

The golden fixtures were produced by running the reference implementation
(tests/golden/make_golden.py).  The oracle restates the same arithmetic in
the same order, so every output is compared BIT-EXACTLY.
"""

import numpy as np
import pytest

from oracle import qgs_oracle as qo
from tests import golden_io

MAPS = ("color", "color_raw", "alpha", "depth", "depth_sq", "depth_median", "normal",
        "curvature", "distortion", "transmittance", "n_fragments")
GRADS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh", "screen_center")


@pytest.fixture(scope="module", params=golden_io.names())
def case(request):
    gc = golden_io.load(request.param)
    vw = qo.prepare(gc.prims, gc.cam, gc.settings)
    tg = qo.forward(vw)
    kg = qo.kernel_grads(vw, tg, gc.upstream)
    gr = qo.chain(vw, kg)
    return request.param, gc.g, vw, tg, kg, gr


def test_prepare_bit_exact(case):
    name, g, vw, _, _, _ = case
    for k in ("scales", "alphas", "colors", "pix_bbox", "planar", "tile_offsets",
              "tile_prims"):
        assert np.array_equal(getattr(vw, k), g[k]), (name, k)
    assert np.array_equal(vw.keys_unsorted, g["keys_unsorted"]), name
    assert np.array_equal(vw.pair_tiles_unsorted, g["pair_tiles_unsorted"]), name


def test_forward_bit_exact(case):
    name, g, _, tg, _, _ = case
    for k in MAPS:
        assert np.array_equal(tg[k], g[f"map_{k}"]), (name, k)
    assert tg["order_violations"] == int(g["order_violations"]), name


def test_backward_bit_exact(case):
    name, g, _, _, kg, gr = case
    if "kg" in g:
        assert np.array_equal(kg, g["kg"]), name
    for k in GRADS:
        assert np.array_equal(gr[k], g[f"grad_{k}"]), (name, k)


# known answers from the reference's own tests ---------------------------------

def test_arc_length_known_answer():
    # test_geodesic.py:13-16
    assert qo.arc_length(0.5, 1.0) == pytest.approx(1.1477935746, abs=1e-10)
    # series / closed-form switch continuity (test_geodesic.py:38-46)
    a = 1e-3 / 2.0
    assert abs(qo.arc_length(a * (1 - 1e-9), 1.0) - qo.arc_length(a * (1 + 1e-9), 1.0)) < 1e-12


def test_sigma_known_answer():
    # test_geodesic.py:84-99: sigma(2, 1, pi/4)
    c = s = np.sqrt(0.5)
    assert qo.sigma_dir(2.0, 1.0, c, s) == pytest.approx(1.264911, abs=1e-6)


def test_arc_length_grad_fd():
    for a, rho in [(0.3, 0.7), (-1.2, 0.4), (1e-4, 0.5), (2.5, 1.3)]:
        l, da, dr = qo.arc_length_grad(a, rho)
        h = 1e-6
        assert da == pytest.approx((qo.arc_length(a + h, rho) - qo.arc_length(a - h, rho)) / (2 * h), rel=1e-6, abs=1e-9)
        assert dr == pytest.approx((qo.arc_length(a, rho + h) - qo.arc_length(a, rho - h)) / (2 * h), rel=1e-6)


def test_linear_branch_known_answer():
    # test_intersect.py:50-57: vertical ray on z = x^2 + y^2, A = 0 exactly
    hit = qo.fragment_geometry(1.0, 1.0, 1.0, 1.0, 1.0, 1.0, (0.5, 0.0, 2.0), (0.0, 0.0, -1.0))
    assert hit[0] and hit[-1] == 1
    assert hit[1] == pytest.approx(1.75, abs=1e-12)
    assert hit[2] == pytest.approx(0.5, abs=1e-12)


def test_oblique_root_known_answer():
    # test_intersect.py:60-72: z = x^2 in y=0, root 0.874032, hit x 0.618034
    d = np.array([1.0, 0.0, -1.0]) / np.sqrt(2)
    hit = qo.fragment_geometry(1.0, 1.0, 1.0, 1.0, 1.0, 1.0, (0.0, 0.0, 1.0), d)
    assert hit[0] and hit[-1] == 0
    assert hit[1] == pytest.approx(0.874032, abs=1e-6)
    assert hit[2] == pytest.approx(0.618034, abs=1e-6)


def test_misses_known_answer():
    # test_intersect.py:75-83
    assert not qo.fragment_geometry(1, 1, 1, 1, 1, 1, (0, 0, -1.0), (0, 0, -1.0))[0]
    assert not qo.fragment_geometry(1, 1, 0, 1, 1, 0, (0, 0, 1.0), (1.0, 0, 0), planar=True)[0]


def test_curved_weight_known_answer():
    # test_geodesic.py:129-135: a(0)=1, rho=1 -> l=1.478943, G=0.334996
    hit = qo.fragment_geometry(1.0, 1.0, 1.0, 1.0, 1.0, 1.0, (1.0, 0.0, 5.0), (0.0, 0.0, -1.0))
    assert hit[0]
    assert hit[8] == pytest.approx(1.478943, abs=1e-6)
    assert hit[10] == pytest.approx(0.334996, abs=1e-6)


def test_planar_disk_known_answer():
    # test_rasterizer_forward.py:37-60: fronto-parallel opaque disk
    from types import SimpleNamespace
    from paper_2411_16392_b200.cameras import Camera, look_at
    prims = SimpleNamespace(
        centers=np.zeros((1, 3)), quats=np.array([[1.0, 0, 0, 0]]),
        raw_scales=np.log(np.array([[4.0, 4.0, 1e-9]])),
        raw_signs=np.array([[15.0, 15.0, 15.0]]),
        raw_opacity=np.array([np.log(0.95 / 0.05)]),
        sh=((np.array([0.8, 0.4, 0.2]) - 0.5) / 0.28209479177387814).reshape(1, 3, 1))
    cam = Camera(fx=40.0, fy=40.0, cx=8, cy=8, width=16, height=16,
                 world_to_camera=look_at((0, 0, 5.0), (0, 0, 0)))
    tg, vw = qo.render(prims, cam)
    assert vw.planar[0] == 1
    o, d = cam.ray_world(8, 8)
    t_plane = -o[2] / d[2]
    assert tg["depth_median"][8, 8] == pytest.approx(t_plane, rel=1e-9)
    r2 = np.sum((o + t_plane * d)[:2] ** 2)
    assert tg["alpha"][8, 8] == pytest.approx(0.95 * np.exp(-r2 / 32.0), rel=1e-9)
    assert np.allclose(tg["normal"][8, 8] / tg["alpha"][8, 8], [0, 0, -1], atol=1e-9)
