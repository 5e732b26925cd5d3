"""CPU-side checks of the C ABI: the in-tree library loads and exports every
entry point include/qgs_b200.h declares (no device calls)."""

import os
import re

from paper_2411_16392_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "qgs_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qgs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for n in ("qgs_preprocess", "qgs_bin", "qgs_forward", "qgs_backward", "qgs_chain"):
        assert n in names


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for n in declared():
        assert hasattr(L, n), n
    assert sorted(_lib.EXPORTS) == declared()


def test_host_only_queries():
    L = _lib.load()
    assert L.qgs_version() >= 1
    assert L.qgs_prep_bytes(1000) >= 1000 * (256 + 128 + 16 + 4 + 8)
    assert L.qgs_bin_workspace_bytes(10, 1000, 64) >= 16 * 1000
    assert isinstance(L.qgs_last_error(), bytes)


def _cam(W=64, H=48, fx=50.0):
    c = _lib.Camera()
    c.fx = c.fy = fx
    c.cx, c.cy = W / 2, H / 2
    c.width, c.height = W, H
    c.R_wc[:] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    return c


def test_argument_errors_before_any_device_work():
    """the new entry points validate on the host and fail loudly (QGS_E_ARG =
    -1, QGS_E_CAPACITY = -3) with a message -- no CUDA call is made"""
    import ctypes
    L = _lib.load()
    fake = ctypes.c_void_p(16)              # never dereferenced: validation fails first
    big = L.qgs_loss_workspace_bytes(48, 64, 3)
    assert big > 48 * 64 * 3 * 24
    # photometric: NULL input, bad channel count, lambda out of range, image below the window
    assert L.qgs_loss_photometric(None, fake, 48, 64, 3, 0.2, 1.0, None, fake, fake, big, None) == -1
    assert L.qgs_loss_photometric(fake, fake, 48, 64, 5, 0.2, 1.0, None, fake, fake, big, None) == -1
    assert L.qgs_loss_photometric(fake, fake, 48, 64, 3, 1.5, 1.0, None, fake, fake, big, None) == -1
    assert L.qgs_loss_photometric(fake, fake, 10, 64, 3, 0.2, 1.0, None, fake, fake, big, None) == -1
    assert b"SSIM window" in L.qgs_last_error()
    assert L.qgs_loss_photometric(fake, fake, 48, 64, 3, 0.2, 1.0, None, fake, fake, 16, None) == -3
    # distortion / normals / consistency
    assert L.qgs_loss_distortion(None, 48, 64, 1.0, None, fake, fake, big, None) == -1
    assert L.qgs_depth_to_normal(fake, fake, None, 0.5, fake, fake, None) == -1
    bad = _cam(fx=-1.0)
    assert L.qgs_depth_to_normal(fake, fake, bad, 0.5, fake, fake, None) == -1
    assert b"focal" in L.qgs_last_error()
    cam = _cam()
    assert L.qgs_loss_normal_consistency(fake, fake, None, fake, None, None, cam, 0.5, 1e-6, 1,
                                         1.0, None, None, None, fake, fake, big, None) == -1
    assert L.qgs_loss_normal_consistency(fake, fake, fake, None, None, None, cam, 0.5, 1e-6, 1,
                                         1.0, None, None, None, fake, fake, big, None) == -1
    # optimizer / densification
    g = _lib.Groups()
    g.P, g.sh_coeffs = 10, 5                 # not (deg+1)^2
    cfg = _lib.AdamConfig()
    cfg.t = 1
    assert L.qgs_adam_step(g, _lib.Grads(), g, g, cfg, None, fake, None) == -1
    g.sh_coeffs = 4
    cfg.t = 0
    assert L.qgs_adam_step(g, _lib.Grads(), g, g, cfg, None, fake, None) == -1
    assert L.qgs_densify_workspace_bytes(1000) > 1000 * (1 + 8 + 12 + 24)
    pp = _lib.Params()
    pp.P, pp.sh_coeffs = 1000, 16
    assert L.qgs_densify_plan(pp, _lib.DensifyStats(), _lib.DensifyConfig(), fake, 8, fake,
                              None) == -3
    # multiview: even patch, oversized patch, missing maps
    m = _lib.MvMaps()
    for f in ("depth", "alpha", "normal", "image"):
        setattr(m, f, 16)
    m.height, m.width, m.image_channels = 48, 64, 3
    mc = _lib.MvConfig()
    mc.patch_size = 6
    ws = L.qgs_multiview_workspace_bytes(48, 64, 48, 64)
    assert L.qgs_multiview_loss(m, cam, m, cam, mc, 1.0, None, None, fake, fake, ws, None) == -1
    mc.patch_size = 15
    assert L.qgs_multiview_loss(m, cam, m, cam, mc, 1.0, None, None, fake, fake, ws, None) == -1
    mc.patch_size = 7
    assert L.qgs_multiview_loss(m, cam, m, cam, mc, 1.0, None, None, fake, fake, 8, None) == -3
    m.image = None
    assert L.qgs_multiview_loss(m, cam, m, cam, mc, 1.0, None, None, fake, fake, ws, None) == -1
