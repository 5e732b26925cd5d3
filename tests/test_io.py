"""On-disk formats: primitive PLY (model.py:193-249),
QGSFMAP1 float maps and PNG (io_maps.py), point PLY (train.py:77-118).

The fixtures under tests/golden/io/ were written and read back by the
reference itself (tests/golden/make_io_golden.py): our readers must return
exactly what the reference read, and our writers must reproduce the
reference's files byte for byte.
"""

import os
import shutil

import numpy as np
import pytest

from paper_2411_16392_b200 import io as qio
from paper_2411_16392_b200.model import ParameterError, PrimitiveSet

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


@pytest.fixture(scope="module")
def parsed():
    return dict(np.load(os.path.join(DIR, "parsed.npz")))


def raw(name):
    with open(os.path.join(DIR, name), "rb") as f:
        return f.read()


def test_ply_roundtrip_byte_exact(parsed, tmp_path):
    ps = qio.load_ply(os.path.join(DIR, "prims.ply"))
    for f in PrimitiveSet.FIELDS:
        np.testing.assert_array_equal(getattr(ps, f), parsed[f"ply_{f}"])
        assert getattr(ps, f).dtype == np.float64
    assert ps.sh_degree == 2
    out = tmp_path / "p.ply"
    qio.save_ply(out, ps)
    assert out.read_bytes() == raw("prims.ply")


def test_ply_errors(tmp_path):
    src = raw("prims.ply")
    cases = {
        "magic": b"plx" + src[3:],
        "ascii": src.replace(b"binary_little_endian", b"ascii", 1),
        "float": src.replace(b"property double x", b"property float x", 1),
        "layout": src.replace(b"property double quat_w", b"property double quat_q", 1),
        "truncated": src[:-8],
        "header": src[:40],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.ply"
        p.write_bytes(data)
        with pytest.raises(ParameterError):
            qio.load_ply(p)
    # an sh count that is not 3 (deg+1)^2: drop the last sh property
    head, body = src.split(b"end_header\n", 1)
    lines = head.split(b"\n")
    lines = [ln for ln in lines if ln != b"property double sh_26"]
    p = tmp_path / "sh.ply"
    p.write_bytes(b"\n".join(lines) + b"end_header\n" + body)
    with pytest.raises(ParameterError):
        qio.load_ply(p)


def test_f32_maps(parsed, tmp_path):
    for name in ("depth", "normal"):
        got = qio.load_f32(os.path.join(DIR, f"{name}.f32"))
        np.testing.assert_array_equal(got, parsed[f"f32_{name}"])
        out = tmp_path / f"{name}.f32"
        qio.save_f32(out, parsed[f"f32_{name}_in"])
        assert out.read_bytes() == raw(f"{name}.f32")
    bad = tmp_path / "bad.f32"
    bad.write_bytes(b"QGSFMAP0" + raw("depth.f32")[8:])
    with pytest.raises(ValueError):
        qio.load_f32(bad)
    bad.write_bytes(raw("depth.f32")[:-4])
    with pytest.raises(ValueError):
        qio.load_f32(bad)
    with pytest.raises(ValueError):
        qio.save_f32(tmp_path / "x.f32", np.zeros(5))


def test_png(parsed, tmp_path):
    for name in ("image", "gray"):
        np.testing.assert_array_equal(qio.load_png(os.path.join(DIR, f"{name}.png")),
                                      parsed[f"png_{name}"])
        out = tmp_path / f"{name}.png"
        qio.save_png(out, parsed[f"png_{name}_in"])
        np.testing.assert_array_equal(qio.load_png(out), parsed[f"png_{name}"])


def test_points_ply(parsed, tmp_path):
    p, c = qio.load_points_ply(os.path.join(DIR, "points_bin.ply"))
    np.testing.assert_array_equal(p, parsed["pts_bin"])
    np.testing.assert_array_equal(c, parsed["pts_bin_colors"])
    p, c = qio.load_points_ply(os.path.join(DIR, "points_ascii.ply"))
    np.testing.assert_array_equal(p, parsed["pts_ascii"])
    assert c is None
    bad = tmp_path / "b.ply"
    bad.write_bytes(raw("points_ascii.ply").replace(b"ascii", b"binary_big_endian"))
    with pytest.raises(ValueError):
        qio.load_points_ply(bad)


@pytest.mark.gpu
def test_ply_device_roundtrip(parsed, tmp_path, cuda_device):
    dp = qio.load_ply_device(os.path.join(DIR, "prims.ply"))
    for f in PrimitiveSet.FIELDS:
        t = getattr(dp, f)
        assert t.is_cuda and str(t.dtype) == "torch.float32"
        np.testing.assert_array_equal(t.cpu().numpy(), parsed[f"ply_{f}"].astype(np.float32))
    out = tmp_path / "d.ply"
    qio.save_ply(out, dp)                           # fp32 values written as doubles
    back = qio.load_ply(out)
    for f in PrimitiveSet.FIELDS:
        np.testing.assert_array_equal(getattr(back, f), parsed[f"ply_{f}"].astype(np.float32))
    shutil.rmtree(tmp_path, ignore_errors=True)
