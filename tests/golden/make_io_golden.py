"""Generate the file-format fixtures (tests/golden/io/) with the REFERENCE
writers and readers: qgsplat.model.save_ply / load_ply (model.py:193-249),
qgsplat.io_maps save_f32 / load_f32 / save_png / load_png, and
qgsplat.train.load_points_ply on hand-made point files (ascii and binary).

Run in the build container (where /root/reference exists):

    python tests/golden/make_io_golden.py

Writes the files themselves plus parsed.npz (what the reference reads back).
Nothing on the GPU box reads /root/reference.
"""

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "qgs_numba_cache"))
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
sys.path.insert(0, "/root/reference/pkg/src")

from qgsplat import io_maps  # noqa: E402
from qgsplat.model import PrimitiveSet, load_ply, save_ply  # noqa: E402
from qgsplat.train import load_points_ply  # noqa: E402


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(7)
    n = 37
    q = rng.normal(size=(n, 4))
    ps = PrimitiveSet(rng.normal(size=(n, 3)), q / np.linalg.norm(q, axis=1, keepdims=True),
                      rng.normal(-3, 1, (n, 3)), rng.normal(size=(n, 3)), rng.normal(size=n),
                      rng.normal(size=(n, 3, 9)))
    save_ply(os.path.join(OUT, "prims.ply"), ps)
    back = load_ply(os.path.join(OUT, "prims.ply"))
    parsed = {f"ply_{f}": getattr(back, f) for f in PrimitiveSet.__init__.__code__.co_varnames[1:7]}
    depth = rng.uniform(1, 5, (9, 13))
    normal = rng.normal(size=(9, 13, 3))
    io_maps.save_f32(os.path.join(OUT, "depth.f32"), depth)
    io_maps.save_f32(os.path.join(OUT, "normal.f32"), normal)
    parsed["f32_depth"] = io_maps.load_f32(os.path.join(OUT, "depth.f32"))
    parsed["f32_normal"] = io_maps.load_f32(os.path.join(OUT, "normal.f32"))
    parsed["f32_depth_in"], parsed["f32_normal_in"] = depth, normal
    img = rng.uniform(-0.1, 1.1, (7, 11, 3))
    gray = rng.uniform(0, 1, (7, 11))
    io_maps.save_png(os.path.join(OUT, "image.png"), img)
    io_maps.save_png(os.path.join(OUT, "gray.png"), gray)
    parsed["png_image"] = io_maps.load_png(os.path.join(OUT, "image.png"))
    parsed["png_gray"] = io_maps.load_png(os.path.join(OUT, "gray.png"))
    parsed["png_image_in"], parsed["png_gray_in"] = img, gray
    # point files (inputs of the dataset loader; written by hand here)
    pts = rng.normal(size=(6, 3)).astype(np.float32)
    rgb = rng.integers(0, 256, (6, 3)).astype(np.uint8)
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex 6\nproperty float x\n"
            "property float y\nproperty float z\nproperty uchar red\nproperty uchar green\n"
            "property uchar blue\nelement face 0\nproperty list uchar int vertex_indices\n"
            "end_header\n")
    rec = np.zeros(6, dtype=[("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "u1"), ("g", "u1"),
                             ("b", "u1")])
    rec["x"], rec["y"], rec["z"] = pts.T
    rec["r"], rec["g"], rec["b"] = rgb.T
    with open(os.path.join(OUT, "points_bin.ply"), "wb") as f:
        f.write(head.encode("ascii") + rec.tobytes())
    with open(os.path.join(OUT, "points_ascii.ply"), "w") as f:
        f.write("ply\nformat ascii 1.0\nelement vertex 4\nproperty double x\nproperty double y\n"
                "property double z\nend_header\n")
        for p in rng.normal(size=(4, 3)):
            f.write(" ".join(repr(float(v)) for v in p) + "\n")
    for tag in ("bin", "ascii"):
        p, c = load_points_ply(os.path.join(OUT, f"points_{tag}.ply"))
        parsed[f"pts_{tag}"] = p
        if c is not None:
            parsed[f"pts_{tag}_colors"] = c
    np.savez_compressed(os.path.join(OUT, "parsed.npz"), **parsed)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
