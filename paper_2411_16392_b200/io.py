"""On-disk formats of the reference -- drop-in for
``qgsplat.model.save_ply / load_ply`` (model.py:193-249),
``qgsplat.io_maps`` (io_maps.py:1-54: the QGSFMAP1 float maps and 8-bit
PNG) and ``qgsplat.train.load_points_ply`` (train.py:77-118).

Files are byte-identical to the reference's for the same values.  The
device side: ``load_ply_device`` parses straight into pinned host memory
and uploads the six groups as fp32 ``DevicePrimitives``; the writers accept
CUDA tensors (one device-to-host copy each).
"""

import struct

import numpy as np
import torch

from .model import ParameterError, PrimitiveSet

# model.py:193-198: binary little-endian PLY, one vertex per primitive
PLY_BASE = ["x", "y", "z",
            "quat_w", "quat_x", "quat_y", "quat_z",
            "raw_scale_1", "raw_scale_2", "raw_scale_3",
            "raw_sign_1", "raw_sign_2", "raw_sign_3",
            "raw_opacity"]
FIELDS = PrimitiveSet.FIELDS
MAGIC = b"QGSFMAP1"                    # io_maps.py:14


def _host64(a):
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, dtype=np.float64)


def save_ply(path, prims):
    """model.py:201-216.  prims: PrimitiveSet (numpy) or DevicePrimitives."""
    g = {f: _host64(getattr(prims, f)) for f in FIELDS}
    n = g["centers"].shape[0]
    n_sh = g["sh"].shape[1] * g["sh"].shape[2]
    names = PLY_BASE + [f"sh_{k}" for k in range(n_sh)]
    head = "\n".join(["ply", "format binary_little_endian 1.0", f"element vertex {n}"] +
                     [f"property double {nm}" for nm in names] + ["end_header"]) + "\n"
    rows = np.empty((n, len(names)), dtype="<f8")
    rows[:, 0:3] = g["centers"]
    rows[:, 3:7] = g["quats"]
    rows[:, 7:10] = g["raw_scales"]
    rows[:, 10:13] = g["raw_signs"]
    rows[:, 13] = g["raw_opacity"]
    rows[:, 14:] = g["sh"].reshape(n, n_sh)
    with open(path, "wb") as f:
        f.write(head.encode("ascii"))
        f.write(rows.tobytes())


def _read_ply_table(path):
    """header (double properties only) -> (names, (n, len(names)) float64)"""
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ParameterError(f"{path}: not a PLY file")
        names, n = [], 0
        while True:
            line = f.readline()
            if not line:
                raise ParameterError(f"{path}: truncated header")
            tok = line.decode("ascii").split()
            if not tok:
                continue
            if tok[0] == "format" and tok[1] != "binary_little_endian":
                raise ParameterError(f"{path}: unsupported PLY format {tok[1]}")
            if tok[0] == "element" and tok[1] == "vertex":
                n = int(tok[2])
            elif tok[0] == "property":
                if tok[1] != "double":
                    raise ParameterError(f"{path}: expected double properties")
                names.append(tok[2])
            elif tok[0] == "end_header":
                break
        payload = f.read(8 * n * len(names))
    if len(payload) != 8 * n * len(names):
        raise ParameterError(f"{path}: truncated payload")
    return names, np.frombuffer(payload, dtype="<f8").reshape(n, len(names))


def _split(path, names, table):
    if names[:len(PLY_BASE)] != PLY_BASE:
        raise ParameterError(f"{path}: unexpected property layout")
    n_sh = len(names) - len(PLY_BASE)
    if n_sh % 3 != 0 or int(round(np.sqrt(n_sh // 3))) ** 2 * 3 != n_sh:
        raise ParameterError(f"{path}: sh property count {n_sh} is not 3*(deg+1)^2")
    n = table.shape[0]
    return (table[:, 0:3], table[:, 3:7], table[:, 7:10], table[:, 10:13], table[:, 13],
            table[:, 14:].reshape(n, 3, n_sh // 3))


def load_ply(path) -> PrimitiveSet:
    """model.py:219-249: float64 PrimitiveSet."""
    names, table = _read_ply_table(path)
    return PrimitiveSet(*(np.ascontiguousarray(a, dtype=np.float64)
                          for a in _split(path, names, table)))


def load_ply_device(path, device=None):
    """load_ply straight onto the GPU: the groups are converted to fp32 in
    pinned host memory and uploaded asynchronously on the current stream."""
    from .rasterizer import DevicePrimitives
    names, table = _read_ply_table(path)
    parts = _split(path, names, table)
    device = device or torch.device("cuda", torch.cuda.current_device())
    out = []
    for a in parts:
        h = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
        h.numpy()[...] = a
        out.append(h.to(device, non_blocking=True))
    return DevicePrimitives(*out)


def save_f32(path, arr):
    """io_maps.py:17-27: b"QGSFMAP1", <III (h, w, c), float32 row-major."""
    if isinstance(arr, torch.Tensor):
        arr = arr.detach().cpu().numpy()
    arr = np.asarray(arr, dtype=np.float32)
    if arr.ndim == 2:
        arr = arr[:, :, None]
    if arr.ndim != 3:
        raise ValueError("expected (H, W) or (H, W, C) array")
    h, w, c = arr.shape
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<III", h, w, c))
        f.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def load_f32(path):
    """io_maps.py:30-40: float64 (H, W) or (H, W, C)."""
    with open(path, "rb") as f:
        magic = f.read(8)
        if magic != MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}")
        h, w, c = struct.unpack("<III", f.read(12))
        data = np.frombuffer(f.read(4 * h * w * c), dtype="<f4")
    if data.size != h * w * c:
        raise ValueError(f"{path}: truncated payload")
    arr = data.reshape(h, w, c).astype(np.float64)
    return arr[:, :, 0] if c == 1 else arr


def save_png(path, img):
    """io_maps.py:43-47: [0, 1] floats -> 8-bit, round half up."""
    from PIL import Image
    if isinstance(img, torch.Tensor):
        img = img.detach().cpu().numpy()
    data = (np.clip(np.asarray(img), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    Image.fromarray(data).save(path)


def load_png(path):
    """io_maps.py:50-54: float64 in [0, 1], alpha channel dropped."""
    from PIL import Image
    img = np.asarray(Image.open(path), dtype=np.float64) / 255.0
    return img[:, :, :3] if img.ndim == 3 and img.shape[2] == 4 else img


_PLY_TYPES = {"float": "<f4", "double": "<f8", "uchar": "u1", "uint8": "u1", "int": "<i4",
              "uint": "<u4"}


def load_points_ply(path):
    """train.py:77-118: x/y/z (+ optional red/green/blue as [0, 1]) from an
    ascii or binary little-endian point PLY."""
    with open(path, "rb") as f:
        if f.readline().strip() != b"ply":
            raise ValueError(f"{path}: not a PLY file")
        fmt, n, props, vertex = None, 0, [], False
        while True:
            tok = f.readline().decode("ascii").split()
            if not tok:
                continue
            key = tok[0]
            if key == "format":
                fmt = tok[1]
            elif key == "element":
                vertex = tok[1] == "vertex"
                n = int(tok[2]) if vertex else n
            elif key == "property" and vertex:
                props.append((tok[1], tok[2]))
            elif key == "end_header":
                break
        if fmt == "ascii":
            table = np.loadtxt(f, max_rows=n).reshape(n, len(props))
        elif fmt == "binary_little_endian":
            dt = np.dtype([(f"c{i}", _PLY_TYPES[t]) for i, (t, _) in enumerate(props)])
            raw = np.frombuffer(f.read(dt.itemsize * n), dtype=dt)
            table = np.column_stack([raw[f"c{i}"].astype(np.float64) for i in range(len(props))])
        else:
            raise ValueError(f"{path}: unsupported PLY format {fmt}")
    names = [nm for _, nm in props]
    pts = table[:, [names.index(c) for c in ("x", "y", "z")]]
    colors = table[:, [names.index(c) for c in ("red", "green", "blue")]] / 255.0 \
        if "red" in names else None
    return pts, colors
