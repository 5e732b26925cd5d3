"""Time the device loss producers (csrc/losses.cu) at a C3 view size and the
Adam step + densification (csrc/optim.cu) at C3's primitive count, and
compare with the float64 CPU oracles on the same inputs.

    python tools/bench_aux.py [--H 1200] [--W 1600] [--P 500000] [--reps 20] [--no-cpu]

Prints one JSON line: device ms (CUDA events, inputs resident, L2 flushed
between repetitions), algorithmic HBM bytes per call and the achieved GB/s
against MEASURED_PEAKS.json, plus the CPU oracles' times (one thread).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import losses as L  # noqa: E402
from paper_2411_16392_b200.rasterizer import zero_upstream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=1200)
ap.add_argument("--W", type=int, default=1600)
ap.add_argument("--P", type=int, default=500_000)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()
H, W = a.H, a.W
dev = torch.device("cuda:0")
rng = np.random.default_rng(0)


class Cam:
    fx = fy = 1400.0
    cx, cy = W / 2, H / 2
    width, height = W, H
    world_to_camera = np.eye(4)


yy, xx = np.mgrid[0:H, 0:W]
maps = {
    "color": rng.uniform(0, 1, (H, W, 3)).astype(np.float32),
    "distortion": rng.exponential(0.01, (H, W)).astype(np.float32),
    "alpha": rng.uniform(0.3, 1.0, (H, W)).astype(np.float32),
    "normal": rng.normal(0, 0.5, (H, W, 3)).astype(np.float32),
    "curvature": rng.normal(0, 2, (H, W)).astype(np.float32),
    "depth_median": (3.0 + 0.3 * np.sin(xx / 90.0) * np.cos(yy / 70.0)).astype(np.float32),
}
gt = np.clip(maps["color"] + rng.normal(0, 0.05, (H, W, 3)), 0, 1).astype(np.float32)


class T:
    pass


t = T()
for k, v in maps.items():
    setattr(t, k, torch.from_numpy(v).to(dev))
gt_d = torch.from_numpy(gt).to(dev)
up = zero_upstream(Cam, dev)
flush = torch.empty((256 << 20,), dtype=torch.uint8, device=dev)
w = L.LossWeights()
px = H * W


def timed(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return float(np.median(ms))


res = {}
res["photometric_ms"] = timed(lambda: L._photometric_dev(t.color, gt_d, w.lambda_photo_ssim, 1.0,
                                                          up["color"], torch.zeros(3, dtype=torch.float64, device=dev)))
res["all_terms_ms"] = timed(lambda: L.accumulate_upstream(t, gt_d, Cam, up, w))
# algorithmic bytes: photometric reads render+gt twice, writes+reads the fp64
# adjoint maps, read-modify-writes d_render; distortion reads the map and
# read-modify-writes its upstream; consistency reads depth, alpha, normal,
# curvature twice and read-modify-writes three upstream maps
b_ph = px * 3 * (4 * 2 * 2 + 8 * 3 * 2 + 4 * 2)
b_di = px * (4 + 8)
b_nc = px * (2 * (4 + 4 + 12 + 4) + 2 * (4 + 12 + 4))
res["photometric_bytes"] = b_ph
res["all_terms_bytes"] = b_ph + b_di + b_nc
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        hbm = float(v)
res["hbm_peak_gbs"] = hbm
res["all_terms_gbs"] = res["all_terms_bytes"] / res["all_terms_ms"] / 1e6
if hbm:
    res["all_terms_frac"] = res["all_terms_gbs"] / hbm
if not a.no_cpu:
    from oracle import losses_oracle as lo
    t0 = time.perf_counter()
    lo.photometric(maps["color"], gt, w.lambda_photo_ssim)
    lo.depth_distortion(maps["distortion"])
    N, m = lo.depth_to_normal(maps["depth_median"], maps["alpha"], (Cam.fx, Cam.fy, Cam.cx, Cam.cy))
    lo.normal_consistency(maps["alpha"], maps["normal"], maps["curvature"], N, m)
    res["cpu_oracle_ms"] = (time.perf_counter() - t0) * 1e3
    res["cpu_cores"] = 1

# ---- Adam step (+ densification statistics) and one densification pass
from paper_2411_16392_b200 import densify, optim  # noqa: E402
from paper_2411_16392_b200.rasterizer import DevicePrimitives, GradientBuffer  # noqa: E402

P, K = a.P, 16
q = rng.normal(size=(P, 4))
host = {"centers": rng.normal(0, 1, (P, 3)), "quats": q / np.linalg.norm(q, axis=1, keepdims=True),
        "raw_scales": rng.normal(-4, 1, (P, 3)), "raw_signs": rng.normal(0, 1.5, (P, 3)),
        "raw_opacity": rng.normal(0, 2.5, P), "sh": rng.normal(0, 0.5, (P, 3, K))}
prims = DevicePrimitives(**{k: torch.from_numpy(v.astype(np.float32)).to(dev) for k, v in host.items()})
gb = GradientBuffer.zeros(prims)
for k in optim.GROUPS + ("screen_center",):
    getattr(gb, k).normal_(0, 0.01)
opt = optim.Adam(prims)
stats = densify.DensifyStats(P, dev)
lrs = {"centers": 1.6e-4, "quats": 1e-3, "raw_scales": 5e-3, "raw_signs": 5e-3,
       "raw_opacity": 0.05, "sh": 2.5e-3}
res["adam_ms"] = timed(lambda: opt.step(prims, gb, lrs, stats=stats))
fl = 3 + 4 + 3 + 3 + 1 + 3 * K
res["adam_bytes"] = P * (fl * 4 * (1 + 2 + 4) + 2 * 4 + (8 + 8 + 24) * 2)
res["adam_gbs"] = res["adam_bytes"] / res["adam_ms"] / 1e6
if hbm:
    res["adam_frac"] = res["adam_gbs"] / hbm
cfg = densify.DensifyConfig(0.3, 0.005, 0.005, 0.5, P + P // 10)
stats.grad_accum.uniform_(0, 1).mul_(3)
stats.grad_count.fill_(2)
densify.densify_and_prune(prims, opt, stats, cfg, 3.0)     # warm-up: workspace, allocator
opt = optim.Adam(prims)
stats = densify.DensifyStats(P, dev)
stats.grad_accum.uniform_(0, 1).mul_(3)
stats.grad_count.fill_(2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
p2 = densify.densify_and_prune(prims, opt, stats, cfg, 3.0)
e1.record()
torch.cuda.synchronize()
res["densify_ms"] = e0.elapsed_time(e1)
res["densify_in_out"] = [P, len(p2)]
if not a.no_cpu:
    from oracle import optim_oracle as oo
    hp = {k: v.astype(np.float32).astype(np.float64) for k, v in host.items()}
    hm = {k: np.zeros_like(v) for k, v in hp.items()}
    hv = {k: np.zeros_like(v) for k, v in hp.items()}
    hg = {k: getattr(gb, k).cpu().numpy().astype(np.float64) for k in optim.GROUPS}
    t0 = time.perf_counter()
    oo.adam_step(hp, hg, hm, hv, 1, lrs)
    res["cpu_oracle_adam_ms"] = (time.perf_counter() - t0) * 1e3

# ---- multi-view reprojection + NCC between two C3-size views of a plane
from paper_2411_16392_b200 import multiview as MV  # noqa: E402


class MvCam:
    def __init__(self, eye_x):
        self.fx = self.fy = 1400.0
        self.cx, self.cy = W / 2, H / 2
        self.width, self.height = W, H
        w2c = np.eye(4)
        w2c[:3, 3] = [-eye_x, 0.0, 3.0]
        self.world_to_camera = w2c


def plane_maps(c):
    uu, vv = np.meshgrid((np.arange(W) + 0.5 - c.cx) / c.fx, (np.arange(H) + 0.5 - c.cy) / c.fy)
    d = np.stack([uu, vv, np.ones_like(uu)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    t = 3.0 / d[..., 2]
    X = t[..., None] * d - c.world_to_camera[:3, 3]
    img = 0.5 + 0.25 * np.sin(30 * X[..., 0]) * np.cos(20 * X[..., 1])
    return {"depth": torch.from_numpy(t.astype(np.float32)).to(dev),
            "alpha": torch.ones((H, W), device=dev),
            "normal": torch.tensor([0.0, 0.0, -1.0], device=dev).expand(H, W, 3).contiguous(),
            "image": torch.from_numpy(img.astype(np.float32)).to(dev)}


cr, cn = MvCam(0.0), MvCam(0.05)
mr, mn = plane_maps(cr), plane_maps(cn)
up_n = zero_upstream(Cam, dev)
vals = [None]


def mv_step():
    vals[0] = MV.accumulate_multiview(mr, cr, mn, cn, up, up_n, 0.05)


res["multiview_ms"] = timed(mv_step)
res["multiview_n_valid"] = int(vals[0][1].item())
print(json.dumps({"workload": f"losses {W}x{H}; adam + densify P={P} SH3; multiview 2x{W}x{H}",
                  **res}))
