"""Per-pixel gradient contributions of ONE primitive, GPU vs the float64
oracle, mapped to raw parameters (diagnostics for gradient violations).

    python tools/grad_frag_diag.py --config c4 --prim 1269412 [--view 0] [--top 10]

GPU: kernel_grads with the view's upstream kept at a single pixel, for each
pixel of the primitive's box (its 16 slots at that pixel), times the chain's
Jacobian (chain of unit slot vectors).  Oracle: qgs_oracle.fragment_contributions
times qgs_oracle.chain_jacobian.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import _lib, rasterizer as rz, scenes  # noqa: E402

GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh", "screen_center")

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--view", type=int, default=0)
ap.add_argument("--prim", type=int, required=True)
ap.add_argument("--top", type=int, default=12)
a = ap.parse_args()
sc = scenes.CONFIGS[a.config](views=a.view + 1)
cam, up = sc.cams[a.view], sc.upstream[a.view]
p = a.prim
H, W = cam.height, cam.width
dev = rz.DevicePrimitives.from_host(sc.prims)
prep = rz.prepare(dev, cam)
tg = rz.forward(prep)
bb = prep.pix_bbox[p].cpu().numpy()
ups = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in up.items()}

# chain Jacobian of primitive p on the GPU: chain(unit slot j)
KG = _lib.KG_STRIDE
J_gpu = []
for j in range(KG):
    kg = torch.zeros((len(dev), KG), dtype=torch.float32, device="cuda")
    kg[p, j] = 1.0
    out = rz.chain(prep, kg)
    J_gpu.append(np.concatenate([getattr(out, g)[p].reshape(-1).double().cpu().numpy()
                                 for g in GROUPS]))
J_gpu = np.stack(J_gpu, axis=1)                      # (raw, 16)

gpu_px = {}
for v in range(bb[2], bb[3] + 1):
    for u in range(bb[0], bb[1] + 1):
        one = {}
        for k, t in ups.items():
            z = torch.zeros_like(t)
            z[v, u] = t[v, u]
            one[k] = z
        kg = rz.kernel_grads(prep, tg, one)
        row = kg[p].double().cpu().numpy()
        if np.any(row != 0):
            gpu_px[v * W + u] = J_gpu @ row
torch.cuda.synchronize()

vw = qo.prepare(sc.prims.astype(np.float64), cam)
ref = qo.forward(vw)
pxs, ts, slots = qo.fragment_contributions(vw, ref, {k: np.asarray(x, np.float64) for k, x in up.items()}, p)
Jr = qo.chain_jacobian(vw, [p])
J_ref = np.concatenate([Jr[g][0] for g in GROUPS], axis=0)   # (raw, 33)
ref_px = {}
for px, sl in zip(pxs.tolist(), slots):
    ref_px[px] = ref_px.get(px, 0) + J_ref @ sl
names = [f"{g}[{i}]" for g in GROUPS for i in range(
    {"centers": 3, "quats": 4, "raw_scales": 3, "raw_signs": 3, "raw_opacity": 1,
     "sh": 3 * sc.prims.sh.shape[2], "screen_center": 2}[g])]
tot_g = sum(gpu_px.values())
tot_r = sum(ref_px.values())
print(f"prim {p}: gpu pixels {len(gpu_px)}, oracle fragments {len(pxs)} at {len(ref_px)} pixels")
for i, n in enumerate(names):
    if n.startswith("sh"):
        continue
    print(f"  {n:16s} gpu {tot_g[i]: .6e} ref {tot_r[i]: .6e} diff {tot_g[i] - tot_r[i]: .3e}")
# pixels with the largest disagreement on the worst raw element
worst = int(np.argmax(np.abs(tot_g - tot_r) / (1e-5 + 1e-3 * np.abs(tot_r))))
print("worst element", names[worst])
allpx = sorted(set(gpu_px) | set(ref_px))
d = [(abs(gpu_px.get(q, np.zeros_like(tot_g))[worst] - ref_px.get(q, np.zeros_like(tot_g))[worst]), q)
     for q in allpx]
d.sort(reverse=True)
for e, q in d[: a.top]:
    gv = gpu_px.get(q, np.zeros_like(tot_g))[worst]
    rv = ref_px.get(q, np.zeros_like(tot_g))[worst]
    print(f"  px u={q % W} v={q // W}: gpu {gv: .6e} ref {rv: .6e} diff {e:.3e}  t_ref "
          f"{ts[pxs == q]}")
