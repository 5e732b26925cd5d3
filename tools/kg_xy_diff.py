import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2411_16392_b200 import rasterizer as rz, scenes
sc = scenes.config5()
cam = sc.cams[0]
up = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in sc.upstream[0].items()}
dev = rz.DevicePrimitives.from_host(sc.prims)
prep = rz.prepare(dev, cam)
tg = rz.forward(prep)
a = rz.kernel_grads(prep, tg, up).cpu().numpy().astype(np.float64)
tg.frag_xy = None
b = rz.kernel_grads(prep, tg, up).cpu().numpy().astype(np.float64)
scale = np.abs(b).max(axis=0) + 1e-30
rel = np.abs(a - b) / scale
idx = np.argsort(rel.max(axis=1))[::-1][:8]
for p in idx:
    s = int(np.argmax(rel[p]))
    print(p, "slot", s, "rel", rel[p, s], "xy", a[p, s], "fp64", b[p, s], "planar", prep.planar.cpu().numpy()[p])
sc_ = prep.scales.cpu().numpy()
print(sc_[idx[:3]])
