"""Compare per-pixel fragment streams (GPU vs oracle) at the worst pixels.

    python tools/trace_diff.py c1 [--k 6]            # a golden scene
    python tools/trace_diff.py --config c3 [--k 6]   # view 0 of a generated config
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import rasterizer as rz  # noqa: E402
from tests import golden_io  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("scene", nargs="?")
    ap.add_argument("--config", default=None)
    ap.add_argument("--k", type=int, default=6)
    a = ap.parse_args()
    if a.config:
        from paper_2411_16392_b200 import scenes
        sc = scenes.CONFIGS[a.config]()
        gc = type("G", (), {})()
        gc.prims, gc.cam = sc.prims, sc.cams[0]
        gc.settings = qo.Settings() if hasattr(qo, "Settings") else rz.RenderSettings()
    else:
        gc = golden_io.load(a.scene)
    st = rz.RenderSettings(background=np.asarray(gc.settings.background),
                           resort=gc.settings.resort,
                           euclidean_density=gc.settings.euclidean_density)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep).to_numpy()
    vw = qo.prepare(gc.prims.astype(np.float64) if a.config else gc.prims, gc.cam, gc.settings)
    ref = qo.forward(vw)
    d = np.abs(tg["color"] - ref["color"]).max(axis=2)
    same = tg["n_fragments"] == ref["n_fragments"]
    order = np.argsort(-(d * same).ravel())[: a.k]
    W = gc.cam.width
    for idx in order:
        v, u = divmod(int(idx), W)
        print(f"=== pixel u={u} v={v} colour err {d[v, u]:.3e} nfrag gpu {tg['n_fragments'][v, u]}"
              f" ref {ref['n_fragments'][v, u]} alpha gpu {tg['alpha'][v, u]:.6f} "
              f"ref {ref['alpha'][v, u]:.6f}")
        ga, ge = prep.trace_pixel(u, v)
        oa, oe = qo.trace_pixel(vw, u, v)
        print(f" accepted: gpu {len(ga['prim'])} ref {len(oa['prim'])}")
        sa, so = set(ga["prim"].tolist()), set(oa["prim"].tolist())
        if sa != so:
            print("  only gpu:", sorted(sa - so)[:10], " only ref:", sorted(so - sa)[:10])
        for i in range(max(len(ge["prim"]), len(oe["prim"]))):
            g = (ge["prim"][i], ge["t"][i], ge["abar"][i], ge["T"][i]) if i < len(ge["prim"]) else None
            o = (oe["prim"][i], oe["t"][i], oe["abar"][i], oe["T"][i]) if i < len(oe["prim"]) else None
            flag = ""
            if g is None or o is None or g[0] != o[0]:
                flag = "  <-- order/membership"
            elif abs(g[2] - o[2]) > 1e-5:
                flag = f"  <-- abar diff {g[2] - o[2]:.2e}"
            gs = f"{g[0]:6d} t={g[1]:.7f} ab={g[2]:.6f}" if g else " " * 30
            os_ = f"{o[0]:6d} t={o[1]:.7f} ab={o[2]:.6f}" if o else ""
            print(f"  {i:3d} gpu {gs} | ref {os_}{flag}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
