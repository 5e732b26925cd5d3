"""Compare kernel-level gradient slots (GPU vs oracle) and locate bad primitives.

    python tools/kg_diff.py c2_small
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import rasterizer as rz  # noqa: E402
from tests import golden_io  # noqa: E402

# oracle 33-slot layout -> folded 22-slot layout
def fold(kg33, wv, sc):
    P = len(kg33)
    out = np.zeros((P, 22))
    out[:, 0:3] = kg33[:, 0:3]
    gM = kg33[:, 3:12].reshape(P, 3, 3) + kg33[:, 22:31].reshape(P, 3, 3).transpose(0, 2, 1)
    out[:, 3:12] = gM.reshape(P, 9)
    out[:, 12] = kg33[:, 12] + kg33[:, 31] * sc[:, 2]
    out[:, 13] = kg33[:, 13] + kg33[:, 32] * sc[:, 2]
    out[:, 14] = kg33[:, 14]
    out[:, 15:17] = kg33[:, 15:17]
    out[:, 17] = kg33[:, 17] + kg33[:, 31] * wv[:, 0] + kg33[:, 32] * wv[:, 1]
    out[:, 18:22] = kg33[:, 18:22]
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2_small"
    gc = golden_io.load(name)
    st = rz.RenderSettings(background=np.asarray(gc.settings.background),
                           resort=gc.settings.resort,
                           euclidean_density=gc.settings.euclidean_density)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    kg = rz.kernel_grads(prep, tg, gc.upstream).cpu().numpy()[:, :22].astype(np.float64)
    vw = qo.prepare(gc.prims, gc.cam, gc.settings)
    fw = qo.forward(vw)
    ko = fold(qo.kernel_grads(vw, fw, gc.upstream), vw.wv, vw.scales)
    names = ["oh0", "oh1", "oh2"] + [f"M{i}" for i in range(9)] + ["w1", "w2", "iw3", "s1", "s2",
                                                                  "s3", "alpha", "c0", "c1", "c2"]
    err = np.abs(kg - ko)
    bad = err > 1e-5 + 1e-3 * np.abs(ko)
    print("violations per slot:", dict(zip(names, bad.sum(axis=0).tolist())))
    cols = [19, 20, 21]
    e = err[:, cols].max(axis=1)
    worst = np.argsort(-e)[:5]
    for p in worst:
        print(f"prim {p}: gpu col {kg[p, cols]} ref {ko[p, cols]} alpha g {kg[p, 18]:.4e} r {ko[p, 18]:.4e}")
    # pixels of the worst primitive: compare per-pixel w from traces
    p = int(worst[0])
    bb = vw.pix_bbox[p]
    up = gc.upstream["color"]
    sg = so = np.zeros(3)
    nd = 0
    for v in range(bb[2], bb[3] + 1):
        for u in range(bb[0], bb[1] + 1):
            _, ge = prep.trace_pixel(u, v)
            _, oe = qo.trace_pixel(vw, u, v)
            wg = [ab * T for pr, ab, T in zip(ge["prim"], ge["abar"], ge["T"]) if pr == p]
            wo = [ab * T for pr, ab, T in zip(oe["prim"], oe["abar"], oe["T"]) if pr == p]
            if wg:
                sg = sg + wg[0] * up[v, u]
            if wo:
                so = so + wo[0] * up[v, u]
            if bool(wg) != bool(wo) or (wg and abs(wg[0] - wo[0]) > 1e-5):
                nd += 1
                if nd <= 5:
                    print(f"  px ({u},{v}) gpu w {wg} ref w {wo}")
    print(f"trace sums: gpu {sg} ref {so}; differing pixels {nd}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
