"""Float64 termination rule on the golden scenes: per scene, pixels whose
fragment count differs from the reference's, and for the first one the GPU
trace (fp32-weight T) beside the reference's emitted T.

    python tools/term_debug.py [SCENE ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import golden_io  # noqa: E402
from paper_2411_16392_b200 import rasterizer as rz  # noqa: E402

names = sys.argv[1:] or golden_io.names()
for name in names:
    gc = golden_io.load(name)
    s = gc.settings
    st = rz.RenderSettings(background=np.asarray(s.background), resort=s.resort,
                           euclidean_density=s.euclidean_density)
    prep = rz.prepare(gc.prims, gc.cam, st)
    tg = rz.forward(prep)
    torch.cuda.synchronize()
    nf = tg.to_numpy()["n_fragments"]
    ref = gc.g["map_n_fragments"]
    bad = np.argwhere(nf != ref)
    print(f"{name}: {len(bad)} count flips of {nf.size} px; frags {nf.sum()} vs {ref.sum()}")
    if len(bad):
        v, u = bad[0]
        acc, em = prep.trace_pixel(u, v)
        print(f"  pixel ({u},{v}) ours {nf[v, u]} ref {ref[v, u]}; trace emits {len(em['prim'])}")
        k = min(len(em["T"]), 8)
        print("  last T before each emitted fragment:", em["T"][-k:])
        print("  ref transmittance", gc.g["map_transmittance"][v, u], "ours",
              tg.to_numpy()["transmittance"][v, u])
