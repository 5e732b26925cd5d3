"""Print a JSON parity report of the GPU path vs the float64 oracle.

    python tools/parity_report.py [--scenes c1,c2] [--views 1] [--out FILE] [--fp32-decisions]

Golden fixtures are compared against the reference outputs stored in them;
generated configs (c1..c5, optionally shrunk with --n/--res) are compared
against the oracle computed in-process on the host cores.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import qgs_oracle as qo  # noqa: E402
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402
from tests import golden_io, parity  # noqa: E402


EXACT = "--fp32-decisions" not in sys.argv    # settings.exact_decisions (the default)


def gpu_run(prims, cam, st, up):
    s = rz.RenderSettings(background=np.asarray(st.background), resort=st.resort,
                          euclidean_density=st.euclidean_density, exact_decisions=EXACT)
    prep = rz.prepare(prims, cam, s)
    tg = rz.forward(prep)
    gr = rz.backward(prep, tg, up)
    torch.cuda.synchronize()
    return prep, tg.to_numpy(), gr.to_numpy()


def compare(name, prims, cam, st, up, ref_maps, ref_grads, ref_prep):
    prep, maps, grads = gpu_run(prims, cam, st, up)
    rec = {"scene": name, "P": len(prims), "n_pairs": prep.n_pairs}
    rec["bbox_equal"] = bool(np.array_equal(prep.pix_bbox.cpu().numpy().astype(np.int64),
                                            ref_prep["pix_bbox"]))
    rec["tile_offsets_equal"] = bool(np.array_equal(
        prep.tile_offsets.cpu().numpy().astype(np.int64), ref_prep["tile_offsets"]))
    tp = prep.tile_prims.cpu().numpy().astype(np.int64)
    rec["tile_prims_equal"] = bool(np.array_equal(tp, ref_prep["tile_prims"]))
    if not rec["tile_prims_equal"] and len(tp) == len(ref_prep["tile_prims"]):
        rec["tile_prims_mismatch"] = int((tp != ref_prep["tile_prims"]).sum())
    rec["image"] = parity.image_report(maps, ref_maps)
    rec["grads"] = parity.grad_report(grads, ref_grads)
    rec["order_violations"] = [int(maps["order_violations"]), int(ref_maps.get("order_violations", -1))]
    return rec


def golden_case(name):
    gc = golden_io.load(name)
    g = gc.g
    ref_maps = {k: g[f"map_{k}"] for k in ("color", "alpha", "depth", "normal", "depth_median",
                                           "transmittance", "curvature", "distortion",
                                           "n_fragments")}
    ref_maps["order_violations"] = int(g["order_violations"])
    ref_grads = {k: g[f"grad_{k}"] for k in parity.GRAD_GROUPS + ("screen_center",)}
    ref_prep = {k: g[k] for k in ("pix_bbox", "tile_offsets", "tile_prims")}
    return compare(name, gc.prims, gc.cam, gc.settings, gc.upstream, ref_maps, ref_grads, ref_prep)


def generated_case(cfg, views, **kw):
    sc = scenes.CONFIGS[cfg](**kw)
    out = []
    for v in range(min(views, len(sc.cams))):
        cam, up = sc.cams[v], sc.upstream[v] if sc.upstream else {}
        prims64 = sc.prims.astype(np.float64)
        t0 = time.time()
        vw = qo.prepare(prims64, cam)
        fw = qo.forward(vw)
        gr = qo.backward(vw, fw, {k: np.asarray(a, np.float64) for k, a in up.items()})
        t_cpu = time.time() - t0
        rec = compare(f"{cfg}_v{v}", sc.prims, cam, qo.Settings(), up, fw, gr,
                      {"pix_bbox": vw.pix_bbox, "tile_offsets": vw.tile_offsets,
                       "tile_prims": vw.tile_prims})
        rec["oracle_seconds"] = t_cpu
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", default="golden,c1,c2")
    ap.add_argument("--views", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fp32-decisions", action="store_true",
                    help="RenderSettings(exact_decisions=False)")
    a = ap.parse_args()
    report = []
    for s in a.scenes.split(","):
        if s == "golden":
            for n in golden_io.names():
                report.append(golden_case(n))
        else:
            report.extend(generated_case(s, a.views))
        print(json.dumps(report[-1]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
