"""Benchmark: QGS tile rasterizer forward+backward Mpixels/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (views sharded, one NCCL all-reduce)

One step = prepare + forward + backward + chain for every camera view of the
config (views sharded round-robin over ranks, primitives replicated), then a
single all-reduce of the packed raw-parameter gradients when N > 1.  Timing:
CUDA events on the launching stream, barrier + synchronize on both sides,
max over ranks.  Inputs are synthetic, seeded (paper_2411_16392_b200/scenes.py).

Rank 0 prints ONE JSON line.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "fwd+bwd Mpixels/s"
UNIT = "Mpx/s"
# SURVEY.md section 8d op costs per candidate / fragment (add+mul, SFU-class)
C_MISS, S_MISS = 63.0, 2.5
C_HIT, S_HIT = 136.0, 18.1
C_COMP = 37.0
C_GRAD, S_GRAD = 428.0, 36.0
BIN_BYTES_PER_PAIR = 20.0   # bucketed composite key write + read (16) + tile_prims write (4)
OUR_LAUNCHES_PER_VIEW = 14  # preprocess, 3 scan, tile_diff, tile_offsets, pixel_rays, pair_key, 2 tile_order, tile_sort, fwd, bwd, chain


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _kg_stride():
    from paper_2411_16392_b200 import _lib
    return _lib.KG_STRIDE


def traffic_bytes(kernel, exact=True):
    """DRAM bytes (read + write) per launch of `kernel` from the newest committed
    `ncu --set full` capture (profiles/*_traffic.json, tools/round_summarize.sh),
    or None.  One launch = one view here, like the roofline's achieved figure.
    The forward of the exact-decision mode is raster_fwd_exact_kernel."""
    import glob
    files = sorted(glob.glob(os.path.join(HERE, "profiles", "*_traffic.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        t = json.load(f)
    names = [kernel + "_exact_kernel", kernel + "_kernel"] if exact else [kernel + "_kernel"]
    for nm in names:
        e = t.get(nm)
        if e is not None:
            return {"bytes_per_launch": e["dram_bytes"], "kernel": nm,
                    "source": os.path.relpath(files[-1], HERE)}
    return None


def hbm_view(traffic, t_launch_s, peaks):
    if not traffic or t_launch_s <= 0:
        return None
    gbs = traffic["bytes_per_launch"] / t_launch_s / 1e9
    return {"bound": "hbm", "unit": "GB/s", "achieved": gbs, "peak": peaks["hbm_gbs"],
            "frac": gbs / peaks["hbm_gbs"], "traffic": traffic["bytes_per_launch"]}


def load_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def measure_compute_peaks(device_index):
    from paper_2411_16392_b200 import build
    lib = ctypes.CDLL(build.PEAKS_LIB)
    f, m = ctypes.c_double(), ctypes.c_double()
    sms, clk = ctypes.c_int(), ctypes.c_int()
    rc = lib.qgs_peaks(device_index, ctypes.byref(f), ctypes.byref(m), ctypes.byref(sms),
                       ctypes.byref(clk))
    if rc != 0:
        raise RuntimeError(f"qgs_peaks failed ({rc})")
    return {"fp32_tflops": f.value, "mufu_tops": m.value, "sms": sms.value,
            "clock_mhz": clk.value / 1000.0}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def scene_for(name):
    from paper_2411_16392_b200 import scenes
    return scenes.CONFIGS[name]()


def workload_desc(sc):
    m = sc.meta
    return (f"{sc.name}: N={m['N']}, {m['res'][0]}x{m['res'][1]}, SH{m['sh_deg']}, "
            f"{m['views']} views")


# --------------------------------------------------------------------- ours

def run_ours(a):
    import torch.distributed as dist

    from paper_2411_16392_b200 import rasterizer as rz
    from paper_2411_16392_b200.dist import gpu_step, shard_views

    rank, world, local = env_rank()
    local = local % torch.cuda.device_count()   # (only the gloo check shares a GPU)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:   # functional check of the multi-rank path on a single-GPU box
            dist.init_process_group(a.dist_backend)
    sc = scene_for(a.config)
    cams = sc.cams
    V = len(cams)
    mine = shard_views(V, rank, world)
    H, W = cams[0].height, cams[0].width
    st = rz.RenderSettings(exact_decisions=not a.fp32_decisions)

    dev = rz.DevicePrimitives.from_host(sc.prims, device)
    ups = {v: {k: torch.from_numpy(np.ascontiguousarray(u)).to(device)
               for k, u in sc.upstream[v].items()} for v in mine}
    grads = rz.GradientBuffer.zeros_flat(dev)
    counters = torch.zeros(5, dtype=torch.int64, device=device)
    side = torch.cuda.Stream(device=device)
    stream = torch.cuda.current_stream()

    def step(hook=None, count=False):
        # dist.gpu_step: this rank's views (pipelined prepare, forward,
        # backward, chain) + one all-reduce -- the same call a user makes
        gpu_step(dev, cams, ups, st, rank, world, grads=grads, views=mine, side=side,
                 hook=hook, counters=counters if count else None)

    # warm-up (also the counted pass for the algorithmic work)
    for w in range(max(a.warmup, 3)):
        step(count=(w == 0))
    torch.cuda.synchronize()
    cnt = counters.cpu().numpy().astype(np.float64)     # this rank's views
    n_pairs_mine = [rz.prepare(dev, cams[v], st).n_pairs for v in mine]

    # timed region: CUDA events on the launching stream at every hook
    K = a.steps
    evs = []

    def hook_for(rec):
        def hook(name, i):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            rec.append((name, i, e))
        return hook

    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record(stream)
        for k in range(K):
            rec = []
            evs.append(rec)
            step(hook=hook_for(rec))
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / K

    def span(rec, a_name, b_name):
        ev = {(n, i): e for n, i, e in rec}
        return [ev[(a_name, i)].elapsed_time(ev[(b_name, i)]) for i in range(len(mine))]

    # the step's own spans (the next view's binning runs beside them on the
    # side stream, so they include its interference) ...
    fwd_ms_step = sum(sum(span(r, "view_begin", "fwd_end")) for r in evs) / K
    bwd_ms_step = sum(sum(span(r, "fwd_end", "bwd_end")) for r in evs) / K
    # ... and the raster kernels alone (this rank's views prepared first, then
    # forward / backward each bracketed by events, nothing beside them): the
    # roofline's launch durations
    fwd_ms, bwd_ms, frag_log = isolated_raster_ms(rz, dev, cams, mine, ups, st, stream)
    view_ms = np.mean([span(r, "view_begin", "view_end") for r in evs], axis=0).tolist() \
        if mine else []
    red_ms = float(np.mean([{n: e for n, _, e in r}["reduce_begin"].elapsed_time(
        {n: e for n, _, e in r}["reduce_end"]) for r in evs]))
    t_ms = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_max = float(t_ms.item())
    total_px = V * H * W
    value = total_px / 1e6 / (ms_max / 1e3)
    mine_rec = {"rank": rank, "views": mine, "ms_per_step": ms, "view_ms": view_ms,
                "allreduce_ms": red_ms}
    per_rank = [mine_rec]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine_rec)

    # end to end through the public API, host buffers in pinned memory
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, rz, sc, mine, device, st, world)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, peaks_kind = load_peaks()
    cp = measure_compute_peaks(local)
    # algorithmic work of this rank's views per step
    n_box, n_acc, n_comp, n_cull, n_coarse = cnt
    n_miss = n_box - n_acc
    F_fwd = n_miss * C_MISS + n_acc * C_HIT + n_comp * C_COMP
    S_fwd = n_miss * S_MISS + n_acc * S_HIT
    F_bwd = n_comp * C_GRAD
    S_bwd = n_comp * S_GRAD
    P32 = cp["fp32_tflops"] * 1e12
    PSF = cp["mufu_tops"] * 1e12
    BW = peaks["hbm_gbs"] * 1e9
    B_bin = BIN_BYTES_PER_PAIR * sum(n_pairs_mine)
    T_roof = max((F_fwd + F_bwd) / P32, (S_fwd + S_bwd) / PSF) + B_bin / BW
    kernels = {"raster_bwd": (F_bwd, S_bwd, bwd_ms), "raster_fwd": (F_fwd, S_fwd, fwd_ms)}
    dom = max(kernels, key=lambda k: kernels[k][2])
    F, S, kms = kernels[dom]
    t_k = kms / 1e3
    roof = {
        "bound": "fp32+sfu", "kernel": dom, "unit": "TFLOP/s",
        "achieved": F / t_k / 1e12, "peak": cp["fp32_tflops"], "frac": F / t_k / P32,
        "sfu_achieved_tops": S / t_k / 1e12, "sfu_peak_tops": cp["mufu_tops"],
        "sfu_frac": S / t_k / PSF,
        "roof_frac": max(F / P32, S / PSF) / t_k,
        "kernel_ms_per_step": kms, "fwd_ms_per_step": fwd_ms, "bwd_ms_per_step": bwd_ms,
        "fwd_ms_per_step_in_pipeline": fwd_ms_step, "bwd_ms_per_step_in_pipeline": bwd_ms_step,
        # dram__bytes_read + dram__bytes_write per launch (one view) of the
        # dominant kernel from the committed ncu --set full capture
        "traffic": (traffic_bytes(dom, st.exact_decisions) or {}).get("bytes_per_launch"),
        "traffic_source": traffic_bytes(dom, st.exact_decisions),
        # the contract's HBM view of the same kernel: its DRAM bytes per launch
        # (ncu) over its measured launch time, against MEASURED_PEAKS' copy
        # bandwidth -- small, because the raster is FP32/SFU-bound, not HBM
        "hbm_view": hbm_view(traffic_bytes(dom, st.exact_decisions), t_k / max(len(mine), 1), peaks),
        "peak_source": f"fp32/mufu measured live (tools/peaks.cu); hbm {peaks_kind} "
                       f"MEASURED_PEAKS.json {peaks['hbm_gbs']} GB/s",
        "step_roofline_ms": T_roof * 1e3,
        "step_roofline_frac": (T_roof * 1e3) / ms if world == 1 else None,
        # both raster kernels against the same peaks (the dominant one is above)
        "per_kernel": {k: {"achieved_tflops": v[0] / (v[2] / 1e3) / 1e12,
                           "frac": v[0] / (v[2] / 1e3) / P32,
                           "sfu_frac": v[1] / (v[2] / 1e3) / PSF, "ms_per_step": v[2]}
                       for k, v in kernels.items() if v[2] > 0},
        "algorithmic": {"candidates": n_box, "accepted": n_acc, "composited": n_comp,
                        "after_conic_cull": n_cull, "after_coarse_test": n_coarse,
                        "pairs": sum(n_pairs_mine), "flop_fwd": F_fwd, "flop_bwd": F_bwd,
                        "sfu_fwd": S_fwd, "sfu_bwd": S_bwd},
    }
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": a.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (seeded, BASELINE config shapes; scenes.py)",
        "config": config_of(sc, a),
        "step": f"{V} full views: prepare + forward + backward + chain each"
                + (", then 1 NCCL all-reduce" if world > 1 else ""),
        "parallelism": f"views sharded over {world} GPU(s), primitives replicated",
        "l2": "working set > L2 (126 MB): per-view sort buffers + maps are GBs",
        "roofline": roof, "clocks": clk.summary(),
        "gpu_launches": OUR_LAUNCHES_PER_VIEW * V * K,
        "compute_peaks": cp,
        "per_rank": per_rank,
        "fragment_log": frag_log,
    }
    if e2e is not None:
        out["e2e"] = e2e
    if world == 1 and not a.no_cpu:
        out["cpu_baseline"] = cpu_baseline(sc)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def isolated_raster_ms(rz, dev, cams, views, ups, st, stream, reps=2):
    """forward and backward (kernel gradients) time per step, each view's
    raster kernels alone on the device (CUDA events on the launching stream)"""
    fwd = bwd = 0.0
    log = {"pages_used": 0, "bytes_used": 0, "bytes_allocated": 0, "fragments": 0}
    for r in range(reps):
        for v in views:
            prep = rz.prepare(dev, cams[v], st)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            tg = rz.forward(prep)
            e[1].record(stream)
            rz.kernel_grads(prep, tg, ups[v])
            e[2].record(stream)
            torch.cuda.synchronize()
            fwd += e[0].elapsed_time(e[1])
            bwd += e[1].elapsed_time(e[2])
            if r == 0 and tg.frag_prim is not None:     # fragment log footprint
                pages = int(tg.frag_pool_next.item())
                slot_b = 4 + 8 + (8 if tg.frag_xy is not None else 0)
                log["pages_used"] += pages
                log["bytes_used"] += pages * rz.FRAG_PAGE * 32 * slot_b
                log["bytes_allocated"] += tg.frag_prim.numel() * slot_b
                log["fragments"] += int(tg.n_fragments.sum().item())
    n = max(len(views), 1)
    log = {k: v // n for k, v in log.items()}
    log["note"] = "per view, paged fragment log (include/qgs_b200.h qgs_targets)"
    return fwd / reps, bwd / reps, log


def run_e2e(a, rz, sc, mine, device, st, world):
    """The same step through the public API from HOST buffers: primitives
    uploaded from pinned memory, every view's upstream maps copied on a copy
    stream (the backward of view i waits for its maps), dist.gpu_step, and
    the all-reduced gradient read back to pinned memory -- all inside the
    timed region."""
    import torch.distributed as dist
    from paper_2411_16392_b200.dist import gpu_step, upload_async
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    host = type("H", (), {})()
    for f in rz.DevicePrimitives.FIELDS:
        setattr(host, f, pin(getattr(sc.prims, f)))
    ups = [{k: pin(u) for k, u in sc.upstream[v].items()} for v in mine]
    h2d = sum(getattr(host, f).numel() * 4 for f in rz.DevicePrimitives.FIELDS)
    h2d += sum(t.numel() * 4 for u in ups for t in u.values())
    out_host = None
    side = torch.cuda.Stream(device=device)

    copy = torch.cuda.Stream(device=device)
    down = torch.cuda.Stream(device=device)     # gradient read-back (the D2H copy engine)
    dev_ups = [{k: torch.empty(t.shape, dtype=t.dtype, device=device) for k, t in u.items()}
               for u in ups]
    by_view = dict(zip(mine, dev_ups))

    def step():
        nonlocal out_host
        # the SH coefficients (~3/4 of the bytes) on the copy stream: view 0
        # is binned from the geometry while they are on their way
        dev = rz.DevicePrimitives.from_host(host, device, non_blocking=True, sh_stream=copy)
        # every view's upstream maps go over on a copy stream under the raster
        evs = upload_async(ups, dev_ups, copy)
        main = torch.cuda.current_stream()

        def hook(name, i):
            if name == "fwd_end":           # view i's backward needs its maps
                main.wait_event(evs[i])
        grads = gpu_step(dev, sc.cams, by_view, st, 0, world, views=mine, side=side, hook=hook)
        if out_host is None:
            out_host = torch.empty(grads.buffer.shape, dtype=grads.buffer.dtype).pin_memory()
        # the read-back runs on its own stream so the next step's upload (the
        # H2D engine) does not queue behind it; the timed region waits for it
        down.wait_stream(main)
        with torch.cuda.stream(down):
            out_host.copy_(grads.buffer, non_blocking=True)
        grads.buffer.record_stream(down)
        return grads.buffer.numel() * 4

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    d2h = 0
    for _ in range(a.steps):
        d2h = step()
    stream.wait_stream(down)                    # the last read-back is inside the timed region
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    t_ms = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms = float(t_ms.item())
    px = len(sc.cams) * sc.cams[0].width * sc.cams[0].height
    h2d_all = torch.tensor([float(h2d)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(h2d_all)
    return {"value": px / 1e6 / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d_all.item()), "d2h_bytes_per_step": int(d2h) * world}


# ---------------------------------------------------------------- CPU side

def config_of(sc, a):
    """the workload both arms report (identical dicts)"""
    return {"workload": workload_desc(sc), "views_per_step": len(sc.cams),
            "exact_decisions": not a.fp32_decisions}


def _cpu_inputs(sc, v=0):
    prims64 = sc.prims.astype(np.float64)
    up = {k: np.asarray(x, np.float64) for k, x in sc.upstream[v].items()}
    return prims64, sc.cams[v], up


def cpu_baseline(sc):
    """The float64 oracle (C + numpy restatement of the reference, OpenMP over
    tiles for the per-pixel loops) on the host cores: ONE WHOLE VIEW of the
    workload timed end to end (prepare + forward + backward + chain), nothing
    sampled or extrapolated."""
    from oracle import qgs_oracle as qo
    prims64, cam, up = _cpu_inputs(sc)
    r = qo.time_full_view(prims64, cam, up)
    px = cam.width * cam.height
    cpu = qo.cpu_model()
    return {"value": px / 1e6 / r["seconds"], "unit": UNIT, "cores": r["threads"],
            "kind": "port", "cpu": cpu["model"], "logical_cores": cpu["logical_cores"],
            "sample": (f"view 0 of {sc.name} in full ({r['pairs']} tile pairs): prepare + "
                       f"forward + backward + chain in {r['seconds']:.1f} s"), "detail": r}


def run_reference(a):
    """Reference arm: the float64 oracle port of the reference path
    (oracle/, kind "port": the reference is Python + numba and is not on the
    GPU box) on all host threads.  One step = ONE WHOLE VIEW of the workload
    (prepare + forward + backward + chain, nothing sampled); views are timed
    until --ref-budget seconds are spent (at least one), and `steps` is the
    number actually timed, so steps x ms_per_step is the measured time."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import qgs_oracle as qo
    from paper_2411_16392_b200 import scenes
    # warm-up on C1 (library load, page-in), then whole views of the workload
    c1 = scenes.CONFIGS["c1"]()
    for _ in range(a.warmup):
        qo.time_full_view(*_cpu_inputs(c1))
    sc = scene_for(a.config)
    secs, runs = [], []
    t_start = time.perf_counter()
    while len(secs) < max(1, a.steps):
        v = len(secs) % len(sc.cams)
        r = qo.time_full_view(*_cpu_inputs(sc, v))
        secs.append(r["seconds"])
        runs.append({"view": v, "seconds": r["seconds"], "phases": r["phases"]})
        if time.perf_counter() - t_start + r["seconds"] > a.ref_budget:
            break
    cam = sc.cams[0]
    px = cam.width * cam.height
    value = px / 1e6 / float(np.mean(secs))
    cpu = qo.cpu_model()
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": len(secs), "warmup": a.warmup,
        "ms_per_step": float(np.mean(secs)) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE config shapes; scenes.py)",
        "config": config_of(sc, a),
        "step": "one whole view of the workload: prepare + forward + backward + chain",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": qo.num_threads(), "kind": "port",
                         "cpu": cpu["model"], "logical_cores": cpu["logical_cores"],
                         "sample": f"{len(secs)} whole view(s) of {sc.name}, timed in full"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "views": runs,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget", type=float, default=100.0,
                    help="reference arm: stop timing whole views after this many seconds")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fp32-decisions", action="store_true",
                    help="RenderSettings(exact_decisions=False): selection decisions in fp32 only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path on one GPU")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
