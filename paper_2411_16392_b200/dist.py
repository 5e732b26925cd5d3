"""Multi-GPU training step: camera views sharded over ranks, primitives
replicated, ONE all-reduce of the packed raw-parameter gradients per step.

SURVEY.md section 8e.  The reference is single-process (train.py:183-261
renders one view at a time); views are independent given replicated
primitives, so rank r takes views {v : v mod W == r}, accumulates its views'
raw gradients on device (rasterizer.backward(..., out=grads)), and a single
NCCL all-reduce (SUM) over NVLink makes every rank hold the full gradient.
The per-view screen-space centre gradient (a densification statistic, not a
parameter gradient, train.py:239-244) is folded per view into the
densification statistics, which are all-reduced with the gradients.

The same code runs over gloo on CPU in the tests, with the per-view backward
supplied by the caller.
"""

import numpy as np
import torch
import torch.distributed as dist

GROUPS = ("centers", "quats", "raw_scales", "raw_signs", "raw_opacity", "sh")


def shard_views(n_views, rank, world):
    """Round-robin view assignment: rank r renders views r, r+W, r+2W, ..."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return list(range(rank, n_views, world))


def group_sizes(shapes):
    return [int(np.prod(shapes[g])) for g in GROUPS]


def pack(grads, like=None):
    """Six raw-gradient groups -> one contiguous fp32 vector (all-reduce layout:
    centers, quats, raw_scales, raw_signs, raw_opacity, sh)."""
    parts = []
    for g in GROUPS:
        a = grads[g] if isinstance(grads, dict) else getattr(grads, g)
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
        parts.append(t.reshape(-1).to(torch.float32))
    flat = torch.cat(parts)
    return flat if like is None else flat.to(like.device)


def unpack(flat, shapes):
    out, o = {}, 0
    for g, n in zip(GROUPS, group_sizes(shapes)):
        out[g] = flat[o:o + n].reshape(shapes[g])
        o += n
    return out


def allreduce_(flat, group=None):
    """In-place SUM over all ranks (NCCL on GPU, gloo on CPU)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def sharded_step(n_views, view_backward, rank, world, shapes, device=None, group=None):
    """One data-parallel step.

    view_backward(v) -> dict of the six raw-gradient arrays for view v (numpy
    or torch).  Returns the all-reduced gradient as a dict of tensors; every
    rank ends with the same values."""
    flat = None
    for v in shard_views(n_views, rank, world):
        part = pack(view_backward(v))
        flat = part if flat is None else flat.add_(part)
    if flat is None:
        flat = torch.zeros(sum(group_sizes(shapes)), dtype=torch.float32)
    if device is not None:
        flat = flat.to(device)
    allreduce_(flat, group)
    return unpack(flat, shapes)


def pipelined_prepare(dev_prims, cams, views, settings, side=None):
    """Yield (i, view, PreparedView) for `views`, each ready on the current
    stream, with view i+1's preprocessing and binning launched on a side
    stream while the caller's forward/backward of view i run on the current
    one (the per-view host read of the pair count no longer drains the GPU,
    and binning overlaps the previous view's raster).  The caller must
    consume each view (launch its work) before advancing the generator."""
    from . import rasterizer as rz
    main = torch.cuda.current_stream()
    side = side if side is not None else torch.cuda.Stream(device=main.device)
    side.wait_stream(main)                  # the primitives were uploaded on main

    def launch(v):
        with torch.cuda.stream(side):
            prep = rz.prepare(dev_prims, cams[v], settings)
            ev = torch.cuda.Event()
            ev.record(side)
        return prep, ev

    nxt = launch(views[0]) if views else None
    for i, v in enumerate(views):
        prep, ev = nxt
        main.wait_event(ev)
        for t in (prep.prep, prep.tile_offsets, prep.tile_prims):
            t.record_stream(main)           # allocated on `side`, used on main
        yield i, v, prep
        nxt = launch(views[i + 1]) if i + 1 < len(views) else None


def upload_async(host_items, dev_items, copy=None):
    """Copy a list of dicts of pinned host tensors into the matching device
    tensors (allocated once by the caller) on a copy stream; returns one
    event per dict.  The caller's stream waits on event i before using dict
    i, so the transfers overlap earlier work (e.g. every view's upstream maps
    while the first views rasterize)."""
    main = torch.cuda.current_stream()
    copy = copy if copy is not None else torch.cuda.Stream(device=main.device)
    copy.wait_stream(main)                   # the previous step is done with the buffers
    evs = []
    with torch.cuda.stream(copy):
        for h, d in zip(host_items, dev_items):
            for k, t in h.items():
                d[k].copy_(t, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
            evs.append(ev)
    return evs


def gpu_step(dev_prims, cams, upstreams, settings, rank, world, grads=None, group=None,
             views=None, side=None, hook=None, counters=None, stats=None):
    """The B200 step (bench.py runs exactly this): this rank's views through
    the sm_100a rasterizer, raw gradients accumulated in one flat device
    buffer, one all-reduce (NCCL over NVLink; gloo in the tests).

    upstreams[v]: the upstream dict of view v (device tensors; a dict keyed
    by view or a list over all views).  views: this rank's views (default:
    the round-robin shard).  hook(event, i): called on the host at
    "view_begin" / "fwd_end" / "bwd_end" / "view_end" of the i-th local view
    and at "reduce_begin" / "reduce_end" (bench.py records CUDA events there).
    counters: forward work counters (rasterizer.forward).  stats: a
    densify.DensifyStats -- each view's screen-space centre gradient norm is
    folded in per view (train.py:239-244 semantics: one norm per rendered
    view), and the sums and counts are all-reduced with the gradients, so
    every rank makes the same densification decisions."""
    from . import rasterizer as rz
    hook = hook or (lambda *_: None)
    if grads is None:
        grads = rz.GradientBuffer.zeros_flat(dev_prims)
    else:
        grads.zero_()
    views = shard_views(len(cams), rank, world) if views is None else views
    for i, v, prep in pipelined_prepare(dev_prims, cams, views, settings, side):
        hook("view_begin", i)
        tg = rz.forward(prep, counters=counters)
        hook("fwd_end", i)
        kg = rz.kernel_grads(prep, tg, upstreams[v])
        hook("bwd_end", i)
        if stats is not None:
            grads.screen_center.zero_()
        rz.chain(prep, kg, grads)
        if stats is not None:
            stats.add_view(grads.screen_center)
        hook("view_end", i)
    hook("reduce_begin", len(views))
    allreduce_(grads.buffer, group)
    if stats is not None:
        stats.allreduce_(group)
    hook("reduce_end", len(views))
    return grads
