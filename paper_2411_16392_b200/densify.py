"""Densification on the device: the clone / split / prune pass and the
opacity reset of the reference trainer (train.py:263-335), over a
``DevicePrimitives`` and an ``optim.Adam``.

``densify_and_prune`` runs two library calls (csrc/optim.cu): a plan that
makes every decision on the device -- mean screen-gradient threshold, the
top-``room`` selection by (-mean, index) when the primitive budget binds,
split vs clone by the in-plane scale, the opacity prune -- and scans the
ordered compaction offsets; and an apply that writes [survivors | clones |
split + | split -] with their Adam state in one pass.  The host reads one
int64 (the output size) between the two to allocate the new arrays.
"""

from dataclasses import dataclass

import torch

from . import _lib
from .optim import GROUPS, Adam, groups_struct, params_struct
from .rasterizer import DevicePrimitives, _ptr, _stream


@dataclass
class DensifyConfig:
    """config.py:24-43 (the densification fields)."""
    densify_grad_threshold: float = 0.3
    percent_dense: float = 0.001
    prune_opacity: float = 0.005
    clone_nudge: float = 0.5
    max_primitives: int = 2000

    def struct(self, extent):
        c = _lib.DensifyConfig()
        c.grad_threshold = float(self.densify_grad_threshold)
        c.percent_dense = float(self.percent_dense)
        c.scene_extent = float(extent)
        c.prune_opacity = float(self.prune_opacity)
        c.clone_nudge = float(self.clone_nudge)
        c.max_primitives = int(self.max_primitives)
        return c


class DensifyStats:
    """train.py:263-267: per-primitive screen-gradient sums and counts and the
    accumulated centre gradient (fp64, device)."""

    def __init__(self, n, device=None):
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.grad_accum = torch.zeros((n,), dtype=torch.float64, device=device)
        self.grad_count = torch.zeros((n,), dtype=torch.float64, device=device)
        self.center_accum = torch.zeros((n, 3), dtype=torch.float64, device=device)

    def struct(self):
        s = _lib.DensifyStats()
        s.grad_accum, s.grad_count = _ptr(self.grad_accum), _ptr(self.grad_count)
        s.center_accum = _ptr(self.center_accum)
        return s

    def reset(self, n):
        self.__init__(n, self.grad_accum.device)

    def add_view(self, screen_center):
        """Fold one rendered view's screen-space centre gradient (P, 2) in:
        train.py:239-243 (norm, seen = norm > 0, accum += norm, count += 1).
        For several views per step (dist.gpu_step) call once per view."""
        g = torch.linalg.vector_norm(screen_center.to(torch.float64), dim=1)
        self.grad_accum += g
        self.grad_count += (g > 0).to(torch.float64)

    def add_centers(self, centers_grad):
        """train.py:244: center_accum += grads.centers"""
        self.center_accum += centers_grad.to(torch.float64)

    def allreduce_(self, group=None):
        """Sum the per-rank sums and counts (every rank then holds the
        statistics of all views and makes the same densification plan)."""
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            flat = torch.cat([self.grad_accum, self.grad_count])
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
            n = self.grad_accum.numel()
            self.grad_accum.copy_(flat[:n])
            self.grad_count.copy_(flat[n:])
        return self


_WS = {}


def densify_and_prune(prims: DevicePrimitives, opt: Adam, stats: DensifyStats,
                      cfg: DensifyConfig, extent):
    """train.py:269-330.  Returns the new DevicePrimitives; ``opt``'s moments
    are replaced by the compacted ones and ``stats`` is reset."""
    L = _lib.load()
    P = len(prims)
    dev = prims.centers.device
    n = int(L.qgs_densify_workspace_bytes(P))
    ws = _WS.get(dev.index)
    if ws is None or ws.numel() < n:
        ws = torch.empty((n,), dtype=torch.uint8, device=dev)
        _WS[dev.index] = ws
    counts = torch.zeros((4,), dtype=torch.int64, device=dev)
    c = cfg.struct(extent)
    st = stats.struct()
    _lib.check(L.qgs_densify_plan(prims.params_struct(), st, c, _ptr(ws), ws.numel(),
                                  _ptr(counts), _stream()), "qgs_densify_plan")
    n_out = int(counts[0].item())
    shapes = {g: (n_out,) + tuple(getattr(prims, g).shape[1:]) for g in GROUPS}
    out = {g: torch.empty(shapes[g], dtype=torch.float32, device=dev) for g in GROUPS}
    om = {g: torch.empty(shapes[g], dtype=torch.float32, device=dev) for g in GROUPS}
    ov = {g: torch.empty(shapes[g], dtype=torch.float32, device=dev) for g in GROUPS}
    kc = prims.sh_coeffs
    _lib.check(L.qgs_densify_apply(prims.params_struct(), params_struct(opt.m), params_struct(opt.v),
                                   st, c, _ptr(ws), groups_struct(out, n_out, kc),
                                   groups_struct(om, n_out, kc), groups_struct(ov, n_out, kc),
                                   _stream()), "qgs_densify_apply")
    opt.m, opt.v = om, ov
    stats.reset(n_out)
    return DevicePrimitives(**out)


def reset_opacity(prims: DevicePrimitives, opt: Adam, cap=0.01):
    """train.py:332-335: opacities above `cap` drop to it; the opacity
    group's Adam state is zeroed."""
    _lib.check(_lib.load().qgs_reset_opacity(groups_struct(prims), groups_struct(opt.m),
                                             groups_struct(opt.v), float(cap), _stream()),
               "qgs_reset_opacity")
