"""Which path of tile_sort_kernel each tile takes, and what its in-bucket
ranking costs (binning.cu: linear buckets over the f32 key bits that vary in
the tile, or sample-sort buckets when a linear bucket exceeds SORT_SKEW).

    python tools/sort_stats.py [--config c3] [--view 0]

Replays the kernel's bucketing decisions on the sorted keys of one view and
prints, per path: tiles, items, mean bucket occupancy seen by an item
(sum c^2 / n, the rank loop's length) and the largest bucket.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16392_b200 import rasterizer as rz, scenes  # noqa: E402

SKEW, MAXB, SMEM, HUGE = 128, 8192, 6144, 49152

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--view", type=int, default=0)
a = ap.parse_args()
sc = scenes.CONFIGS[a.config]()
dev = rz.DevicePrimitives.from_host(sc.prims)
prep = rz.prepare(dev, sc.cams[a.view])
keys = prep.sorted_keys()
torch.cuda.synchronize()
off = prep.tile_offsets.long()
cnt = off[1:] - off[:-1]
T = cnt.numel()
tile = torch.repeat_interleave(torch.arange(T, device=cnt.device), cnt)
bits = keys.view(torch.int64)
h = ((bits >> 29) - (960 << 23)) & 0xFFFFFFFF
kmin = torch.full((T,), 1 << 40, dtype=torch.int64, device=h.device).scatter_reduce(0, tile, h, "amin")
kmax = torch.zeros(T, dtype=torch.int64, device=h.device).scatter_reduce(0, tile, h, "amax")
rng = (kmax - kmin).clamp(min=0)
nb = torch.full((T,), 64, dtype=torch.int64, device=h.device)
for _ in range(8):
    nb = torch.where((nb < MAXB) & (nb * 2 < cnt), nb * 2, nb)
shift = torch.zeros(T, dtype=torch.int64, device=h.device)
for _ in range(40):
    shift = torch.where((rng >> shift) >= nb, shift + 1, shift)
b = (h - kmin[tile]) >> shift[tile]
gb = tile * MAXB + b
bc = torch.bincount(gb, minlength=T * MAXB).view(T, MAXB)
maxcnt = bc.max(1).values
skew = (maxcnt > SKEW) & (cnt >= 512)
sq = (bc.double() ** 2).sum(1)


def rep(name, m):
    n = cnt[m].sum().item()
    if n == 0:
        print(f"{name:28s} tiles 0")
        return
    print(f"{name:28s} tiles {int(m.sum()):5d}  items {n / 1e6:7.2f}M ({100 * n / cnt.sum().item():5.1f} %)"
          f"  rank len {sq[m].sum().item() / n:7.2f}  max bucket {int(maxcnt[m].max())}")


print(f"{a.config} view {a.view}: tiles {T}, pairs {int(cnt.sum())}")
big = cnt > SMEM
rep("all", cnt > 1)
rep("linear, smem-staged", (~skew) & (~big) & (cnt > 1))
rep("linear, L2-staged", (~skew) & big & (cnt <= HUGE))
rep("sample-sort (skewed)", skew)
rep("huge (> 49152)", cnt > HUGE)
# for the skewed tiles: how far does one far key stretch the range?
if skew.any():
    # share of the range that the top 1 % of keys occupy
    s = torch.nonzero(skew).flatten()[:2000]
    fr = []
    for t in s.tolist():
        hh = h[off[t]:off[t + 1]]          # sorted ascending
        n = hh.numel()
        q99 = hh[int(0.99 * (n - 1))]
        fr.append(((hh[-1] - q99).double() / max(int(hh[-1] - hh[0]), 1)).item())
    fr = torch.tensor(fr)
    print(f"skewed tiles: range share of the top 1 % of keys: median {fr.median():.3f}, "
          f"p10 {fr.quantile(0.1):.3f}, p90 {fr.quantile(0.9):.3f}")

# ---- what other first-level bucketings would give (rank length sum c^2 / n)
# over the L2-staged tiles (n > SMEM), nb buckets each as the kernel picks
m = (cnt > SMEM)
sel = m[tile]
ti, hh, kk = tile[sel], h[sel], keys[sel]
nbt = nb[ti]


def rank_len(bid):
    g = ti * MAXB + bid.clamp(0, MAXB - 1)
    c = torch.bincount(g, minlength=T * MAXB).double()
    return ((c ** 2).sum() / sel.sum()).item()


print(f"L2-staged tiles: rank length, linear in sort_h {rank_len((hh - kmin[ti]) >> shift[ti]):.2f}")
kmin_d = torch.full((T,), float('inf'), dtype=torch.float64, device=h.device).scatter_reduce(0, tile, keys, "amin")
kmax_d = torch.full((T,), -float('inf'), dtype=torch.float64, device=h.device).scatter_reduce(0, tile, keys, "amax")
lin = ((kk - kmin_d[ti]) / (kmax_d[ti] - kmin_d[ti]).clamp(min=1e-300) * (nbt - 1)).floor().long()
print(f"  linear in depth {rank_len(lin):.2f}")
# equi-depth coarse cells from a strided sample of S keys, L linear sub-buckets each
for S in (256, 1024):
    L = MAXB // S
    starts = off[:-1]
    # position of each item inside its tile (keys are sorted per tile)
    pos = torch.arange(keys.numel(), device=h.device) - starts[tile]
    # the sorted sample's splitters: key at rank floor(i * n / S), i = 1..S-1 -> for sorted
    # keys, the coarse cell of an item is the number of splitters <= its key ~ pos * S // n
    coarse = (pos[sel] * S) // cnt[ti]
    # sub-bucket linear inside the cell's key range
    cell = ti * S + coarse
    lo = torch.full((T * S,), float('inf'), dtype=torch.float64, device=h.device).scatter_reduce(0, cell, kk, "amin")
    hi = torch.full((T * S,), -float('inf'), dtype=torch.float64, device=h.device).scatter_reduce(0, cell, kk, "amax")
    sub = ((kk - lo[cell]) / (hi[cell] - lo[cell]).clamp(min=1e-300) * (L - 1)).floor().long()
    print(f"  equi-depth {S} cells x {L} linear sub-buckets {rank_len(coarse * L + sub):.2f}")
print(f"  Poisson ideal (n / nb per bucket) {(1 + cnt[m].double() / nb[m].double()).mul(cnt[m].double()).sum().item() / cnt[m].sum().item():.2f}")
