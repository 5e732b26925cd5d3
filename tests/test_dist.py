"""Multi-rank data-parallel step on CPU (gloo, world_size 2).

Each rank renders its shard of the views through the float64 oracle as the
per-view backward, the packed raw gradients are all-reduced once, and every
rank must end with exactly the single-process sum over all views.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_16392_b200 import dist as qd


def test_shard_views_partition():
    for world in (1, 2, 3, 4, 8):
        got = sorted(v for r in range(world) for v in qd.shard_views(10, r, world))
        assert got == list(range(10))
        assert all(len(qd.shard_views(10, r, world)) in (10 // world, 10 // world + 1)
                   for r in range(world))
    with pytest.raises(ValueError):
        qd.shard_views(4, 2, 2)


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    shapes = {"centers": (5, 3), "quats": (5, 4), "raw_scales": (5, 3), "raw_signs": (5, 3),
              "raw_opacity": (5,), "sh": (5, 3, 4)}
    g = {k: rng.normal(size=s).astype(np.float32) for k, s in shapes.items()}
    back = qd.unpack(qd.pack(g), shapes)
    for k in shapes:
        assert np.array_equal(back[k].numpy(), g[k])


def _scene():
    from paper_2411_16392_b200 import scenes
    sc = scenes.config1(seed=11, n=96, res=32)
    # four views of the same primitives
    cams = [scenes.pinhole(32, 32, e) for e in 3.0 * np.array(
        [[1, 0, 0.2], [0, 1, 0.3], [-1, 0.2, 0.1], [0.3, -1, 0.4]]) / 1.05]
    rng = np.random.default_rng(5)
    ups = [{"color": rng.normal(size=(32, 32, 3)), "alpha": rng.normal(size=(32, 32)),
            "depth": rng.normal(size=(32, 32)), "normal": rng.normal(size=(32, 32, 3))}
           for _ in cams]
    return sc.prims.astype(np.float64), cams, ups


def _view_backward(prims, cams, ups):
    from oracle import qgs_oracle as qo

    def f(v):
        vw = qo.prepare(prims, cams[v])
        return qo.backward(vw, qo.forward(vw), ups[v])
    return f


def _shapes(prims):
    return {g: tuple(np.shape(getattr(prims, g))) for g in qd.GROUPS}


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prims, cams, ups = _scene()
    g = qd.sharded_step(len(cams), _view_backward(prims, cams, ups), rank, world, _shapes(prims))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **{k: v.numpy() for k, v in g.items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_two_rank_allreduce_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    prims, cams, ups = _scene()
    ref = qd.sharded_step(len(cams), _view_backward(prims, cams, ups), 0, 1, _shapes(prims))
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    for k in qd.GROUPS:
        assert np.array_equal(r0[k], r1[k]), k            # identical on every rank
        assert np.allclose(r0[k], ref[k].numpy(), rtol=1e-5, atol=1e-6), k
    # the gradient is non-trivial and every view contributed
    assert np.abs(r0["sh"]).max() > 0


def test_single_rank_without_process_group():
    prims, cams, ups = _scene()
    g = qd.sharded_step(len(cams), _view_backward(prims, cams, ups), 0, 1, _shapes(prims))
    assert g["centers"].shape == (96, 3)


@pytest.mark.gpu
def test_upload_async_and_pipelined_prepare(cuda_device):
    """the e2e helpers: upstream maps copied on a copy stream land intact
    before the backward that waits on their event, and the pipelined
    prepare yields the same binning as the plain one"""
    import numpy as np
    import torch
    from paper_2411_16392_b200 import dist as D, rasterizer as rz, scenes
    sc = scenes.config2(seed=3, n=3000, res=96, views=3)
    dev = rz.DevicePrimitives.from_host(sc.prims)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    host = [{k: pin(v) for k, v in sc.upstream[i].items()} for i in range(3)]
    dst = [{k: torch.empty(t.shape, dtype=t.dtype, device=cuda_device) for k, t in h.items()}
           for h in host]
    evs = D.upload_async(host, dst)
    main = torch.cuda.current_stream()
    st = rz.RenderSettings()
    for i, v, prep in D.pipelined_prepare(dev, sc.cams, [0, 1, 2], st):
        ref = rz.prepare(dev, sc.cams[v], st)
        assert torch.equal(prep.tile_prims, ref.tile_prims)
        main.wait_event(evs[i])
        for k, t in host[i].items():
            assert torch.equal(dst[i][k].cpu(), t), k


@pytest.mark.gpu
def test_deferred_sh_upload_prepare_is_identical(cuda_device):
    """SH coefficients still in flight on a copy stream: prepare() bins the
    view from the geometry (qgs_preprocess_geometry) and adds the colour when
    they land (qgs_preprocess_color) -- the prepared state, the sort and the
    images are bit-identical to the one-kernel qgs_preprocess"""
    import numpy as np
    import torch
    from paper_2411_16392_b200 import rasterizer as rz, scenes
    sc = scenes.config2(seed=5, n=4000, res=96, views=2)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    host = type("H", (), {f: pin(getattr(sc.prims, f)) for f in rz.DevicePrimitives.FIELDS})()
    st = rz.RenderSettings()
    ref_dev = rz.DevicePrimitives.from_host(sc.prims)
    copy = torch.cuda.Stream()
    for v in range(2):
        with torch.cuda.stream(copy):
            torch.cuda._sleep(200_000_000)      # keep the SH copy pending at prepare()
        dev = rz.DevicePrimitives.from_host(host, cuda_device, non_blocking=True, sh_stream=copy)
        assert dev.sh_ready is not None and not dev.sh_ready.query()
        prep = rz.prepare(dev, sc.cams[v], st)
        ref = rz.prepare(ref_dev, sc.cams[v], st)
        P = len(ref_dev)
        a256 = lambda n: (n + 255) // 256 * 256  # noqa: E731  (qgs_common.cuh prep_view)
        o = 0
        for size in (256 * P, 128 * P, 32 * P, 16 * P, 4 * P, 8 * (P + 1)):
            # Geo64, PrimRec, ConicRec, boxes, tile counts, pair offsets
            assert torch.equal(prep.prep[o:o + size], ref.prep[o:o + size]), o
            o += a256(size)
        assert torch.equal(prep.tile_offsets, ref.tile_offsets)
        assert torch.equal(prep.tile_prims, ref.tile_prims)
        a, b = rz.forward(prep), rz.forward(ref)
        assert torch.equal(a.color, b.color) and torch.equal(a.alpha, b.alpha)


# ------------------------------------------------ densification statistics

def _stats_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_16392_b200.densify import DensifyStats
    sc_views = _screen_views()
    st = DensifyStats(7, device=torch.device("cpu"))
    for v in qd.shard_views(len(sc_views), rank, world):
        st.add_view(sc_views[v])
    st.allreduce_()
    np.savez(os.path.join(out_dir, f"stats{rank}.npz"), accum=st.grad_accum.numpy(),
             count=st.grad_count.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _screen_views():
    rng = np.random.default_rng(9)
    out = []
    for v in range(5):
        sc = rng.normal(size=(7, 2))
        sc[rng.random(7) < 0.4] = 0.0           # unseen primitives in this view
        out.append(torch.from_numpy(sc.astype(np.float32)))
    return out


@pytest.mark.timeout(300)
def test_densify_stats_allreduce_matches_single_process(tmp_path):
    """each rank folds ONE norm per rendered view (train.py:239-243)
    and the sums / counts are all-reduced, so every rank makes the same
    densification plan as one process rendering all the views."""
    from paper_2411_16392_b200.densify import DensifyStats
    world = 2
    mp.spawn(_stats_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ref = DensifyStats(7, device=torch.device("cpu"))
    acc = np.zeros(7)
    cnt = np.zeros(7)
    for sc in _screen_views():
        ref.add_view(sc)
        g = np.linalg.norm(sc.numpy().astype(np.float64), axis=1)   # train.py:239-243
        acc[g > 0] += g[g > 0]
        cnt[g > 0] += 1
    assert np.allclose(ref.grad_accum.numpy(), acc, rtol=1e-12)
    assert np.array_equal(ref.grad_count.numpy(), cnt)
    for r in range(world):
        d = np.load(tmp_path / f"stats{r}.npz")
        assert np.allclose(d["accum"], acc, rtol=1e-12), r
        assert np.array_equal(d["count"], cnt), r


# ------------------------------------- the CUDA step over two ranks (gloo)

def _gpu_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_16392_b200 import rasterizer as rz, scenes
    from paper_2411_16392_b200.densify import DensifyStats
    sc = scenes.config2(seed=3, n=4000, res=96, views=4)
    dev = rz.DevicePrimitives.from_host(sc.prims)
    ups = {v: {k: torch.from_numpy(np.ascontiguousarray(a)).cuda() for k, a in sc.upstream[v].items()}
           for v in range(4)}
    stats = DensifyStats(len(dev))
    g = qd.gpu_step(dev, sc.cams, ups, rz.RenderSettings(), rank, world, stats=stats)
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"gpu{rank}.npz"), flat=g.buffer.cpu().numpy(),
             accum=stats.grad_accum.cpu().numpy(), count=stats.grad_count.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_rank_cuda_step_matches_single_process(tmp_path, cuda_device):
    """dist.gpu_step with the sm_100a rasterizer on two ranks (gloo, both on
    cuda:0): every rank ends with the single-process sum over all four views
    (to fp32-atomic reordering), and the same densification statistics."""
    from paper_2411_16392_b200 import rasterizer as rz, scenes
    from paper_2411_16392_b200.densify import DensifyStats
    world = 2
    mp.spawn(_gpu_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sc = scenes.config2(seed=3, n=4000, res=96, views=4)
    dev = rz.DevicePrimitives.from_host(sc.prims)
    ups = {v: {k: torch.from_numpy(np.ascontiguousarray(a)).cuda() for k, a in sc.upstream[v].items()}
           for v in range(4)}
    stats = DensifyStats(len(dev))
    ref = qd.gpu_step(dev, sc.cams, ups, rz.RenderSettings(), 0, 1, stats=stats)
    ref_flat = ref.buffer.cpu().numpy()
    scale = np.abs(ref_flat).max()
    assert scale > 0
    r = [np.load(tmp_path / f"gpu{k}.npz") for k in range(world)]
    assert np.array_equal(r[0]["flat"], r[1]["flat"])          # identical on every rank
    assert np.allclose(r[0]["flat"], ref_flat, rtol=1e-4, atol=1e-6 * scale)
    for k in range(world):
        assert np.array_equal(r[k]["count"], stats.grad_count.cpu().numpy())
        assert np.allclose(r[k]["accum"], stats.grad_accum.cpu().numpy(), rtol=1e-5, atol=1e-9)
