"""Integration: the device pieces compose into the reference's training
iteration (train.py:183-262) -- prepare, forward, the fused loss block
(losses.accumulate_upstream), backward into raw-parameter gradients, Adam
with the densification statistics, then one densify_and_prune -- all on one
GPU, no host round trip except the loss read for the check.  The photometric
loss against a target rendered from perturbed primitives must fall.
"""

import numpy as np
import pytest


@pytest.mark.gpu
def test_training_iterations_reduce_the_loss(cuda_device):
    import torch
    from paper_2411_16392_b200 import densify, losses, optim, rasterizer as rz, scenes
    sc = scenes.config1(n=2048, res=128)
    cam = sc.cams[0]
    target = rz.DevicePrimitives.from_host(sc.prims)
    gt = rz.forward(rz.prepare(target, cam)).color.clone()
    # start from perturbed colours and opacities
    start = rz.DevicePrimitives.from_host(sc.prims)
    g = torch.Generator(device="cuda").manual_seed(0)
    start.sh.add_(0.3 * torch.randn(start.sh.shape, device="cuda", generator=g))
    start.raw_opacity.add_(0.5 * torch.randn(start.raw_opacity.shape, device="cuda", generator=g))
    prims = start
    opt = optim.Adam(prims)
    stats = densify.DensifyStats(len(prims))
    w = losses.LossWeights(lambda_d=0.0, lambda_n=0.0)       # photometric only
    lrs = {"centers": 1e-5, "quats": 1e-4, "raw_scales": 1e-4, "raw_signs": 1e-4,
           "raw_opacity": 0.05, "sh": 0.02}
    hist = []
    for it in range(25):
        prep = rz.prepare(prims, cam)
        tg = rz.forward(prep)
        up = rz.zero_upstream(cam)
        parts = losses.accumulate_upstream(tg, gt, cam, up, w, use_distortion=False,
                                           use_normal=False)
        grads = rz.backward(prep, tg, up)
        opt.step(prims, grads, lrs, stats=stats)
        hist.append(float(parts[0].item()))
    assert np.all(np.isfinite(hist))
    assert hist[-1] < 0.7 * hist[0], hist
    # statistics accumulated for every primitive seen; a densification pass
    # keeps the set well formed and the step still runs afterwards
    assert float(stats.grad_count.max()) == 25.0
    cfg = densify.DensifyConfig(densify_grad_threshold=float(np.median(
        (stats.grad_accum / stats.grad_count.clamp(min=1)).cpu().numpy())),
        percent_dense=0.01, max_primitives=len(prims) + 300)
    p2 = densify.densify_and_prune(prims, opt, stats, cfg, extent=2.0)
    assert 0 < len(p2) <= len(prims) + 300        # the budget binds (half the set qualifies)
    assert opt.m["sh"].shape[0] == len(p2)
    prep = rz.prepare(p2, cam)
    tg = rz.forward(prep)
    up = rz.zero_upstream(cam)
    losses.accumulate_upstream(tg, gt, cam, up, w, use_distortion=False, use_normal=False)
    opt.step(p2, rz.backward(prep, tg, up), lrs, stats=stats)
    torch.cuda.synchronize()
    assert all(torch.isfinite(getattr(p2, f)).all() for f in optim.GROUPS)
