"""Data-parallel path on the GPU (a9 / SURVEY 8e): two ranks sharing cuda:0 over gloo run the
CUDA path on their tile shards; the all-reduced [dV | dIOR | dsigma] of a sharded C2 step
equals the single-process gradient (this also checks the loss_scale global-mean semantics and
that the ray-independent regulariser is added exactly once), and after several steps -- with a
periodic mesh pass run by rank 0 and broadcast -- the parameters are bitwise identical on both
ranks.  (gloo stages the reduction through host memory; on a B200 box bench.py runs the same
RefineOptimizer hook with NCCL.)"""
import dataclasses
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(pid_np, rank=0, world=1, hook=None, bcast=None, reg=False):
    from paper_2603_00413_b200 import scenes as S
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    dev = torch.device("cuda:0")
    sc = S.config_c2()
    tr = Tracer(dev)
    tgt_ds = DeviceScene(dataclasses.replace(sc, ior=1.45), dev)
    tr.build_bvh(tgt_ds.V, tgt_ds.F)
    target_full = tr.trace_forward(tgt_ds).rgb.clone()
    ds = DeviceScene(sc, dev)
    pid = None if pid_np is None else torch.as_tensor(pid_np, device=dev)
    target = target_full if pid is None else target_full[pid].contiguous()
    n_local = sc.n_pixels if pid is None else pid.numel()
    cfg = RefineConfig(freeze_iters=0, reg_every=2 if reg else 0, reg_inner=3)
    opt = RefineOptimizer(tr, ds, cfg, seed=5, grad_hook=hook, loss_scale=n_local / sc.n_pixels, rank=rank,
                          broadcast=bcast)
    masks = None
    if reg:
        tr.build_bvh(tgt_ds.V, tgt_ds.F)
        _, _, masks = tr.mask_loss(tgt_ds, torch.zeros(sc.n_pixels, device=dev), 0.0, want_mask=True)
        masks = masks.contiguous()
    return opt, target, pid, masks


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2603_00413_b200 import dist as DD
    from paper_2603_00413_b200 import scenes as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = S.config_c2()
    pid = DD.tile_pixel_ids(sc.cams.n_views, sc.cams.width, sc.cams.height, rank, world)

    def bcast(t):
        h = t.cpu()
        dist.broadcast(h, 0)
        t.copy_(h)

    opt, target, pid_t, _ = _setup(pid, rank, world, hook=lambda f: DD.allreduce_flat(f))
    opt.step(target, pid_t)
    torch.cuda.synchronize()
    g1 = opt.grads.flat.cpu().numpy().copy()
    # several steps with the periodic mesh pass (rank 0) and its broadcast
    opt2, target2, pid2, masks = _setup(pid, rank, world, hook=lambda f: DD.allreduce_flat(f), bcast=bcast, reg=True)
    for _ in range(4):
        opt2.step(target2, pid2, gt_masks=masks)
    torch.cuda.synchronize()
    q.put((rank, g1, opt2.V.cpu().numpy(), opt2.sigma.cpu().numpy(), float(opt2.ior.cpu()[0]), opt2.it))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gradient_equals_single_process_and_params_stay_identical():
    import torch.multiprocessing as mp
    from tests._parity import rel_l2
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single process, all pixels
    opt, target, pid, _ = _setup(None)
    opt.step(target, pid)
    torch.cuda.synchronize()
    ref = opt.grads.flat.cpu().numpy()
    nv = opt.V.shape[0]
    g = res[0][1]
    assert np.array_equal(res[0][1], res[1][1])                       # the all-reduce result is shared
    e_v = rel_l2(g[:3 * nv], ref[:3 * nv])
    e_i = abs(g[3 * nv] - ref[3 * nv]) / abs(ref[3 * nv])
    e_s = rel_l2(g[3 * nv + 1:], ref[3 * nv + 1:])
    assert e_v <= 1e-5 and e_i <= 1e-5 and e_s <= 1e-5, (e_v, e_i, e_s)
    # parameters after 4 steps (2 periodic mesh passes on rank 0, broadcast): bitwise identical
    a, b = res[0], res[1]
    assert a[5] == b[5] == 4
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3]) and a[4] == b[4]


def test_tile_shard_equals_pixel_list():
    """dt_cameras.tile: a cyclic tile shard and an explicit tile list trace the same
    rays in the same order as the equivalent pixel-id list -- bit-identical radiance, and the
    same gradient up to the float atomics' order."""
    from paper_2603_00413_b200 import dist as DD
    from paper_2603_00413_b200 import scenes as S
    from paper_2603_00413_b200.tracer import DeviceScene, TileShard, Tracer
    from tests._parity import rel_l2
    dev = torch.device("cuda:0")
    sc = S.config_c2(n_views=3, res=128)
    ds = DeviceScene(sc, dev)
    tr = Tracer(dev)
    tr.build_bvh(ds.V, ds.F)
    W, H, nv = sc.cams.width, sc.cams.height, sc.cams.n_views
    for rank, world in ((0, 1), (1, 3)):
        pid = torch.as_tensor(DD.tile_pixel_ids(nv, W, H, rank, world), device=dev)
        a = tr.trace_forward(ds, pid).rgb.clone()
        g = torch.as_tensor(S.upstream_grad(pid.numel(), 3), device=dev)
        gA = [t.clone() for t in tr.trace_backward(g)]
        for sh in (TileShard(32, rank, world),
                   TileShard(32, tile_ids=torch.as_tensor(DD.shard_tiles(nv, W, H, rank, world), dtype=torch.int32,
                                                          device=dev))):
            b = tr.trace_forward(ds, sh).rgb
            assert b.shape == a.shape and torch.equal(a, b)
            gB = tr.trace_backward(g)
            assert rel_l2(gB[0].cpu().numpy(), gA[0].cpu().numpy()) < 1e-5
            assert abs(float(gB[1]) - float(gA[1])) <= 1e-5 * abs(float(gA[1])) + 1e-7


def test_empty_tile_shard():
    """A rank with no tiles (more ranks than tiles, or an empty LPT list) traces zero rays and
    its backward contributes zero gradients."""
    from paper_2603_00413_b200 import scenes as S
    from paper_2603_00413_b200.tracer import DeviceScene, TileShard, Tracer
    dev = torch.device("cuda:0")
    sc = S.config_c2(n_views=1, res=64)               # 4 tiles of 32 x 32
    ds = DeviceScene(sc, dev)
    tr = Tracer(dev)
    tr.build_bvh(ds.V, ds.F)
    for sh in (TileShard(32, 5, 8), TileShard(32, tile_ids=torch.zeros(0, dtype=torch.int32, device=dev))):
        out = tr.trace_forward(ds, sh)
        assert out.rgb.shape == (0, 3)
        gV, gI, gS = tr.trace_backward(torch.zeros((0, 3), device=dev))
        assert float(gV.abs().sum()) == 0.0 and float(gI.abs().sum()) == 0.0
