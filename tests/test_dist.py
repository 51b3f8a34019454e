"""Multi-rank path on CPU (gloo, world size 2): tile sharding covers every pixel exactly once,
and the per-rank gradients summed by the all-reduce equal the single-process gradient.
The per-rank compute here is the oracle (test infrastructure); on a GPU box the same
dist.py code runs with NCCL around libdifftrans."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_00413_b200 import dist as DD
from paper_2603_00413_b200 import scenes as S


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("W,H", [(64, 64), (100, 37), (256, 256)])
def test_tiles_partition_all_pixels(world, W, H):
    nv = 3
    parts = [DD.tile_pixel_ids(nv, W, H, r, world) for r in range(world)]
    allp = np.concatenate(parts)
    assert len(allp) == nv * W * H
    assert np.array_equal(np.sort(allp), np.arange(nv * W * H))
    if world > 1 and W * H >= 4096:
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 32 * 32 * nv        # balanced to within a tile per view


def test_tiles_warp_coherent():
    pid = DD.tile_pixel_ids(1, 64, 64, 0, 1)
    y, x = np.divmod(pid[:32], 64)
    assert x.max() - x.min() == 7 and y.max() - y.min() == 3   # first warp = one 8x4 block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = S.config_c1()
    pid = DD.tile_pixel_ids(1, sc.cams.width, sc.cams.height, rank, world, tile=16)
    g = S.upstream_grad(sc.n_pixels, 3)[pid]
    gV, gi, gs = O.backward(O.OracleScene(sc), g, pid, nthreads=2)
    gV = torch.as_tensor(gV, dtype=torch.float32)
    gi = torch.tensor([gi], dtype=torch.float32)
    gs = torch.as_tensor(gs, dtype=torch.float32)
    DD.allreduce_grads(gV, gi, gs)
    if rank == 0:
        out.put((gV.numpy(), float(gi[0]), gs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_allreduce_equals_single_process():
    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gV, gi, gs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = S.config_c1()
    pid = np.arange(sc.n_pixels)
    rV, ri, rs = O.backward(O.OracleScene(sc), S.upstream_grad(sc.n_pixels, 3), pid)
    assert np.linalg.norm(gV - rV) / np.linalg.norm(rV) < 1e-6
    assert abs(gi - ri) < 1e-5 * max(1.0, abs(ri))
    assert np.abs(gs - rs).max() < 1e-4 * max(1.0, np.abs(rs).max())


def test_grad_buffer_views_and_allreduce_grads_roundtrip():
    buf = DD.GradBuffer(10, (4, 4, 4, 3), "cpu")
    buf.gV.copy_(torch.randn(10, 3))
    buf.gI.fill_(2.5)
    buf.gS.copy_(torch.randn(4, 4, 4, 3))
    assert buf.flat.numel() == 30 + 1 + 192
    assert torch.equal(buf.flat[:30], buf.gV.reshape(-1)) and float(buf.flat[30]) == 2.5
    assert torch.equal(buf.flat[31:], buf.gS.reshape(-1))
    # without a process group allreduce_grads is the identity
    gV, gi, gs = buf.gV.clone(), buf.gI.clone(), buf.gS.clone()
    DD.allreduce_grads(gV, gi, gs)
    assert torch.equal(gV, buf.gV) and torch.equal(gi, buf.gI) and torch.equal(gs, buf.gS)


def test_lpt_assign_properties():
    """Greedy LPT: a partition of the tiles; loads within the largest tile of
    each other and of the mean; the known optimum on a small case; a cyclic split of skewed
    costs is worse."""
    g = np.random.default_rng(3)
    for world in (1, 2, 3, 8):
        costs = g.pareto(1.5, size=500) * 100
        parts = DD.lpt_assign(costs, world)
        allt = np.concatenate(parts)
        assert np.array_equal(np.sort(allt), np.arange(500))
        loads = np.array([costs[p].sum() for p in parts])
        assert loads.max() - loads.min() <= costs.max() + 1e-9
        # greedy list scheduling: makespan <= mean load + largest job (and >= the mean load)
        assert costs.sum() / world - 1e-9 <= loads.max() <= costs.sum() / world + costs.max() + 1e-9
    # exact small cases: {7,6,5,4,3,2} on 2 ranks -> 14 / 13 (optimum 14 / 13); ties to lowest rank
    parts = DD.lpt_assign([7, 6, 5, 4, 3, 2], 2)
    assert [sorted(p.tolist()) for p in parts] == [[0, 3, 4], [1, 2, 5]]
    # skewed costs: one heavy view -- cyclic splits it unevenly, LPT balances it
    costs = np.ones(64)
    costs[:16] = 20.0
    cyc = [costs[np.arange(r, 64, 3)].sum() for r in range(3)]
    lpt = [costs[p].sum() for p in DD.lpt_assign(costs, 3)]
    assert max(lpt) < max(cyc) and max(lpt) - min(lpt) <= 20.0


def test_tile_costs_and_tiles_pixel_ids():
    n_views, W, H = 2, 70, 40
    tx, ty = DD.tile_grid(W, H)
    pid = DD.tiles_pixel_ids(np.arange(n_views * tx * ty), W, H)
    assert np.array_equal(np.sort(pid), np.arange(n_views * W * H))
    seg = (pid % 7).astype(np.int32)
    costs = DD.tile_costs(pid, seg, n_views, W, H)
    assert costs.shape == (n_views * tx * ty,) and costs.sum() == seg.sum()
    # tile 0 of view 1: pixels x < 32, y < 32 of view 1
    v1 = np.arange(W * H, 2 * W * H)
    y, x = np.divmod(v1 - W * H, W)
    m = (x < 32) & (y < 32)
    assert costs[tx * ty] == (v1[m] % 7).sum()
    # an LPT split's pixel lists partition the image
    parts = DD.lpt_assign(costs, 3)
    allp = np.concatenate([DD.tiles_pixel_ids(p, W, H) for p in parts])
    assert np.array_equal(np.sort(allp), np.arange(n_views * W * H))


def test_tile_shard_order_and_costs():
    """TileShard (dt_cameras.tile): the cyclic shard's tiles and ray count match the pixel-id
    path's, and per-ray segment counts fold back into per-tile costs."""
    from paper_2603_00413_b200.tracer import TileShard
    n_views, W, H, world = 3, 64, 96, 4
    total = n_views * (W // 32) * (H // 32)
    for r in range(world):
        sh = TileShard(32, r, world)
        tiles = DD.shard_tiles(n_views, W, H, r, world)
        assert sh.n_tiles(n_views, W, H) == len(tiles)
        assert sh.n_rays(n_views, W, H) == len(DD.tile_pixel_ids(n_views, W, H, r, world))
        seg = np.arange(len(tiles) * 1024) % 7
        c = DD.shard_tile_costs(tiles, seg, total)
        assert c.sum() == seg.sum() and np.all(c[np.setdiff1d(np.arange(total), tiles)] == 0)
        np.testing.assert_array_equal(
            c, DD.tile_costs(DD.tile_pixel_ids(n_views, W, H, r, world), seg, n_views, W, H))
