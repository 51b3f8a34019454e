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


def test_flat_roundtrip():
    gV = torch.randn(10, 3)
    gi = torch.randn(1)
    gs = torch.randn(4, 4, 4, 3)
    f = DD.flat_grads(gV, gi, gs)
    a, b, c = torch.zeros_like(gV), torch.zeros_like(gi), torch.zeros_like(gs)
    DD.unflat_grads(f, a, b, c)
    assert torch.equal(a, gV) and torch.equal(b, gi) and torch.equal(c, gs)
