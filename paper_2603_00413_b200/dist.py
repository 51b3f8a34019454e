"""Multi-GPU data parallelism over rays.

Every pixel's ray tree is independent, so rays shard with no data-path exchange:
each rank owns the (view, tile) tiles with tile_index % world == rank, traces them
against its own replica of the mesh / LBVH (rebuilt locally every step), and the only
collective is one all-reduce(SUM) of the flat [dV | dIOR | dsigma] gradient buffer
(NCCL over NVLink 5 / NVSwitch on a B200 box; gloo on CPU for the tests).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch
import torch.distributed as dist


def tile_pixel_ids(n_views: int, W: int, H: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """Pixel ids (view*H*W + y*W + x) of this rank's tiles, cyclic over (view, tile row, tile
    col) in view-major order.  Inside a tile the pixels are ordered in 8x4 micro-tiles so a
    warp's 32 rays are a compact screen-space block (coherent traversal)."""
    assert tile % 8 == 0 and tile % 4 == 0
    tx, ty = (W + tile - 1) // tile, (H + tile - 1) // tile
    n_tiles = n_views * tx * ty
    mine = np.arange(rank, n_tiles, world, dtype=np.int64)
    view = mine // (tx * ty)
    rem = mine % (tx * ty)
    ox = (rem % tx) * tile
    oy = (rem // tx) * tile
    # offsets inside one tile: micro-tile m (8x4), lane l
    m = np.arange((tile // 8) * (tile // 4))
    l = np.arange(32)
    mx = (m % (tile // 8)) * 8
    my = (m // (tile // 8)) * 4
    dx = (mx[:, None] + (l % 8)[None, :]).ravel()
    dy = (my[:, None] + (l // 8)[None, :]).ravel()
    X = ox[:, None] + dx[None, :]
    Y = oy[:, None] + dy[None, :]
    ok = (X < W) & (Y < H)
    pid = (view[:, None] * H + Y) * W + X
    return pid[ok].astype(np.int64)


def flat_grads(gV: torch.Tensor, gior: torch.Tensor, gsig: torch.Tensor, out: Optional[torch.Tensor] = None):
    n = gV.numel() + gior.numel() + gsig.numel()
    if out is None or out.numel() != n:
        out = torch.empty(n, dtype=torch.float32, device=gV.device)
    a, b = gV.numel(), gior.numel()
    out[:a].copy_(gV.reshape(-1))
    out[a:a + b].copy_(gior.reshape(-1))
    out[a + b:].copy_(gsig.reshape(-1))
    return out


def unflat_grads(flat: torch.Tensor, gV: torch.Tensor, gior: torch.Tensor, gsig: torch.Tensor):
    a, b = gV.numel(), gior.numel()
    gV.view(-1).copy_(flat[:a])
    gior.view(-1).copy_(flat[a:a + b])
    gsig.view(-1).copy_(flat[a + b:])


def allreduce_grads(gV: torch.Tensor, gior: torch.Tensor, gsig: torch.Tensor, flat: Optional[torch.Tensor] = None,
                    group=None):
    """Sum the gradients of all ranks in place: one all-reduce of one flat buffer."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return flat
    flat = flat_grads(gV, gior, gsig, flat)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    unflat_grads(flat, gV, gior, gsig)
    return flat
