"""Multi-GPU data parallelism over rays.

Every pixel's ray tree is independent, so rays shard with no data-path exchange: each rank
owns a set of (view, 32x32 tile) tiles, traces them against its own replica of the mesh /
LBVH (rebuilt locally every step), and the only collective is one all-reduce(SUM) of the
flat [dV | dIOR | dsigma] gradient buffer (NCCL over NVLink 5 / NVSwitch on a B200 box;
gloo on CPU for the tests).

Tile assignment: cyclic over (view, tile row, tile col) by default; `lpt_assign` balances
the tiles by the previous step's per-tile traced-segment counts (greedy longest processing
time first) when the cyclic split is uneven.
"""
from __future__ import annotations

import heapq
from typing import Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def tile_grid(W: int, H: int, tile: int = 32):
    """Tiles per row and per column of one view."""
    return (W + tile - 1) // tile, (H + tile - 1) // tile


def cyclic_tiles(n_views: int, W: int, H: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """Global tile ids (view-major, then tile row, then tile col) of this rank: id % world == rank."""
    tx, ty = tile_grid(W, H, tile)
    return np.arange(rank, n_views * tx * ty, world, dtype=np.int64)


def tiles_pixel_ids(tiles: np.ndarray, W: int, H: int, tile: int = 32) -> np.ndarray:
    """Pixel ids (view*H*W + y*W + x) of the given tiles, tile by tile; inside a tile the pixels
    are ordered in 8x4 micro-tiles so a warp's 32 rays are a compact screen-space block
    (coherent traversal).  Pixels outside the image (ragged last tiles) are dropped."""
    assert tile % 8 == 0 and tile % 4 == 0
    tiles = np.asarray(tiles, np.int64)
    tx, ty = tile_grid(W, H, tile)
    view = tiles // (tx * ty)
    rem = tiles % (tx * ty)
    ox = (rem % tx) * tile
    oy = (rem // tx) * tile
    m = np.arange((tile // 8) * (tile // 4))
    lane = np.arange(32)
    mx = (m % (tile // 8)) * 8
    my = (m // (tile // 8)) * 4
    dx = (mx[:, None] + (lane % 8)[None, :]).ravel()
    dy = (my[:, None] + (lane // 8)[None, :]).ravel()
    X = ox[:, None] + dx[None, :]
    Y = oy[:, None] + dy[None, :]
    ok = (X < W) & (Y < H)
    pid = (view[:, None] * H + Y) * W + X
    return pid[ok].astype(np.int64)


def tile_pixel_ids(n_views: int, W: int, H: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """Pixel ids of this rank's cyclic tile share (see cyclic_tiles / tiles_pixel_ids)."""
    return tiles_pixel_ids(cyclic_tiles(n_views, W, H, rank, world, tile), W, H, tile)


def tile_costs(pixel_ids: np.ndarray, seg_count: np.ndarray, n_views: int, W: int, H: int,
               tile: int = 32) -> np.ndarray:
    """Per-tile cost (traced segments) from per-ray segment counts (dt_trace_opts.seg_count)
    of the rays pixel_ids: float64 [n_views * tiles per view], zero for tiles not covered."""
    tx, ty = tile_grid(W, H, tile)
    pid = np.asarray(pixel_ids, np.int64)
    view = pid // (W * H)
    rem = pid % (W * H)
    t = view * (tx * ty) + ((rem // W) // tile) * tx + (rem % W) // tile
    return np.bincount(t, weights=np.asarray(seg_count, np.float64), minlength=n_views * tx * ty)


def shard_tiles(n_views: int, W: int, H: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """The global tile ids of the cyclic tile shard (rank, world) in ray order (TileShard)."""
    return cyclic_tiles(n_views, W, H, rank, world, tile)


def shard_tile_costs(tiles: np.ndarray, seg_count: np.ndarray, n_tiles_total: int, tile: int = 32) -> np.ndarray:
    """Per-tile cost from per-ray segment counts of a TileShard forward (rays tile by tile,
    tile^2 per tile): float64 [n_tiles_total], zero for tiles of other shards."""
    seg = np.asarray(seg_count, np.float64).reshape(len(tiles), tile * tile).sum(1)
    out = np.zeros(n_tiles_total, np.float64)
    out[np.asarray(tiles, np.int64)] = seg
    return out


def lpt_assign(costs: Sequence[float], world: int) -> list:
    """Greedy longest-processing-time assignment: tiles in decreasing cost order, each to the
    currently least-loaded rank (ties: lowest rank; equal costs: lowest tile id first).  Returns
    one sorted int64 array of tile ids per rank.  Makespan <= (4/3 - 1/(3 world)) x optimal
    (Graham 1969)."""
    costs = np.asarray(costs, np.float64)
    order = np.lexsort((np.arange(len(costs)), -costs))      # cost descending, then id ascending
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for t in order:
        load, r = heapq.heappop(heap)
        out[r].append(int(t))
        heapq.heappush(heap, (load + float(costs[t]), r))
    return [np.array(sorted(x), np.int64) for x in out]


class GradBuffer:
    """One persistent flat fp32 buffer [dV (3 nv) | dIOR (1) | dsigma]; gV / gI / gS are views
    into it, so the backward writes the gradients in place and the all-reduce needs no copy."""

    def __init__(self, nv: int, sigma_shape, device):
        n_sig = int(np.prod(sigma_shape))
        self.flat = torch.zeros(3 * nv + 1 + n_sig, dtype=torch.float32, device=device)
        self.gV = self.flat[:3 * nv].view(nv, 3)
        self.gI = self.flat[3 * nv:3 * nv + 1]
        self.gS = self.flat[3 * nv + 1:].view(tuple(sigma_shape))


def allreduce_flat(flat: torch.Tensor, group=None, async_op: bool = False):
    """Sum `flat` over the ranks in place: one all-reduce.  NCCL runs it on its own stream (the
    caller's stream waits on the returned work, or at once when async_op is False); gloo
    reduces a host copy (functional tests on one GPU)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    if flat.is_cuda and dist.get_backend(group) == "gloo":
        host = flat.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        flat.copy_(host)
        return None
    return dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def allreduce_grads(gV: torch.Tensor, gior: torch.Tensor, gsig: torch.Tensor, flat: Optional[torch.Tensor] = None,
                    group=None):
    """Sum separately allocated gradients of all ranks in place (one all-reduce of one flat
    buffer; `flat` is reused when it has the right size).  RefineOptimizer instead keeps its
    gradients in a GradBuffer and all-reduces that directly."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return flat
    n = gV.numel() + gior.numel() + gsig.numel()
    if flat is None or flat.numel() != n:
        flat = torch.empty(n, dtype=torch.float32, device=gV.device)
    a, b = gV.numel(), gior.numel()
    flat[:a].copy_(gV.reshape(-1))
    flat[a:a + b].copy_(gior.reshape(-1))
    flat[a + b:].copy_(gsig.reshape(-1))
    allreduce_flat(flat, group)
    gV.view(-1).copy_(flat[:a])
    gior.view(-1).copy_(flat[a:a + b])
    gsig.view(-1).copy_(flat[a + b:])
    return flat
