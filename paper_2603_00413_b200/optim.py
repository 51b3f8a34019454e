"""The refine-stage optimisation loop around the tracer.

One iteration, every arithmetic step in libdifftrans kernels:
  dt_build_bvh -> dt_trace_forward -> dt_loss_rt (L_color + L_tone)
  -> dt_trace_backward -> dt_sigma_regularizers (L_mat-smooth, L_vol)
  -> dt_adam_step on sigma ("material", lr 3e-3), IoR (lr 1e-4 while the geometry is
     frozen, then 1e-3) and, after the first k iterations, the vertices (AdamUniform, lr 1e-3).
Every reg_every iterations of the joint stage (given ground-truth masks) the periodic mesh pass
 runs reg_inner AdamUniform steps on L_mask + L_edge + L_lap (dt_mask_loss,
dt_mesh_regularizers).
Adam: beta = (0.9, 0.999), weight decay 1e-6.  Loss weights lambda_1 = 1,
lambda_2 = 0.001, lambda_4 = 0.0005; lambda_3 is not given by the paper (SPEC
default 0.01).  The IoR stays in [1, 3] and sigma >= 0 (projection after each update).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import torch

from . import _native as N
from .dist import GradBuffer
from .tracer import DeviceScene, Tracer


@dataclass
class RefineConfig:
    freeze_iters: int = 300                 # k, P:513-525 ("k = 300 / 500 / 1000")
    lr_material: float = 3e-3
    lr_ior_frozen: float = 1e-4
    lr_ior: float = 1e-3                    # P:527 (after the freeze-geometry stage)
    lr_vertices: float = 1e-3               # P:527, AdamUniform
    betas: tuple = (0.9, 0.999)
    weight_decay: float = 1e-6
    eps: float = 1e-8
    lambda_color: float = 1.0               # lambda_1
    lambda_tone: float = 0.001              # lambda_2
    lambda_smooth: float = 0.01             # lambda_3: unstated in the paper (SPEC default)
    lambda_vol: float = 0.0005              # lambda_4
    n_reg_points: int = 4096
    reg_sigma_perturb: float = 0.02         # xi ~ N(0, s^2) as a fraction of the sigma box
    ior_range: tuple = (1.0, 3.0)
    # periodic mesh regularisation (NEXT-4): every reg_every iterations of the
    # joint stage, reg_inner AdamUniform steps on the vertices of
    # lambda_mask L_mask + lambda_edge L_edge + lambda_lap L_lap (weights unstated: R33)
    reg_every: int = 100
    reg_inner: int = 200
    lambda_mask: float = 1.0
    lambda_edge: float = 0.01
    lambda_lap: float = 1.0


@dataclass
class StepResult:
    loss: torch.Tensor                      # [4] device: L_color, L_tone, L_mat-smooth, L_vol
    ior: torch.Tensor                       # [1] device: the IoR after this step's update


class HostTargets:
    """Double-buffered asynchronous upload of per-step targets from pinned host memory: the
    copy of step i+1's target runs on a side stream (copy engine) while step i computes.

        up = HostTargets(shape, device)
        k = up.upload(host)                   # step 0's target
        for i in range(n):
            tgt = up.get(k)                   # current stream waits for that copy
            k_next = up.upload(host_next)     # overlaps with the step below
            opt.step(tgt); up.release(k)
            k = k_next
    """

    def __init__(self, shape, device):
        self.buf = [torch.empty(shape, dtype=torch.float32, device=device) for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.used = [None, None]
        self.stream = torch.cuda.Stream(device)
        self.i = 0

    def upload(self, host: torch.Tensor) -> int:
        k = self.i % 2
        self.i += 1
        if self.used[k] is not None:                  # the step that last read buffer k is done
            self.stream.wait_event(self.used[k])
        with torch.cuda.stream(self.stream):
            self.buf[k].copy_(host, non_blocking=True)
            self.done[k].record(self.stream)
        return k

    def get(self, k: int) -> torch.Tensor:
        torch.cuda.current_stream().wait_event(self.done[k])
        return self.buf[k]

    def release(self, k: int):
        e = torch.cuda.Event()
        e.record(torch.cuda.current_stream())
        self.used[k] = e


class RefineOptimizer:
    """Jointly optimises vertices, IoR and absorption of a DeviceScene against target images.

    Data parallel (dist.py): every rank traces its own rays into one persistent
    flat gradient buffer (dist.GradBuffer); the regularisers that do not depend on the rays
    (L_mat-smooth / L_vol) are added on rank 0 only, before the gradient hook all-reduces the
    buffer, so every rank applies the same summed gradient and the parameters stay identical
    (the updates are deterministic); the periodic mesh pass runs on rank 0 and its vertices are
    broadcast."""

    def __init__(self, tracer: Tracer, ds: DeviceScene, cfg: Optional[RefineConfig] = None, seed: int = 0,
                 grad_hook: Optional[Callable] = None, loss_scale: float = 1.0, rank: int = 0,
                 broadcast: Optional[Callable] = None):
        """grad_hook(flat): called on the flat [dV | dIOR | dsigma] buffer (GradBuffer.flat) after the
        ray-loss backward and rank 0's regularisers, before the updates (data parallel:
        dist.allreduce_flat).  loss_scale scales lambda_color / lambda_tone; with rays sharded over
        ranks, n_local / n_global makes the summed gradient that of the global mean (loss_rt
        normalises by the local ray count).  rank: this process's rank (rank 0 adds the
        ray-independent regularisers).  broadcast(tensor): rank 0's tensor to every rank (the
        vertices after the periodic mesh pass)."""
        self.tr, self.ds, self.cfg = tracer, ds, cfg or RefineConfig()
        self.grad_hook, self.loss_scale = grad_hook, float(loss_scale)
        self.rank, self.broadcast = int(rank), broadcast
        dev = ds.V.device
        self.V = ds.V.clone().contiguous()
        self.ior = torch.tensor([ds.ior], dtype=torch.float32, device=dev)
        self.sigma = ds.sigma.clone().contiguous()
        self.mV, self.vV = torch.zeros_like(self.V), torch.zeros(1, device=dev)          # AdamUniform: scalar v
        self.mI, self.vI = torch.zeros_like(self.ior), torch.zeros_like(self.ior)
        self.mS, self.vS = torch.zeros_like(self.sigma), torch.zeros_like(self.sigma)
        self.grads = GradBuffer(self.V.shape[0], tuple(self.sigma.shape), dev)
        self.gen = torch.Generator(device=dev)
        self.gen.manual_seed(seed)
        self.it = 0
        self.dropped = 0                      # asynchronous steps dropped by an arena overflow
        self.t_dev = None                     # device Adam step counts [sigma, IoR, V] (CUDA graphs)
        self.loss = torch.zeros(4, dtype=torch.float32, device=dev)

    def _reg_points(self):
        ab = self.ds.absorption
        dev = self.sigma.device
        n = self.cfg.n_reg_points
        lo = torch.tensor(list(ab.box_lo), device=dev)
        hi = torch.tensor(list(ab.box_hi), device=dev)
        pts = lo + (hi - lo) * torch.rand((n, 3), generator=self.gen, device=dev)
        xi = torch.randn((n, 3), generator=self.gen, device=dev) * (self.cfg.reg_sigma_perturb * (hi - lo))
        return pts.contiguous(), xi.contiguous()

    def regularize(self, gt_masks: torch.Tensor, iters: Optional[int] = None) -> torch.Tensor:
        """The periodic mesh pass: `iters` (default cfg.reg_inner) AdamUniform steps
        on the vertices of lambda_mask L_mask + lambda_edge L_edge + lambda_lap L_lap against the
        ground-truth masks [n_views][H][W]; the LBVH is rebuilt before every step.  Returns the
        last losses (L_mask, L_edge, L_lap) on the device."""
        c, tr, ds = self.cfg, self.tr, self.ds
        iters = c.reg_inner if iters is None else iters
        m, v = torch.zeros_like(self.V), torch.zeros(1, device=self.V.device)
        g = torch.zeros_like(self.V)
        out = torch.zeros(3, dtype=torch.float32, device=self.V.device)
        for t in range(1, iters + 1):
            ds.set_vertices(self.V)
            tr.build_bvh(ds.V, ds.F)
            g.zero_()
            lm, _, _ = tr.mask_loss(ds, gt_masks, c.lambda_mask, grad_V=g)
            lr_, _ = tr.mesh_regularizers(c.lambda_edge, c.lambda_lap, grad_V=g)
            tr.adam_step(self.V, g, m, v, t, c.lr_vertices, c.betas, c.eps, 0.0, uniform=True)
            out[:1] = lm
            out[1:] = lr_
        return out

    def _forward(self, pixel_ids, async_):
        """The step's forward.  An asynchronous forward's arena overflow is reported by the NEXT
        call as DT_ERR_RETRY: that earlier step changed nothing (its updates were skipped on the
        device through dt_adam.skip_if), so it is dropped -- its iteration count is taken back --
        and this step's forward runs again on the grown arena."""
        try:
            return self.tr.trace_forward(self.ds, pixel_ids, ior_device=self.ior, async_=async_)
        except N.DiffTransError as e:
            if e.status != N.DT_ERR_RETRY:
                raise
            self.it -= 1
            self.dropped += 1
            return self.tr.trace_forward(self.ds, pixel_ids, ior_device=self.ior, async_=async_)

    def step(self, target: torch.Tensor, pixel_ids: Optional[torch.Tensor] = None, async_: bool = False,
             gt_masks: Optional[torch.Tensor] = None) -> StepResult:
        """One iteration, queued on the current stream.  async_: the forward does not wait for its
        arena-overflow check (an overflow surfaces as DT_ERR_RETRY on the next call, which then
        drops that step; see _forward) so consecutive steps queue back to back with no host stall."""
        c, tr, ds, G = self.cfg, self.tr, self.ds, self.grads
        ds.set_vertices(self.V)
        ds.set_sigma(self.sigma)
        tr.build_bvh(ds.V, ds.F)
        # the kernels read the IoR from self.ior (dt_trace_opts.ior_device): no host round trip
        out = self._forward(pixel_ids, async_)
        self.it += 1
        lrt, grad_rgb = tr.loss_rt(out.rgb, target, c.lambda_color * self.loss_scale, c.lambda_tone * self.loss_scale)
        tr.trace_backward(grad_rgb, grad_V=G.gV, grad_ior=G.gI, grad_sigma=G.gS)
        if ds.absorption.kind in (1, 2):          # grid / hash texture: sampled regularisers
            pts, xi = self._reg_points()
        else:
            pts = xi = None
        w = 1.0 if self.rank == 0 else 0.0        # ray-independent: added once, on rank 0
        lreg = tr.sigma_regularizers(ds, pts, xi, G.gS, c.lambda_smooth * w, c.lambda_vol * w)
        if self.grad_hook is not None:
            self.grad_hook(G.flat)
        frozen = self.it <= c.freeze_iters
        skip = tr.overflow_flag()                 # an overflowed forward's gradients are invalid
        td = [None, None, None] if self.t_dev is None else [self.t_dev[i:i + 1] for i in range(3)]
        tr.adam_step(self.sigma, G.gS, self.mS, self.vS, self.it, c.lr_material, c.betas, c.eps, c.weight_decay,
                     clamp=(0.0, float("inf")), skip_if=skip, step_device=td[0])
        tr.adam_step(self.ior, G.gI, self.mI, self.vI, self.it, c.lr_ior_frozen if frozen else c.lr_ior, c.betas, c.eps,
                     c.weight_decay, clamp=c.ior_range, skip_if=skip, step_device=td[1])
        if not frozen:
            tr.adam_step(self.V, G.gV, self.mV, self.vV, self.it - c.freeze_iters, c.lr_vertices, c.betas, c.eps,
                         c.weight_decay, uniform=True, skip_if=skip, step_device=td[2])
        self.loss[:2] = lrt
        self.loss[2:] = lreg
        if gt_masks is not None and not frozen and c.reg_every > 0 and self.it % c.reg_every == 0:
            if self.rank == 0:                    # float atomics: one rank runs it, the others copy
                self.regularize(gt_masks)
            if self.broadcast is not None:
                self.broadcast(self.V)
        return StepResult(self.loss, self.ior)

    def capture_step(self, target: torch.Tensor, pixel_ids: Optional[torch.Tensor] = None,
                     prepare: Optional[Callable] = None) -> torch.cuda.CUDAGraph:
        """One post-freeze optimisation step (LBVH rebuild, forward, loss, backward, regularisers,
        gradient hook, Adam) captured into a CUDA graph: each replay runs the whole step with no
        host work and no launch overhead (the launch-bound regime of the paper's 5,000-ray batches,
        P:531).  The Adam step counts move to the device (dt_adam.step_device) so every replay
        applies the right bias correction; `self.it` stops advancing (see sync_steps).
        prepare(): optional work captured before the step (e.g. drawing this replay's random
        pixel batch into `pixel_ids` / `target`, whose addresses must stay fixed).  The periodic
        mesh pass is not captured (host-driven, every reg_every steps).  After replays,
        synchronise and call self.tr.get_stats(): DT_ERR_RETRY means a replay overflowed the
        record arena (its updates were skipped on the device; capture again)."""
        c = self.cfg
        assert self.it >= c.freeze_iters, "capture the post-freeze phase (the schedule is host logic)"
        dev = self.V.device
        self.t_dev = torch.tensor([self.it + 1, self.it + 1, self.it + 1 - c.freeze_iters], dtype=torch.int32,
                                  device=dev)

        def one():
            if prepare is not None:
                prepare()
            self.step(target, pixel_ids, async_=True)

        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):          # warm-up (allocations, persistent grids, arena size)
            for _ in range(2):
                one()
                self.tr.get_stats()
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            one()
        return g

    def sync_steps(self) -> None:
        """After CUDA-graph replays: the host step count from the device counters."""
        if self.t_dev is not None:
            self.it = int(self.t_dev[0].item()) - 1
