"""Benchmark: one optimisation step of the DiffTrans refine-stage tracer on B200.

A step = one RefineOptimizer.step (the paper's refine loop after the freeze-geometry
stage): LBVH rebuild (dt_build_bvh) + recursive forward trace of every ray of
the workload (dt_trace_forward, IoR read on the device) + fused L_color/L_tone loss and
gradient (dt_loss_rt) + backward replay (dt_trace_backward) [+ NCCL all-reduce of the
gradients when N > 1] + L_mat-smooth/L_vol (dt_sigma_regularizers) + Adam on sigma and
the IoR and AdamUniform on the vertices (dt_adam_step).
Metric (BASELINE.json): Mray.bounce/s fwd+bwd = traced segments / step time.

  python bench.py [--gpus N --steps K --warmup W --config C3 --impl ours|reference]

N > 1: launched by torchrun, one rank per GPU; rays shard by (view, 32x32 tile) across
ranks (strong scaling: the C3 step's total work is fixed), and rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import dataclasses
import glob
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "Mray*bounce/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def hbm_peak():
    try:
        return float(json.load(open(PEAKS))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML polled every 10 ms
    from a thread (so short runs still get samples), else nvidia-smi -lms 200."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []           # (sm_mhz, max_mhz, set of reasons)
        self.stop_flag = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.nvml = pynvml

            def poll():
                while not self.stop_flag.is_set():
                    sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, mx, {n for n, b in bits.items() if r & b}))
                    time.sleep(0.01)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()                      # wait for nvidia-smi to come up, then keep
            while not self.lines and time.time() - t0 < 5:   # only samples of the timed region
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.t.join(timeout=1)
            src = "nvml"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            src = "nvidia-smi"
            for ln in self.lines:
                p = [x.strip() for x in ln.split(",")]
                if len(p) < 7:
                    continue
                try:
                    self.samples.append((float(p[0]), float(p[1]),
                                         {nm for nm, v in zip(self.NAMES, p[3:7]) if v.lower().startswith("active")}))
                except ValueError:
                    continue
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(x[1] for x in self.samples) if self.samples else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def target_scene(sc):
    """Ground truth for the loss: the same scene rendered with IoR 1.45, sigma x 1.2 and the
    vertices jittered by 0.5% of the radius."""
    from paper_2603_00413_b200 import scenes as S
    g = S.rng(777, 81)
    r = float(np.linalg.norm(sc.V, axis=1).max())
    V = (sc.V + g.normal(size=sc.V.shape) * 0.005 * r / np.sqrt(3)).astype(np.float32)
    ab = dataclasses.replace(sc.absorption, sigma=(sc.absorption.sigma * 1.2).astype(np.float32))
    return dataclasses.replace(sc, V=V, ior=1.45, absorption=ab)


def oracle_sample(sc, n_pix: int, seed: int = 9, backward: bool = True, nthreads: int = 0):
    """Bounded oracle run (forward [+ backward]) on n_pix object pixels: (seconds, segments,
    threads); nthreads = 0 uses every host core."""
    import oracle as O
    from paper_2603_00413_b200 import scenes as S
    osc = O.OracleScene(sc)
    pid = S.central_pixels(sc.cams, n_pix, seed)
    g = S.upstream_grad(len(pid), seed)
    t0 = time.perf_counter()
    out = O.render(osc, pid, nthreads=nthreads)
    if backward:
        O.backward(osc, g, pid, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return dt, int(out["segments"].sum()), nthreads or os.cpu_count()


def algorithmic_bytes(stats, prof, steps: int):
    """Algorithmic bytes per step and launch class: record
    streams, shading gathers, children writes, and for traversal the wide-BVH nodes (64 B)
    and triangles (48 B) the rays fetch, counted on the device (most are served by L2)."""
    seg = stats["segments_per_depth"]
    D = len(seg) - 1
    # traversal (k >= 1): float64 ray in (o, d: 64 B), hit out (16 B), node and triangle fetches
    nodes = (prof["node_visits"] - prof["node_visits_primary"]) / steps
    tris = (prof["tri_tests"] - prof["tri_tests_primary"]) / steps
    trace = sum(seg[k] * 80 for k in range(1, D + 1)) + nodes * 64 + tris * 48
    # shading (all levels): record in (o, d float64 64 B + thr, hit 32 B), hit/tau/lsub out
    # (48 B), vertex gather (3 ids 12 B + 3 positions 48 B + 3 float64 normals 96 B), children
    # out (o, d, thr: 80 B each)
    shade = sum(seg[k] * (96 + 48 + 156) + (seg[k + 1] if k < D else 0) * 80 for k in range(0, D + 1))
    # backward: record in (o, d, thr, hit, tau, lsub: 128 B) + grad_rgb (12 B) + slots out
    # (32 B) + gather (156 B) + 6 float4 atomics RMW (192 B) + children's slots/radiance in
    # (48 B each)
    bwd = sum(seg[k] * (128 + 12 + 32 + 156 + 192) + (seg[k + 1] if k < D else 0) * 48 for k in range(0, D + 1))
    # traversal lane operations: 130 per 4-wide node visit (15 setup + 4 x 21
    # child slab test + 25 ordering + 6 push / pop), 37 per Moller-Trumbore triangle test
    ops = nodes * OPS_PER_VISIT + tris * OPS_PER_TEST
    return {"trace": trace, "shade": shade, "bwd": bwd, "trace_launches": D, "shade_launches": D + 1,
            "bwd_launches": D + 1, "trace_ops": ops}


OPS_PER_VISIT, OPS_PER_TEST = 130, 37


def walk_peaks():
    """Scattered float4 gather / atomic rates (tools/microbench/l2_gather.cu, measured on the
    GPU box): the texture walks' roofline peaks; None if the measurement is absent."""
    f = os.path.join(ROOT, "profiles", "r02_l2_gather.json")
    try:
        return json.load(open(f)), "measured (profiles/r02_l2_gather.json)"
    except Exception:
        return None


def alu_peak(sm_count: int):
    """SIMT lane-operation issue peak (B200_PROFILING.md / B300_MICROARCH.md unit counts): 4
    schedulers x 32 lanes per SM issue one operation per clock at the max SM clock."""
    try:
        mhz = float(json.load(open(PEAKS))["sm_max_mhz"])
        src = "derived: SMs x 128 lanes x sm_max_mhz (MEASURED_PEAKS.json)"
    except Exception:
        mhz, src = 1965.0, "derived: SMs x 128 lanes x 1965 MHz (fallback)"
    return sm_count * 128 * mhz * 1e6 / 1e12, src


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2603_00413_b200 import dist as DD
    from paper_2603_00413_b200 import scenes as S
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer

    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    sc = S.CONFIGS[args.config]()
    ds = DeviceScene(sc, dev)
    tr = Tracer(dev)
    pid = None
    if world > 1:
        from paper_2603_00413_b200.tracer import TileShard
        W, H, nvw = sc.cams.width, sc.cams.height, sc.cams.n_views
        # the rank's (view, 32x32 tile) shard goes to the kernels as dt_cameras.tile (no pixel
        # list: the kernels enumerate the tiles' pixels); ragged images fall back to pixel lists
        tiled = W % 32 == 0 and H % 32 == 0
        pid = TileShard(32, rank, world) if tiled else \
            torch.as_tensor(DD.tile_pixel_ids(nvw, W, H, rank, world), device=dev)
        if args.balance == "lpt" and tiled:
            # tile balancing: one untimed forward of this rank's cyclic share
            # counts the traced segments per ray; the per-tile costs of all ranks are summed into
            # one vector and every rank runs the same greedy LPT assignment on it
            tr.build_bvh(ds.V, ds.F)
            nr = pid.n_rays(nvw, W, H)
            segc = torch.zeros(nr, dtype=torch.int32, device=dev)
            tr.trace_forward(ds, pid, seg_count=segc)
            total = nvw * (W // 32) * (H // 32)
            costs = torch.as_tensor(DD.shard_tile_costs(DD.shard_tiles(nvw, W, H, rank, world), segc.cpu().numpy(),
                                                        total), device=dev)
            dist.all_reduce(costs, op=dist.ReduceOp.SUM)
            mine = DD.lpt_assign(costs.cpu().numpy(), world)[rank]
            pid = TileShard(32, tile_ids=torch.as_tensor(mine, dtype=torch.int32, device=dev))
    n_rays = ds.n_pixels if pid is None else (pid.numel() if torch.is_tensor(pid) else
                                             pid.n_rays(sc.cams.n_views, sc.cams.width, sc.cams.height))
    infer = args.mode == "infer"
    rgb = torch.empty((n_rays, 3), dtype=torch.float32, device=dev)
    if infer:
        # NEXT-3 inference (relighting / novel views): forward only, fixed mesh (its
        # BVH built once), every view re-rendered each step under the scene's (swapped) env
        tr.build_bvh(ds.V, ds.F)

        def step(async_=True):
            tr.trace_forward(ds, pid, rgb=rgb, async_=async_)
    else:
        # ground-truth colours for the loss (not timed)
        tgt_sc = target_scene(sc)
        dt_ = DeviceScene(tgt_sc, dev)
        tr.build_bvh(dt_.V, dt_.F)
        target = tr.trace_forward(dt_, pid).rgb.clone()
        del dt_
        # the paper's refine loop after the freeze-geometry stage: vertices
        # (AdamUniform), IoR and sigma all updated every step; gradients all-reduced across ranks
        # before the updates
        n_global = ds.n_pixels
        hook = (lambda flat: DD.allreduce_flat(flat)) if world > 1 else None
        bcast = (lambda t: dist.broadcast(t, 0)) if world > 1 else None
        opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0), seed=5, grad_hook=hook,
                              loss_scale=n_rays / n_global, rank=rank, broadcast=bcast)

        def step(async_=True):
            opt.step(target, pid, async_=async_)

    for w in range(args.warmup):
        step(async_=w > 0)          # the first (synchronous) step sizes the record arena
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tr.profile(reset=True)
    import gc
    gc.collect()
    gc.disable()                    # no host GC pauses between asynchronously queued steps
    tr.set_profiling(os.environ.get("BENCH_NO_PROF") is None)
    clocks = ClockSampler(local_rank)
    if os.environ.get("BENCH_NO_CLOCKS") is None:
        clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    gc.enable()
    last = tr.get_stats()           # raises DT_ERR_RETRY if an asynchronous step overflowed
    tr.set_profiling(False)
    prof = tr.profile(reset=True)
    segs = prof["segments"]         # counted on the device by every timed forward
    eager = None
    ms_eager = ms
    if world == 1 and args.graph:
        # the same step captured once into a CUDA graph and replayed (no per-kernel launch gaps,
        # no profiling events); the eager run above supplies the phase split and launch counts
        eager = {"ms_per_step": round(ms / args.steps, 3), "value": round(segs / (ms / 1e3) / 1e6, 3),
                 "note": "same step launched kernel by kernel, with per-phase profiling events"}
        if infer:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                for _ in range(2):
                    step()
                    tr.get_stats()
            torch.cuda.current_stream(dev).wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
        else:
            graph = opt.capture_step(target, pid)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        tr.get_stats()
        tr.profile(reset=True)
        clocks = ClockSampler(local_rank)
        if os.environ.get("BENCH_NO_CLOCKS") is None:
            clocks.start()
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        clk = clocks.stop()
        tr.get_stats()              # raises DT_ERR_RETRY if a replay overflowed the arena
        segs = tr.profile(reset=True)["segments"]
        if not infer:
            opt.sync_steps()
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms, float(segs), float(n_rays)], dtype=torch.float64, device=dev)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms, segs, rays_total = float(mx[0]), float(t[1]), int(t[2])
    else:
        rays_total = int(n_rays)
    value = segs / (ms / 1e3) / 1e6

    # ---- end-to-end through the public API with host buffers (pinned), same metric
    e2e = None
    if not args.no_e2e:
        if infer:
            # per step: the swapped environment's textures in from pinned host memory, the
            # rendered image back -- the image read-back of step i on a side stream while step
            # i+1 renders into the other buffer
            env_dev = [t for t in (ds.voxel, ds.planes) if t is not None]
            env_host = [t.cpu().pin_memory() for t in env_dev]
            himg = torch.empty((n_rays, 3), dtype=torch.float32, pin_memory=True)
            rgbs = [rgb, torch.empty_like(rgb)]
            d2h_stream = torch.cuda.Stream(dev)
            d2h_done = [None, None]
            state = {"i": 0}

            def e2e_step():
                k = state["i"] % 2
                state["i"] += 1
                if d2h_done[k] is not None:
                    torch.cuda.current_stream().wait_event(d2h_done[k])   # buffer k read back
                for d_, h_ in zip(env_dev, env_host):
                    d_.copy_(h_, non_blocking=True)
                tr.trace_forward(ds, pid, rgb=rgbs[k], async_=True)
                rendered = torch.cuda.Event()
                rendered.record(torch.cuda.current_stream())
                d2h_stream.wait_event(rendered)
                with torch.cuda.stream(d2h_stream):
                    himg.copy_(rgbs[k], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(d2h_stream)
                d2h_done[k] = ev

            def e2e_finish():                                # the timed region ends after the
                for ev in d2h_done:                          # side-stream copies too
                    if ev is not None:
                        torch.cuda.current_stream().wait_event(ev)
            h2d_bytes = sum(t.numel() * 4 for t in env_host)
            d2h_bytes = himg.numel() * 4
        else:
            # per step: this step's target pixels in from pinned host memory, the losses and the
            # updated IoR back (the optimiser state -- V, sigma, moments -- stays resident in HBM)
            # (the next step's target is uploaded on a side stream while this step computes,
            # optim.HostTargets)
            from paper_2603_00413_b200.optim import HostTargets
            htgt = torch.empty((n_rays, 3), dtype=torch.float32, pin_memory=True)
            htgt.copy_(target.cpu())
            hloss = torch.empty(4, pin_memory=True)
            hior = torch.empty(1, pin_memory=True)
            up = HostTargets(tuple(target.shape), dev)
            state = {"k": up.upload(htgt)}

            def e2e_step():
                k = state["k"]
                tgt = up.get(k)
                state["k"] = up.upload(htgt)                 # next step's target, overlapped
                r = opt.step(tgt, pid, async_=True)
                up.release(k)
                hloss.copy_(r.loss, non_blocking=True)
                hior.copy_(r.ior, non_blocking=True)

            def e2e_finish():
                up.get(state["k"])                           # the last upload is inside the region
            h2d_bytes = htgt.numel() * 4
            d2h_bytes = hloss.numel() * 4 + hior.numel() * 4

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tr.profile(reset=True)
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e2e_finish()
        e1.record()
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1)
        tr.get_stats()
        s2 = tr.profile(reset=True)["segments"]
        if world > 1:
            t = torch.tensor([ms2, float(s2)], dtype=torch.float64, device=dev)
            mx = t.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            ms2, s2 = float(mx[0]), float(t[1])
        h2d, d2h = h2d_bytes, d2h_bytes
        e2e = {"value": s2 / (ms2 / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms2 / args.steps}

    if rank != 0:
        return None
    # ---- roofline of the dominant launch class, device time measured live (CUDA events)
    peak, peak_src = hbm_peak()
    ab = algorithmic_bytes(last, prof, args.steps)
    ph = prof["ms"]
    cls = max(("trace", "shade", "bwd"), key=lambda c: ph[c])
    launches = prof["launches"][cls]
    ms_per_launch = ph[cls] / max(launches, 1)
    bytes_per_launch = ab[cls] / max(ab[f"{cls}_launches"], 1)
    achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9
    kname = {"trace": "k_traverse_level", "shade": "k_shade_level", "bwd": "k_backward_level"}[cls]
    traffic, traffic_src = None, None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json"))):
        try:
            t = json.load(open(f))
        except Exception:
            continue
        if t.get("config") == args.config and t.get("kernel") == kname:
            traffic, traffic_src = float(t["dram_bytes_per_launch"]), os.path.relpath(f, ROOT)
    l2 = None
    try:                                      # L2 read bandwidth, tools/microbench/l2_bw.cu
        l2 = float(json.load(open(os.path.join(ROOT, "profiles", "r01_l2_bandwidth.json")))["l2_read_gbs"])
    except Exception:
        pass
    hbm_view = {"unit": "GB/s", "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src,
                "frac": round(achieved / peak, 4), "bytes_per_launch": int(bytes_per_launch),
                "l2_read_peak_gbs": l2, "frac_of_l2": round(achieved / l2, 4) if l2 else None}
    ncu = {}
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json"))):
        try:
            t = json.load(open(f))
        except Exception:
            continue
        if t.get("config") == args.config and t.get("kernel") == kname:
            ncu = t
    if cls == "trace":
        # the traversal is bound by instruction issue (ncu: IPC ~3.2 of 4, ~17 of 32 lanes
        # active, L2-resident LBVH, DRAM at a few % of peak): its roofline is lane operations
        # against the SIMT issue peak; the algorithmic-bytes view is kept alongside
        apk, apk_src = alu_peak(torch.cuda.get_device_properties(dev).multi_processor_count)
        ops_launch = ab["trace_ops"] / max(ab["trace_launches"], 1)
        a_ops = ops_launch / (ms_per_launch / 1e3) / 1e12
        roofline = {"bound": "alu", "kernel": kname, "achieved": round(a_ops, 3), "peak": round(apk, 2),
                    "peak_source": apk_src, "unit": "Tlane-op/s", "frac": round(a_ops / apk, 4),
                    "ops_per_node_visit": OPS_PER_VISIT, "ops_per_triangle_test": OPS_PER_TEST,
                    "ops_per_launch": int(ops_launch)}
    elif cls == "bwd" and prof.get("walk_cells_bwd", 0) > 0 and walk_peaks() is not None:
        # texture walks (sigma grid C4 / hash texture C4H): the backward is bound by the L2
        # serving its corner fetches and float4 adjoint atomics, counted on the device per cell
        # visit (grid: 4 x-pair loads; hash: 8 entry loads; both: 8 atomics).  Peak: the time
        # those operations take at the L2's measured ceilings for the same operations
        # (coalesced float4 loads / REDs, tools/microbench/l2_gather.cu); the same at the
        # measured rates of fully scattered accesses (the walks sit in between: neighbouring
        # rays and samples share cells) and the record-bytes view are kept alongside
        wp, wp_src = walk_peaks()
        hashed = sc.absorption.kind == 2
        cells = prof["walk_cells_bwd"] / max(launches, 1)
        g_ops, r_ops = cells * (8 if hashed else 4), cells * 8
        t = ms_per_launch / 1e3
        achieved = (g_ops + r_ops) / t / 1e9

        def peak_of(g, r):
            return (g_ops + r_ops) / (g_ops / (g * 1e9) + r_ops / (r * 1e9)) / 1e9
        pk = peak_of(wp["gather_coalesced_gops"], wp["red_coalesced_gops"])
        size = "128mb" if hashed else "8mb"
        pk_s = peak_of(wp[f"gather_{size}_gops"], wp[f"red_{size}_gops"])
        roofline = {"bound": "l2", "kernel": kname + ("_hash" if hashed else "_grid"), "achieved": round(achieved, 2),
                    "peak": round(pk, 2), "peak_source": wp_src + ": coalesced float4 load / RED ceilings",
                    "unit": "Gop/s", "frac": round(achieved / pk, 4),
                    "ops": "L2 accesses of the walk: corner fetches + float4 adjoint atomics",
                    "cell_visits_per_launch": int(cells), "gathers_per_launch": int(g_ops),
                    "atomics_per_launch": int(r_ops), "gather_gops": round(g_ops / t / 1e9, 2),
                    "atomic_gops": round(r_ops / t / 1e9, 2),
                    "scattered_view": {"peak": round(pk_s, 2), "frac": round(achieved / pk_s, 4),
                                       "table": size, "source": wp_src + ": hashed-index float4 load / RED rates"},
                    "hbm_view": hbm_view}
    elif cls == "bwd" and prof.get("env_samples_bwd", 0) > 0 and walk_peaks() is not None:
        # volumetric env (C3V): the backward replays every exterior segment's env-volume samples,
        # each 8 voxel + 12 plane float4 texel fetches (frozen env: no atomics), counted on the
        # device; peak: the L2's coalesced float4 load ceiling (scattered view beside it)
        wp, wp_src = walk_peaks()
        samp = prof["env_samples_bwd"] / max(launches, 1)
        g_ops = samp * 20
        t = ms_per_launch / 1e3
        achieved = g_ops / t / 1e9
        pk, pk_s = wp["gather_coalesced_gops"], wp["gather_128mb_gops"]
        roofline = {"bound": "l2", "kernel": kname + "_vol", "achieved": round(achieved, 2), "peak": round(pk, 2),
                    "peak_source": wp_src + ": coalesced float4 load ceiling", "unit": "Gop/s",
                    "frac": round(achieved / pk, 4), "ops": "env-volume texel fetches (8 voxel + 12 plane per sample)",
                    "samples_per_launch": int(samp), "fetches_per_launch": int(g_ops),
                    "scattered_view": {"peak": round(pk_s, 2), "frac": round(achieved / pk_s, 4), "table": "128mb",
                                       "source": wp_src + ": hashed-index float4 load rate"},
                    "hbm_view": hbm_view}
    else:
        roofline = {"bound": "hbm", "kernel": kname, **{k: v for k, v in hbm_view.items() if k != "bytes_per_launch"},
                    "bytes_per_launch": int(bytes_per_launch)}
    roofline.update({"traffic": traffic, "traffic_source": traffic_src, "ms_per_launch": round(ms_per_launch, 3),
                     "share_of_step": round(ph[cls] / ms_eager, 4)})
    if traffic is not None:
        roofline["dram_frac"] = round(traffic / (ms_per_launch / 1e3) / 1e9 / peak, 4)
    for key in ("l2_hit_pct", "l1_hit_pct", "lanes_per_inst", "ipc", "issue_active_pct"):
        if key in ncu:
            roofline[key] = ncu[key]
    if cls == "trace":
        roofline["hbm_view"] = hbm_view
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        dt, osegs, cores = oracle_sample(sc, args.cpu_pixels, backward=not infer)
        n1 = max(args.cpu_pixels // 32, 1)                  # also one thread
        dt1, osegs1, _ = oracle_sample(sc, n1, seed=10, backward=not infer, nthreads=1)
        cpu = {"value": osegs / dt / 1e6, "unit": UNIT, "cores": cores, "kind": "oracle",
               "value_1thread": osegs1 / dt1 / 1e6, "sample_1thread": f"{n1} object pixels, 1 thread",
               "sample": f"{args.cpu_pixels} object pixels of {args.config}, {'fwd' if infer else 'fwd+bwd'}, "
                         f"fp64 brute force, "
                         f"{osegs} segments in {dt:.1f}s"}
    line = {
        "metric": METRIC if not infer else "Mrays·bounces/s forward-only (relighting / novel-view inference, D 8)",
        "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, sc, infer),
                   "rays_per_step": rays_total, "segments_per_step": int(segs / args.steps),
                   "segments_per_depth": last["segments_per_depth"], "parallelism": f"rays{world}", "balance": args.balance if world > 1 else None,
                   "l2": "working set > L2: path-record arena "
                         f"{last['arena_capacity'] * 160 / 1e9:.1f} GB streamed every step; "
                         + ("LBVH built once (fixed mesh)" if infer else "LBVH rebuilt in-step")},
        "clocks": clk, "e2e": e2e, "gpu_launches": int(prof["kernel_launches"]), "roofline": roofline,
        "cuda_graph": eager is not None, "eager": eager,
        "cpu_baseline": cpu,
        "phase_ms_per_step": {k: round(v / args.steps, 3) for k, v in ph.items()},
        "counters_per_step": {"node_visits": prof["node_visits"] // args.steps,
                              "tri_tests": prof["tri_tests"] // args.steps,
                              "walk_cells_fwd": prof["walk_cells_fwd"] // args.steps,
                              "walk_cells_bwd": prof["walk_cells_bwd"] // args.steps,
                              "env_samples_bwd": prof["env_samples_bwd"] // args.steps},
    }
    return line


def workload_name(config, sc, infer):
    """The config's `workload` string (identical on both arms)."""
    return (f"{config}: {sc.F.shape[0]} tris, {sc.cams.n_views} views "
            f"{sc.cams.width}x{sc.cams.height}, depth {sc.max_depth}, "
            f"{['const', 'grid', 'hash-grid'][sc.absorption.kind]} sigma, "
            f"{['analytic', 'voxel+triplane', 'volumetric voxel+triplane'][sc.env.kind]} env, "
            f"{'forward only' if infer else 'fwd+bwd+optimiser step'}")


def run_reference(args, rank, world):
    """The oracle (fp64 CPU, brute force) as it stands, on a bounded sample of the workload."""
    if rank != 0:
        return None
    from paper_2603_00413_b200 import scenes as S
    sc = S.CONFIGS[args.config]()
    bwd = args.mode != "infer"
    for _ in range(args.warmup):
        oracle_sample(sc, max(args.ref_pixels // 4, 1), seed=100, backward=bwd)
    tot_t, tot_s = 0.0, 0
    for k in range(args.steps):
        dt, segs, cores = oracle_sample(sc, args.ref_pixels, seed=200 + k, backward=bwd)
        tot_t += dt
        tot_s += segs
    v = tot_s / tot_t / 1e6
    sample = (f"each step: {args.ref_pixels} object pixels of {args.config} (fp64 brute force "
              f"{'fwd+bwd' if bwd else 'fwd'}); "
              f"{tot_s} segments in {tot_t:.1f}s")
    metric = METRIC if bwd else "Mrays·bounces/s forward-only (relighting / novel-view inference, D 8)"
    return {"impl": "reference", "metric": metric, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, sc, not bwd)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_batch(args, rank, world, local_rank):
    """The paper's own training iteration: a random batch of --batch rays per step drawn
    over all pixels of all views, with the LBVH rebuilt every step (the mesh moves).  At 5,000
    rays the step is launch- and build-bound, so it is captured once into a CUDA graph
    (RefineOptimizer.capture_step; the random draw and the target gather are captured too) and
    replayed; the eager (per-call launch) time of the same step is measured beside it."""
    import torch

    from paper_2603_00413_b200 import scenes as S
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer

    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    sc = S.CONFIGS[args.config]()
    ds = DeviceScene(sc, dev)
    tr = Tracer(dev)
    tgt_sc = target_scene(sc)
    dt_ = DeviceScene(tgt_sc, dev)
    tr.build_bvh(dt_.V, dt_.F)
    target_full = tr.trace_forward(dt_).rgb.clone()
    del dt_
    # a build serves only B rays here: the plain Karras hierarchy (no treelet passes) is cheaper
    tr.set_bvh_quality(0)
    B, npix = args.batch, ds.n_pixels
    torch.manual_seed(11 + rank)
    pid = torch.empty(B, dtype=torch.int64, device=dev)
    tgt = torch.empty((B, 3), dtype=torch.float32, device=dev)

    def prepare():                       # this step's random rays and their target colours
        torch.randint(0, npix, (B,), device=dev, out=pid)
        torch.index_select(target_full, 0, pid, out=tgt)

    opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0), seed=5)
    prepare()
    opt.step(tgt, pid)                   # synchronous: sizes the record arena
    for _ in range(max(args.warmup - 1, 1)):
        prepare()
        opt.step(tgt, pid, async_=True)
    tr.get_stats()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # eager: every kernel launched by the host each step
    tr.profile(reset=True)
    tr.set_profiling(False)
    e0.record()
    for _ in range(args.steps):
        prepare()
        opt.step(tgt, pid, async_=True)
    e1.record()
    torch.cuda.synchronize()
    ms_eager = e0.elapsed_time(e1)
    tr.get_stats()
    p_eager = tr.profile(reset=True)
    # CUDA graph of the same step
    g = opt.capture_step(tgt, pid, prepare=prepare)
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    tr.get_stats()
    tr.profile(reset=True)
    clocks = ClockSampler(local_rank)
    if os.environ.get("BENCH_NO_CLOCKS") is None:
        clocks.start()
    e0.record()
    for _ in range(args.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    tr.get_stats()                       # raises DT_ERR_RETRY if a replay overflowed the arena
    segs = tr.profile(reset=True)["segments"]
    opt.sync_steps()
    value = segs / (ms / 1e3) / 1e6
    launches_per_step = p_eager["kernel_launches"] / args.steps
    return {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} mesh ({ds.F.shape[0]} tris) with the paper's training batch: {B} random "
                               f"rays per step over {sc.cams.n_views} views {sc.cams.width}x{sc.cams.height} "
                               f"(P:531), depth {sc.max_depth}, LBVH rebuilt every step, fwd+bwd+optimiser step",
                   "batch": B, "segments_per_step": round(segs / args.steps), "cuda_graph": True,
                   "l2": "per-step working set (LBVH, mesh, records) is L2-resident; the target image is 768 MB"},
        "iterations_per_s": round(1e3 * args.steps / ms, 1),
        "eager": {"ms_per_step": round(ms_eager / args.steps, 4),
                  "value": round(p_eager["segments"] / (ms_eager / 1e3) / 1e6, 3),
                  "iterations_per_s": round(1e3 * args.steps / ms_eager, 1)},
        "graph_speedup": round(ms_eager / ms, 3),
        "clocks": clk, "gpu_launches": int(round(launches_per_step * args.steps)),
        "gpu_launches_per_step": launches_per_step,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, help="default C3 (train) / C3R (infer)")
    ap.add_argument("--mode", default="train", choices=["train", "infer"],
                    help="train: one refine-loop optimisation step; infer: forward-only rendering (NEXT-3)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-pixels", type=int, default=1024, help="oracle sample for cpu_baseline (~10-30 s)")
    ap.add_argument("--ref-pixels", type=int, default=192, help="oracle pixels per --impl reference step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--balance", default="lpt", choices=["lpt", "cyclic"],
                    help="N > 1: tile assignment (greedy LPT on measured per-tile segments, or cyclic)")
    ap.add_argument("--graph", action="store_true",
                    help="N = 1: also capture the full-image step into a CUDA graph and time its replays (measured: "
                         "no gain at C3, the kernels are long enough to hide launch gaps; default off)")
    ap.add_argument("--batch", type=int, default=0,
                    help="> 0: the paper's training iteration with this many random rays per step (P:531: 5000), "
                         "captured into a CUDA graph; 0: full images (default)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "C3R" if args.mode == "infer" else "C3"
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # functional check of the multi-rank path on a box with fewer GPUs than ranks (tests only;
    # never used for a reported number): BENCH_SHARE_GPU=1 maps ranks onto the visible devices
    # and BENCH_DIST_BACKEND picks the process-group backend (default nccl)
    if os.environ.get("BENCH_SHARE_GPU") == "1":
        import torch
        local_rank %= max(torch.cuda.device_count(), 1)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
            else:
                dist.init_process_group(backend)
        line = run_batch(args, rank, world, local_rank) if args.batch > 0 else run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
