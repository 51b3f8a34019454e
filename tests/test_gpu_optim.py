"""GPU parity of the optimisation-step kernels (NEXT-1) against oracle/optim.py, and an
end-to-end desk-scale recovery check of the whole refine loop (Table 2 analog)."""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import optim as OO
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T
from tests._parity import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tracer():
    from paper_2603_00413_b200.tracer import Tracer
    return Tracer("cuda:0")


def test_loss_rt_matches_oracle(tracer):
    g = np.random.default_rng(3)
    n = 10000
    rgb = g.uniform(0, 3, (n, 3)).astype(np.float32)
    tgt = g.uniform(0, 3, (n, 3)).astype(np.float32)
    tgt[:10] = 0.0                      # black targets (zero weight, tone pair skipped)
    mask = g.uniform(0, 1, n).astype(np.float32)
    d = lambda a: torch.as_tensor(a, device="cuda:0")
    loss, grad = tracer.loss_rt(d(rgb), d(tgt), 1.0, 0.25, mask=d(mask))
    Lc, Lt, go = OO.loss_rt(rgb, tgt, mask, 1.0, 0.25)
    l = loss.cpu().numpy()
    assert abs(l[0] - Lc) < 1e-5 * abs(Lc) and abs(l[1] - Lt) < 1e-4 * max(abs(Lt), 1e-3)
    assert rel_l2(grad.cpu().numpy(), go) < 1e-5


def test_sigma_regularizers_match_oracle(tracer):
    from paper_2603_00413_b200.tracer import DeviceScene
    V, F = S.icosphere(2)
    sc = T.scene(V, F, T.one_view(8, 8, (0, 0, 3)), absorption=T.small_sigma_grid(V, 10))
    ds = DeviceScene(sc, torch.device("cuda:0"))
    g = np.random.default_rng(4)
    ab = sc.absorption
    pts = g.uniform(ab.box_lo, ab.box_hi, (3000, 3)).astype(np.float32)
    xi = (g.normal(size=(3000, 3)) * 0.05).astype(np.float32)
    gs = torch.zeros_like(ds.sigma)
    loss = tracer.sigma_regularizers(ds, torch.as_tensor(pts, device="cuda:0"), torch.as_tensor(xi, device="cuda:0"),
                                     gs, 0.3, 0.7)
    Lm, Lv, go = OO.sigma_regularizers(ab, pts, xi, 0.3, 0.7)
    l = loss.cpu().numpy()
    assert abs(l[0] - Lm) < 1e-4 * Lm and abs(l[1] - Lv) < 1e-4 * Lv
    assert rel_l2(gs.cpu().numpy(), go) < 1e-4
    sc = T.scene(V, F, T.one_view(8, 8, (0, 0, 3)), sigma=(0.2, 0.5, 1.0))
    ds = DeviceScene(sc, torch.device("cuda:0"))
    gs = torch.zeros(3, device="cuda:0")
    loss = tracer.sigma_regularizers(ds, None, None, gs, 0.3, 0.5)
    np.testing.assert_allclose(loss.cpu().numpy(), [0.0, 1.29], rtol=1e-6)
    np.testing.assert_allclose(gs.cpu().numpy(), [0.2, 0.5, 1.0], rtol=1e-6)


def test_sigma_regularizers_hash_match_oracle(tracer):
    from paper_2603_00413_b200.tracer import DeviceScene
    V, F = S.icosphere(2)
    sc = T.scene(V, F, T.one_view(8, 8, (0, 0, 3)), absorption=T.small_hash_grid(V, levels=4, log2_size=8, top=16))
    ds = DeviceScene(sc, torch.device("cuda:0"))
    g = np.random.default_rng(6)
    ab = sc.absorption
    pts = g.uniform(ab.box_lo, ab.box_hi, (2000, 3)).astype(np.float32)
    xi = (g.normal(size=(2000, 3)) * 0.05).astype(np.float32)
    gs = torch.zeros_like(ds.sigma)
    loss = tracer.sigma_regularizers(ds, torch.as_tensor(pts, device="cuda:0"), torch.as_tensor(xi, device="cuda:0"),
                                     gs, 0.3, 0.7)
    Lm, Lv, go = OO.sigma_regularizers(ab, pts, xi, 0.3, 0.7)
    l = loss.cpu().numpy()
    assert abs(l[0] - Lm) < 1e-4 * Lm and abs(l[1] - Lv) < 1e-4 * Lv
    assert rel_l2(gs.cpu().numpy(), go) < 1e-4


@pytest.mark.parametrize("uniform", [False, True])
def test_adam_matches_oracle(tracer, uniform):
    g = np.random.default_rng(5)
    n = 5000
    p = g.normal(size=n).astype(np.float32)
    pt = torch.as_tensor(p, device="cuda:0")
    m = torch.zeros(n, device="cuda:0")
    v = torch.zeros(1 if uniform else n, device="cuda:0")
    po, mo, vo = p.astype(np.float64), np.zeros(n), np.zeros(1 if uniform else n)
    for t in range(1, 6):
        grad = g.normal(size=n).astype(np.float32) * (10.0 if t == 3 else 1.0)
        tracer.adam_step(pt, torch.as_tensor(grad, device="cuda:0"), m, v, t, 1e-3, weight_decay=1e-6,
                         uniform=uniform, clamp=(-2.0, 2.0))
        f32 = lambda x: float(np.float32(x))       # the ABI takes float32 hyper-parameters
        po, mo, vo = OO.adam(po, grad, mo, vo, t, f32(1e-3), betas=(f32(0.9), f32(0.999)), eps=f32(1e-8),
                             weight_decay=f32(1e-6), uniform=uniform, clamp=(-2.0, 2.0))
    assert np.abs(pt.cpu().numpy() - po).max() < 1e-6
    assert rel_l2(v.cpu().numpy(), vo) < 1e-5


def test_refine_loop_recovers_ior_and_absorption():
    """Desk-scale analog of Table 2 (IoR recovery) + constant absorption recovery: render a
    target with eta* = 1.5, sigma* = (0.5, 1, 2), start from eta = 1.3, sigma = 0.2, geometry
    frozen; the on-device loop must recover both."""
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    V, F = S.icosphere(3)
    cams = S.hemisphere_cameras(6, 48, 48, 3.0, 1.0, 7, fill=0.8)
    truth = T.scene(V, F, cams, env=S.analytic_env(2), ior=1.5, sigma=(0.5, 1.0, 2.0), D=4)
    tr = Tracer("cuda:0")
    dt = DeviceScene(truth, torch.device("cuda:0"))
    tr.build_bvh(dt.V, dt.F)
    target = tr.trace_forward(dt).rgb.clone()
    init = T.scene(V, F, cams, env=S.analytic_env(2), ior=1.3, sigma=(0.2, 0.2, 0.2), D=4)
    ds = DeviceScene(init, torch.device("cuda:0"))
    cfg = RefineConfig(freeze_iters=10 ** 9, lr_material=0.03, lr_ior_frozen=0.005, lambda_tone=0.0,
                       lambda_smooth=0.0, lambda_vol=0.0)
    opt = RefineOptimizer(tr, ds, cfg, seed=1)
    first = None
    for it in range(400):
        r = opt.step(target)
        if first is None:
            first = float(r.loss[0])
    last = float(r.loss[0])
    assert last < 1e-2 * first
    assert abs(float(opt.ior.item()) - 1.5) < 0.02, float(opt.ior.item())   # SPEC acceptance 4: <= 0.02
    s = opt.sigma.cpu().numpy()
    np.testing.assert_allclose(s[:2], [0.5, 1.0], rtol=0.02)
    # the sigma = 2 channel transmits e^-4 ~ 2% through the sphere: weak signal, slow but
    # monotone convergence; require 20% and the right rank order (SPEC acceptance 5)
    assert abs(s[2] - 2.0) < 0.4 and s[0] < s[1] < s[2], s


def test_ior_device_pointer_matches_scalar(tracer):
    """dt_trace_opts.ior_device: the IoR read on the device gives bit-identical radiance and
    gradients (up to atomic summation order) to the same IoR passed by value (forward and the matching backward)."""
    from paper_2603_00413_b200.tracer import DeviceScene
    V, F = S.icosphere(3)
    sc = T.scene(V, F, T.one_view(32, 32, (0, 0, 3)), ior=1.37, sigma=(0.3, 0.6, 0.9), D=5)
    ds = DeviceScene(sc, torch.device("cuda:0"))
    tracer.build_bvh(ds.V, ds.F)
    g = torch.as_tensor(S.upstream_grad(ds.n_pixels, 3), device="cuda:0")
    ref = tracer.trace_forward(ds).rgb.clone()
    ref_g = [t.clone() for t in tracer.trace_backward(g)]
    ds.ior = 1.0                                   # ignored: the pointer wins
    ior_t = torch.tensor([1.37], dtype=torch.float32, device="cuda:0")
    out = tracer.trace_forward(ds, ior_device=ior_t).rgb
    got_g = tracer.trace_backward(g)
    assert torch.equal(out, ref)
    for a, b in zip(got_g, ref_g):                 # float atomics: summation order may differ
        assert rel_l2(a.cpu().numpy(), b.cpu().numpy()) < 1e-6


@pytest.mark.parametrize("mesh", ["ico3_noisy", "c2_cube_sphere"])
def test_mesh_regularizers_match_oracle(tracer, mesh):
    """NEXT-4 L_edge and L_lap (R31) and their vertex gradients."""
    from oracle import mesh_reg as MR
    g = np.random.default_rng(8)
    if mesh == "ico3_noisy":
        V, F = S.icosphere(3)
        V = (V * (1 + 0.05 * g.normal(size=V.shape))).astype(np.float32)
    else:
        V, F = S.cube_sphere(65, 2)
    Vd = torch.as_tensor(V, device="cuda:0")
    Fd = torch.as_tensor(F.astype(np.int32), device="cuda:0")
    tracer.build_bvh(Vd, Fd)
    le, ll = 0.7, 1.3
    loss, gV = tracer.mesh_regularizers(le, ll)
    Le, ge = MR.loss_edge(V.astype(np.float64), F)
    Ll, gl = MR.loss_lap(V.astype(np.float64), F)
    l = loss.cpu().numpy()
    assert abs(l[0] - Le) < 1e-4 * Le and abs(l[1] - Ll) < 1e-4 * Ll, (l, Le, Ll)
    assert rel_l2(gV.cpu().numpy(), le * ge + ll * gl) < 1e-4
    # accumulation into a caller buffer; deterministic (no atomics in the gradient)
    loss2, gV2 = tracer.mesh_regularizers(le, ll, grad_V=gV.clone())
    torch.testing.assert_close(gV2, 2 * gV, rtol=1e-5, atol=1e-6 * float(gV.abs().max()))
    _, gV3 = tracer.mesh_regularizers(le, ll)
    assert torch.equal(gV3, gV)


@pytest.mark.parametrize("case", ["ico2-1view", "ico3-3views"])
def test_mask_loss_matches_oracle(tracer, case):
    """NEXT-4 L_mask and its silhouette-edge-sampling gradient (R32) vs the oracle,
    at the north_star gradient bar (rel-L2 <= 1e-3), the rendered mask identical and the loss
    within 1e-6.  No sample is excluded.  tools/mask_diag.py found none of the 235 silhouette
    samples of the 1-view case within 1e-4 px of a visibility change or of a ground-truth pixel
    boundary, so float32 and float64 take the same sample decisions.  Measured rel-L2: 2.5e-7
    (1 view) and 4.8e-7 (3 views); the round-1 tolerance of 2e-2 had no justification."""
    import oracle as O
    from oracle import mask as OM
    from paper_2603_00413_b200.tracer import DeviceScene
    if case == "ico2-1view":
        V, F = S.icosphere(2)
        cams = T.one_view(48, 48, (0.3, 0.2, 3.0), fov_deg=50, up=(0.0, 1.0, 0.0))
    else:
        V, F = S.icosphere(3)
        cams = S.hemisphere_cameras(3, 40, 40, 3.0, 1.0, 7, fill=0.7)
    sc = T.scene(V, F, cams, D=0)
    osc = O.OracleScene(sc)
    ms = np.stack([OM.rendered_mask(osc, cams, v) for v in range(cams.n_views)])
    ys, xs = np.mgrid[0:cams.height, 0:cams.width]
    gt = np.stack([((xs + 0.5 - 0.54 * cams.width) ** 2 + (ys + 0.5 - 0.46 * cams.height) ** 2
                    <= (0.8 * np.sqrt(ms[v].sum() / np.pi)) ** 2) for v in range(cams.n_views)]).astype(np.float32)
    ds = DeviceScene(sc, torch.device("cuda:0"))
    tracer.build_bvh(ds.V, ds.F)
    loss, gV, mask = tracer.mask_loss(ds, torch.as_tensor(gt, device="cuda:0").contiguous(), 1.0, want_mask=True)
    mg = mask.cpu().numpy().reshape(ms.shape)
    assert (mg != ms).sum() == 0
    assert abs(float(loss.cpu()[0]) - OM.loss(osc, cams, gt)) <= 1e-6
    go = OM.gradient(osc, sc, gt)
    e = rel_l2(gV.cpu().numpy(), go)
    print(f"mask gradient rel-L2 {e:.3e} ({case})")
    assert e <= 1e-3, e


def test_periodic_mesh_pass_fits_the_mask():
    """The periodic regularisation pass moves a sphere toward a larger
    ground-truth silhouette: the mask loss drops and the silhouette vertices move outward."""
    from oracle import mask as OM
    import oracle as O
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    V, F = S.icosphere(3)
    cams = S.hemisphere_cameras(4, 40, 40, 3.0, 1.0, 3, fill=0.7)
    sc = T.scene(V, F, cams, D=1)
    big = T.scene(V * 1.15, F, cams, D=1)
    osc = O.OracleScene(big)
    gt = np.stack([OM.rendered_mask(osc, cams, v) for v in range(cams.n_views)]).astype(np.float32)
    tr = Tracer("cuda:0")
    ds = DeviceScene(sc, torch.device("cuda:0"))
    opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0, lr_vertices=3e-3), seed=2)
    gtd = torch.as_tensor(gt, device="cuda:0").contiguous()
    first = float(opt.regularize(gtd, 1)[0])
    last = opt.regularize(gtd, 60).cpu().numpy()
    assert last[0] < 0.5 * first, (first, last)
    r = np.linalg.norm(opt.V.cpu().numpy(), axis=1)
    assert r.max() > 1.05 and r.min() > 0.98, (r.min(), r.max())   # silhouette vertices moved out


def test_overflowed_async_step_changes_nothing_and_is_dropped():
    """ADVICE (api.cu:485): an asynchronous step whose forward overflows the record arena must not
    update the parameters (dt_adam.skip_if = dt_forward_overflow_flag) and is dropped: the next
    step takes its iteration count back and runs on the grown arena."""
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    sc = S.config_c2()
    sc = T.scene(sc.V, sc.F, sc.cams, env=sc.env, D=8)
    dev = torch.device("cuda:0")
    tr = Tracer(dev)
    ds = DeviceScene(sc, dev)
    tr.build_bvh(ds.V, ds.F)
    target = tr.trace_forward(ds).rgb.clone() * 0.9
    opt = RefineOptimizer(Tracer(dev), ds, RefineConfig(freeze_iters=0), seed=3)
    full = opt.V.clone()
    opt.V.copy_(full * 0.05)                   # a tiny object: the synchronous step measures a small need
    opt.step(target)
    opt.V.copy_(full)
    before = (opt.V.clone(), opt.sigma.clone(), opt.ior.clone(), opt.mV.clone(), opt.vV.clone(), opt.mI.clone())
    opt.step(target, async_=True)              # arena sized from the small need: overflows
    torch.cuda.synchronize()
    after = (opt.V, opt.sigma, opt.ior, opt.mV, opt.vV, opt.mI)
    for x, y in zip(before, after):
        assert torch.equal(x, y)
    assert opt.it == 2
    opt.step(target, async_=True)              # reports the overflow: that step is dropped, this one runs
    torch.cuda.synchronize()
    assert opt.dropped == 1 and opt.it == 2
    assert not torch.equal(opt.V, before[0])
    opt.tr.get_stats()                         # no further overflow pending


def test_cuda_graph_step_matches_eager():
    """RefineOptimizer.capture_step: a CUDA graph of one step (LBVH rebuild, async forward, loss,
    backward, regularisers, Adam with device step counts) replayed 3 times reaches the same
    parameters as 5 eager steps (the capture runs 2 eager warm-up steps first), up to the float
    atomics' summation order; the device step counters advance once per replay."""
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    sc = S.config_c2(n_views=2, res=96)
    dev = torch.device("cuda:0")
    tr0 = Tracer(dev)
    ds0 = DeviceScene(dataclasses.replace(sc, ior=1.45), dev)
    tr0.build_bvh(ds0.V, ds0.F)
    pid = torch.as_tensor(S.central_pixels(sc.cams, 3000, 9), device=dev)
    target = tr0.trace_forward(ds0, pid).rgb.clone()
    res = []
    for graph in (False, True):
        tr = Tracer(dev)
        ds = DeviceScene(sc, dev)
        opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0), seed=4)
        opt.step(target, pid)                       # synchronous first step sizes the arena
        tr.get_stats()
        if graph:
            g = opt.capture_step(target, pid)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            tr.get_stats()
            assert opt.t_dev.tolist() == [7, 7, 7]
            opt.sync_steps()
        else:
            for _ in range(5):
                opt.step(target, pid, async_=True)
            torch.cuda.synchronize()
            tr.get_stats()
        assert opt.it == 6
        res.append((opt.V.clone(), opt.ior.clone(), opt.sigma.clone()))
    (Va, ia, sa), (Vb, ib, sb) = res
    assert rel_l2(Vb.cpu().numpy(), Va.cpu().numpy()) < 1e-5
    assert abs(float(ib) - float(ia)) < 1e-5 and rel_l2(sb.cpu().numpy(), sa.cpu().numpy()) < 1e-5


def test_cuda_graph_replay_overflow_is_reported_and_changes_nothing():
    """A replay whose forward overflows the record arena (the arena was sized when the graph
    was captured) skips its updates on the device (dt_adam.skip_if) and is reported by
    dt_get_stats as DT_ERR_RETRY after the replays."""
    from paper_2603_00413_b200 import _native as N
    from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    sc = S.config_c2(n_views=2, res=96)
    sc = T.scene(sc.V, sc.F, sc.cams, env=sc.env, D=8)
    dev = torch.device("cuda:0")
    tr = Tracer(dev)
    ds = DeviceScene(sc, dev)
    tr.build_bvh(ds.V, ds.F)
    target = tr.trace_forward(ds).rgb.clone() * 0.9
    tr = Tracer(dev)                           # a fresh context: its arena is sized by the tiny object
    opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0), seed=3)
    full = opt.V.clone()
    opt.V.copy_(full * 0.05)                   # a tiny object: the arena is sized for few segments
    opt.step(target)
    tr.get_stats()
    g = opt.capture_step(target)
    torch.cuda.synchronize()
    tr.get_stats()
    opt.V.copy_(full)                          # the captured build reads opt.V: now far more segments
    before = [t.clone() for t in (opt.V, opt.sigma, opt.ior, opt.mV, opt.vV, opt.t_dev)]
    g.replay()
    torch.cuda.synchronize()
    with pytest.raises(N.DiffTransError) as e:
        tr.get_stats()
    assert e.value.status == N.DT_ERR_RETRY
    for x, y in zip(before, (opt.V, opt.sigma, opt.ior, opt.mV, opt.vV, opt.t_dev)):
        assert torch.equal(x, y)
