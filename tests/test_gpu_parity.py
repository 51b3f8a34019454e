"""GPU parity: libdifftrans (through the C ABI) against the fp64 oracle, same seeded inputs.

Bars (north_star): hit ids bit-exact vs brute force (ties excluded); radiance max-abs
<= 1e-4 with <= 1e-4 of pixels path-divergent; gradients rel-L2 <= 1e-3.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T
from tests._parity import GRAD_TOL, assert_forward, compare_forward, grad_upstream, oracle_forward, rel_l2, report

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tracer():
    from paper_2603_00413_b200.tracer import Tracer
    return Tracer("cuda:0")


def run_gpu(tracer, sc, pixel_ids=None, grad=None, full_launch_grad=None):
    from paper_2603_00413_b200.tracer import DeviceScene
    ds = DeviceScene(sc, torch.device("cuda:0"))
    tracer.build_bvh(ds.V, ds.F)
    pid_t = None if pixel_ids is None else torch.as_tensor(pixel_ids, dtype=torch.int64, device="cuda:0")
    out = tracer.trace_forward(ds, pid_t, want_capped=True, want_sig=True, stats=True)
    res = dict(rgb=out.rgb.cpu().numpy(), sig=out.sig_topo.cpu().numpy(), capw=out.capped_w.cpu().numpy(),
               stats=out.stats)
    g = grad if grad is not None else full_launch_grad
    if g is not None:
        gV, gi, gs = tracer.trace_backward(torch.as_tensor(g, dtype=torch.float32, device="cuda:0").contiguous())
        res.update(gV=gV.cpu().numpy(), gior=float(gi.cpu()[0]), gsig=gs.cpu().numpy())
    torch.cuda.synchronize()
    return res


def parity_case(tracer, sc, pixel_ids, label, grad_seed=11):
    """Forward + backward parity on the given pixels (pixel_ids launch)."""
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pixel_ids)
    gpu = run_gpu(tracer, sc, pixel_ids)
    cmp = compare_forward(gpu["rgb"], gpu["sig"], orc)
    assert_forward(cmp, label)
    # capped weight (a diagnostic output: the sum of the capped branches' R/T path weights)
    ok = ~cmp["div_mask"]
    if ok.any():
        assert np.abs(gpu["capw"][ok] - orc["capped_w"][ok]).max() <= 1e-4, label
    g = grad_upstream(S.upstream_grad(len(pixel_ids), grad_seed), cmp)
    gpu = run_gpu(tracer, sc, pixel_ids, grad=g)
    gV, gi, gs = O.backward(osc, g, pixel_ids)
    errs = dict(V=rel_l2(gpu["gV"], gV), sigma=rel_l2(gpu["gsig"], gs))
    # scalar blocks (IOR; constant sigma): a single sum of random-sign per-pixel terms can
    # cancel to ~0, so compare the vector of per-group partial gradients instead
    errs["ior"], es = scalar_block_errors(tracer, osc, pixel_ids, g, sc.absorption.kind == S.ABS_CONST)
    if es is not None:
        errs["sigma_groups"] = es
    report(label + " grad", {"n": len(pixel_ids)}, {k: float(e) for k, e in errs.items()})
    for k, e in errs.items():
        assert e <= GRAD_TOL, (label, k, errs)
    return cmp, errs, gpu["stats"]


def scalar_block_errors(tracer, osc, pixel_ids, g, const_sigma, n_groups=32, n_full=None):
    """rel-L2 over per-group partial gradients of the scalar blocks.  n_full: the forward was
    a full-image launch of n_full rays and pixel_ids index into it."""
    groups = np.array_split(np.arange(len(pixel_ids)), min(n_groups, len(pixel_ids)))
    gi_g, gi_o, gs_g, gs_o = [], [], [], []
    for grp in groups:
        gg = np.zeros_like(g)
        gg[grp] = g[grp]
        if n_full is None:
            gdev = gg
        else:
            gdev = np.zeros((n_full, 3), np.float32)
            gdev[np.asarray(pixel_ids)] = gg
        _, a, b = tracer.trace_backward(torch.as_tensor(gdev, dtype=torch.float32, device="cuda:0"))
        _, oi, os_ = O.backward(osc, gg[grp], np.asarray(pixel_ids)[grp])
        gi_g.append(float(a.cpu()[0]))
        gi_o.append(oi)
        if const_sigma:
            gs_g.append(b.cpu().numpy())
            gs_o.append(os_)
    return rel_l2(gi_g, gi_o), (rel_l2(np.array(gs_g), np.array(gs_o)) if const_sigma else None)


# ----------------------------------------------------------------------------- BVH
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_bvh_structure_and_bit_exact_vs_brute_force(tracer, cfg):
    sc = S.CONFIGS[cfg]() if cfg in ("C1", "C2") else None
    if cfg == "C3":
        V, F = S.cube_sphere(204, 3)
    elif cfg == "C5":
        V, F = S.cube_sphere(289, 5)
    elif cfg == "C4":
        V, F = S.knot_and_gems(4)
    else:
        V, F = sc.V, sc.F
    Vt = torch.as_tensor(V, device="cuda:0")
    Ft = torch.as_tensor(F, device="cuda:0")
    tracer.build_bvh(Vt, Ft)
    chk = tracer.bvh_check()
    assert chk["bad_boxes"] == 0 and chk["leaves"] == F.shape[0] and chk["distinct_faces"] == F.shape[0], chk
    assert chk["depth"] < 128
    g = np.random.default_rng(5)
    n = 20000 if cfg != "C1" else 5000
    r = 1.3 * np.abs(V).max()
    o = g.normal(size=(n, 3))
    o = o / np.linalg.norm(o, axis=1, keepdims=True) * r * g.uniform(1.0, 3.0, (n, 1))
    tgt = g.uniform(-0.8, 0.8, (n, 3)) * np.abs(V).max()
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    inner = g.uniform(-0.3, 0.3, (n // 4, 3))            # rays starting inside the object
    din = g.normal(size=(n // 4, 3))
    din /= np.linalg.norm(din, axis=1, keepdims=True)
    rays = np.concatenate([np.concatenate([o, d], 1), np.concatenate([inner, din], 1)]).astype(np.float32)
    rt = torch.as_tensor(rays, device="cuda:0")
    for t_lo in (0.0, 1e-4):
        f_bvh, tuv_bvh = tracer.closest_hit(rt, t_lo, brute_force=False)
        f_bf, tuv_bf = tracer.closest_hit(rt, t_lo, brute_force=True)
        assert torch.equal(f_bvh, f_bf)
        assert torch.equal(tuv_bvh.view(torch.int32), tuv_bf.view(torch.int32))   # bit-exact t, u, v
    # against the fp64 oracle brute force: identical face ids except flagged ties / edges
    m = 3000 if cfg in ("C3", "C4") else 1500 if cfg == "C5" else len(rays)
    osc = O.OracleScene(S.Scene("t", V, F, 1.5, S.const_absorption(), S.analytic_env(1),
                                T.one_view(2, 2, (0, 0, 3)), 2))
    f_o, tuv_o, fl = O.closest_hit(osc, rays[:m].astype(np.float64))
    f_g = f_bvh.cpu().numpy()[:m]
    # the candidate search is float32 (the shade pass then recomputes the chosen face's hit in
    # float64): its barycentric rounding on these triangles (edges ~1e-2 of |o|) reaches ~1e-5,
    # so rays within 1e-4 of an edge, or flagged by the oracle (near miss / tie), may pick the
    # neighbouring face; every other ray must pick the oracle's face
    mb = np.minimum(np.minimum(1 - tuv_o[:, 1] - tuv_o[:, 2], tuv_o[:, 1]), tuv_o[:, 2])
    ok = (fl == 0) & ((f_o < 0) | (mb >= 1e-4))
    assert ok.mean() > 0.97, ok.mean()
    assert (f_g[ok] == f_o[ok]).all(), int((f_g[ok] != f_o[ok]).sum())
    hit = ok & (f_o >= 0)
    np.testing.assert_allclose(tuv_bvh.cpu().numpy()[:m][hit, 0], tuv_o[hit, 0], rtol=2e-5, atol=2e-5)


def test_vertex_normals_match_oracle(tracer):
    sc = S.config_c2()
    tracer.build_bvh(torch.as_tensor(sc.V, device="cuda:0"), torch.as_tensor(sc.F, device="cuda:0"))
    n = tracer.vertex_normals(sc.V.shape[0]).cpu().numpy()
    no = O.vertex_normals(O.OracleScene(sc))
    assert np.abs(n - no).max() < 2e-6


# ----------------------------------------------------------------------------- forward + backward
def test_c1_full_image(tracer):
    sc = S.config_c1()
    cmp, errs, st = parity_case(tracer, sc, np.arange(sc.n_pixels), "C1")
    assert cmp["sig_mismatch"] == 0 and cmp["divergent_unflagged"] == 0


def test_c1_axis_pixel_slab_series(tracer):
    """The C1 axis pixel reproduces the oracle-pinned slab series on the GPU."""
    sc = S.config_c1()
    gpu = run_gpu(tracer, sc, np.array([31 * 64 + 31]))
    orc = O.render(O.OracleScene(sc), [31 * 64 + 31])
    np.testing.assert_allclose(gpu["rgb"][0], orc["rgb"][0], atol=2e-6)


@pytest.mark.parametrize("D,cap", [(0, S.CAP_ZERO), (1, S.CAP_ENV), (4, S.CAP_ZERO), (5, S.CAP_ENV)])
def test_c1_depths_and_cap_policies(tracer, D, cap):
    base = S.config_c1()
    sc = T.scene(base.V, base.F, base.cams, env=base.env, D=D, cap=cap)
    parity_case(tracer, sc, np.arange(sc.n_pixels), f"C1-D{D}-cap{cap}")


def test_c2_grid_env_sampled_pixels(tracer):
    sc = S.config_c2()
    pid = S.central_pixels(sc.cams, 2048, 2)
    cmp, errs, st = parity_case(tracer, sc, pid, "C2")


def test_c2_full_launch_sampled_compare(tracer):
    """Full-image launch (the bench's configuration); compare 2048 sampled pixels, and the
    gradient of a loss living only on those pixels."""
    sc = S.config_c2()
    pid = S.central_pixels(sc.cams, 2048, 3)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    gpu = run_gpu(tracer, sc, None)
    cmp = compare_forward(gpu["rgb"][pid], gpu["sig"][pid], orc)
    assert_forward(cmp, "C2-full")
    gfull = np.zeros((sc.n_pixels, 3), np.float32)
    g = grad_upstream(S.upstream_grad(len(pid), 12), cmp)
    gfull[pid] = g
    gpu = run_gpu(tracer, sc, None, full_launch_grad=gfull)
    gV, gi, gs = O.backward(osc, g, pid)
    e_v = rel_l2(gpu["gV"], gV)
    e_ior, e_sig = scalar_block_errors(tracer, osc, pid, g, True, n_full=sc.n_pixels)
    report("C2-full grad", {"n": len(pid)}, {"V": e_v, "ior": e_ior, "sigma_groups": e_sig})
    assert e_v <= GRAD_TOL and e_ior <= GRAD_TOL and e_sig <= GRAD_TOL, (e_v, e_ior, e_sig)


def test_sigma_grid_and_far_field(tracer):
    V, F = S.icosphere(2)
    cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)           # ragged 8x4 tiles
    sc = T.scene(V, F, cams, env=T.small_grid_env(far_field=1), absorption=T.small_sigma_grid(V, 8), D=4)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-sigmagrid-farfield")
    sc = T.scene(V, F, cams, env=T.small_grid_env(far_field=0), absorption=T.small_sigma_grid(V, 8), D=3,
                 cap=S.CAP_ENV)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-sigmagrid-capenv")


def test_hash_texture(tracer):
    """NEXT-2: hash-grid absorption (R29), dense and hashed (colliding) levels, both caps."""
    V, F = S.icosphere(2)
    cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
    ab = T.small_hash_grid(V, levels=4, log2_size=8, base=2, top=16, n_samples=24)
    sc = T.scene(V, F, cams, env=T.small_grid_env(far_field=1), absorption=ab, D=4)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-hash")
    sc = T.scene(V, F, cams, env=T.lobe_env(kappa=3.0), absorption=ab, D=3, cap=S.CAP_ENV)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-hash-capenv")


def test_volume_env(tracer):
    """NEXT-3: volumetric env (R30) -- exterior segments volume rendered, escaping rays to the
    shell; both cap policies, with a sigma grid inside."""
    V, F = S.icosphere(2)
    cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
    sc = T.scene(V, F, cams, env=T.small_volume_env(), D=4)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-volenv")
    sc = T.scene(V, F, cams, env=T.small_volume_env(seed=9, density=0.3), absorption=T.small_sigma_grid(V, 6), D=3,
                 cap=S.CAP_ENV)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "ico2-volenv-capenv-grid")


def test_c3v_volume_env_full_size_sampled(tracer):
    """NEXT-3 workload at full size (bench launch), 128 sampled object pixels."""
    sc = S.config_c3v()
    pid = S.central_pixels(sc.cams, 128, 6)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    gpu = run_gpu(tracer, sc, None)
    cmp = compare_forward(gpu["rgb"][pid], gpu["sig"][pid], orc)
    assert_forward(cmp, "C3V")
    gfull = np.zeros((sc.n_pixels, 3), np.float32)
    g = grad_upstream(S.upstream_grad(len(pid), 17), cmp)
    gfull[pid] = g
    gpu = run_gpu(tracer, sc, None, full_launch_grad=gfull)
    gV, gi, gs = O.backward(osc, g, pid)
    e_v = rel_l2(gpu["gV"], gV)
    report("C3V grad", {"n": len(pid)}, {"V": e_v})
    assert e_v <= GRAD_TOL, e_v


def test_hash_dense_level_equals_grid(tracer):
    """One dense hash level is the vertex grid (R29 special case): same radiance/gradients."""
    import dataclasses
    V, F = S.icosphere(2)
    cams = T.one_view(32, 32, (0.5, 0.3, 2.7), fov_deg=50)
    grid = T.small_sigma_grid(V, 8)
    R = grid.sigma.shape[0]
    tab = np.zeros((1, 1024, 3), np.float32)
    tab[0, :R ** 3] = grid.sigma.reshape(-1, 3)
    hashed = S.Absorption(S.ABS_HASH, tab, grid.box_lo, grid.box_hi, grid.n_samples, np.array([R - 1], np.int32))
    a = T.scene(V, F, cams, env=T.lobe_env(kappa=3.0), absorption=grid, D=4)
    b = dataclasses.replace(a, absorption=hashed)
    g = S.upstream_grad(a.n_pixels, 21)
    ra = run_gpu(tracer, a, np.arange(a.n_pixels), grad=g)
    rb = run_gpu(tracer, b, np.arange(b.n_pixels), grad=g)
    np.testing.assert_allclose(rb["rgb"], ra["rgb"], atol=2e-5)
    assert rel_l2(rb["gV"], ra["gV"]) < 1e-4
    assert rel_l2(rb["gsig"][0, :R ** 3], ra["gsig"].reshape(-1, 3)) < 1e-4
    assert np.abs(rb["gsig"][0, R ** 3:]).max() == 0.0


@pytest.mark.parametrize("log2_size,n_pix", [(16, 128), (19, 48)])
def test_c4h_hash_texture_full_mesh_sampled(tracer, log2_size, n_pix):
    """NEXT-2 workload: C4's knot + gems with the 16-level hash texture, sampled pixels; the
    2^19-entry table is the bench's (fewer pixels: the oracle keeps a per-thread float64
    adjoint of the whole table)."""
    sc = S.config_c4h(log2_size=log2_size)
    pid = S.central_pixels(sc.cams, n_pix, 7)
    parity_case(tracer, sc, pid, f"C4H-2^{log2_size}")


def test_flat_facets_and_tir(tracer):
    """Unwelded flat gems (flat normals, TIR-rich) and the tetrahedron."""
    Vg, Fg = S.gem()
    cams = T.one_view(48, 48, (0.3, 0.5, 2.8), fov_deg=50)
    sc = T.scene(Vg.astype(np.float32), Fg, cams, env=T.lobe_env(kappa=4.0), ior=2.4, D=6)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "gem")
    Vt, Ft = S.tetrahedron()
    sc = T.scene(Vt, Ft, cams, env=T.small_grid_env(), D=3)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "tet")


def test_c3_full_size_sampled(tracer):
    """BASELINE configs[2] at full size in the bench's launch configuration (all 64M rays of
    100 views x 800^2, D 4); 256 sampled object pixels against the oracle."""
    sc = S.config_c3()
    pid = S.central_pixels(sc.cams, 256, 3)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    gpu = run_gpu(tracer, sc, None)
    cmp = compare_forward(gpu["rgb"][pid], gpu["sig"][pid], orc)
    assert_forward(cmp, "C3")
    gfull = np.zeros((sc.n_pixels, 3), np.float32)
    g = grad_upstream(S.upstream_grad(len(pid), 13), cmp)
    gfull[pid] = g
    gpu = run_gpu(tracer, sc, None, full_launch_grad=gfull)
    gV, gi, gs = O.backward(osc, g, pid)
    e_v = rel_l2(gpu["gV"], gV)
    e_ior, e_sig = scalar_block_errors(tracer, osc, pid, g, True, n_full=sc.n_pixels)
    report("C3 grad", {"n": len(pid)}, {"V": e_v, "ior": e_ior, "sigma_groups": e_sig})
    assert e_v <= GRAD_TOL and e_ior <= GRAD_TOL and e_sig <= GRAD_TOL, (e_v, e_ior, e_sig)


def test_c5_full_size_sampled(tracer):
    """BASELINE configs[4], the largest single-GPU launch: 1M triangles, all 209,715,200 rays of
    200 views x 1024^2 at D 4; 256 sampled object pixels against the oracle (forward and the
    gradient of a loss living on those pixels, same full launch)."""
    sc = S.config_c5()
    pid = S.central_pixels(sc.cams, 256, 6)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    gpu = run_gpu(tracer, sc, None)
    cmp = compare_forward(gpu["rgb"][pid], gpu["sig"][pid], orc)
    assert_forward(cmp, "C5")
    gfull = np.zeros((sc.n_pixels, 3), np.float32)
    g = grad_upstream(S.upstream_grad(len(pid), 17), cmp)
    gfull[pid] = g
    gpu = run_gpu(tracer, sc, None, full_launch_grad=gfull)
    del gfull
    gV, gi, gs = O.backward(osc, g, pid)
    e_v = rel_l2(gpu["gV"], gV)
    e_ior, e_sig = scalar_block_errors(tracer, osc, pid, g, True, n_groups=8, n_full=sc.n_pixels)
    report("C5 grad", {"n": len(pid)}, {"V": e_v, "ior": e_ior, "sigma_groups": e_sig})
    assert e_v <= GRAD_TOL and e_ior <= GRAD_TOL and e_sig <= GRAD_TOL, (e_v, e_ior, e_sig)


def test_c3r_relighting_depth8_full_size_sampled(tracer):
    """NEXT-3 inference workload: C3's mesh under a swapped env at D_max = 8, the bench's
    full-image forward launch; 256 sampled object pixels against the oracle."""
    sc = S.config_c3r()
    pid = S.central_pixels(sc.cams, 256, 5)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    gpu = run_gpu(tracer, sc, None)
    cmp = compare_forward(gpu["rgb"][pid], gpu["sig"][pid], orc)
    assert_forward(cmp, "C3R")
    assert gpu["stats"]["segments_per_depth"][8] > 0


def test_c4_sigma_grid_full_mesh_sampled(tracer):
    """BASELINE configs[3]: knot + gems, 64^3 sigma grid, D 6; 256 sampled pixels."""
    sc = S.config_c4()
    pid = S.central_pixels(sc.cams, 256, 4)
    parity_case(tracer, sc, pid, "C4")


# ----------------------------------------------------------------------------- edge cases
def test_edge_cases(tracer):
    from paper_2603_00413_b200.tracer import DeviceScene
    from paper_2603_00413_b200._native import DiffTransError
    # one-triangle mesh, ragged image
    V = np.array([[-1, -1, 0], [1, -1, 0], [0, 1, 0]], np.float32)
    F = np.array([[0, 1, 2]], np.int32)
    sc = T.scene(V, F, T.one_view(13, 7, (0.1, 0.2, 3.0)), env=T.lobe_env(), D=3)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "one-tri")
    # empty pixel list
    ds = DeviceScene(S.config_c1(), torch.device("cuda:0"))
    tracer.build_bvh(ds.V, ds.F)
    out = tracer.trace_forward(ds, torch.zeros(0, dtype=torch.int64, device="cuda:0"))
    assert out.rgb.shape == (0, 3)
    gV, gi, gs = tracer.trace_backward(torch.zeros((0, 3), device="cuda:0"))
    assert float(gV.abs().max()) == 0.0
    # duplicated pixels give identical radiance
    pid = torch.tensor([100, 2080, 100, 2080], dtype=torch.int64, device="cuda:0")
    out = tracer.trace_forward(ds, pid)
    assert torch.equal(out.rgb[0], out.rgb[2]) and torch.equal(out.rgb[1], out.rgb[3])
    # errors are loud
    with pytest.raises(DiffTransError, match="EMPTY_GEOMETRY"):
        tracer.build_bvh(torch.zeros((0, 3), device="cuda:0"), torch.zeros((0, 3), dtype=torch.int32, device="cuda:0"))
    with pytest.raises(DiffTransError, match="INVALID_ARG"):
        tracer.build_bvh(ds.V, ds.F)
        tracer.trace_forward(ds, max_depth=99)


def test_forward_deterministic(tracer):
    from paper_2603_00413_b200.tracer import DeviceScene
    ds = DeviceScene(S.config_c2(), torch.device("cuda:0"))
    tracer.build_bvh(ds.V, ds.F)
    a = tracer.trace_forward(ds, want_sig=True).rgb.clone()
    tracer.build_bvh(ds.V, ds.F)
    b = tracer.trace_forward(ds, want_sig=True).rgb
    assert torch.equal(a, b)


def test_async_forward_matches_and_reports_overflow(tracer):
    """opts.async: identical results to the synchronous forward; an arena overflow of an
    asynchronous forward is reported by the next call as DT_ERR_RETRY, after which the
    step re-runs correctly."""
    from paper_2603_00413_b200.tracer import DeviceScene, Tracer
    from paper_2603_00413_b200._native import DiffTransError
    tr = Tracer("cuda:0")
    sc = S.config_c2()
    ds = DeviceScene(sc, torch.device("cuda:0"))
    tr.build_bvh(ds.V, ds.F)
    ref = tr.trace_forward(ds).rgb.clone()
    g = torch.as_tensor(S.upstream_grad(sc.n_pixels, 3), device="cuda:0")
    gV_ref = tr.trace_backward(g)[0].clone()
    for _ in range(2):
        tr.build_bvh(ds.V, ds.F)
        out = tr.trace_forward(ds, async_=True)
        gV = tr.trace_backward(g)[0]
    torch.cuda.synchronize()
    assert torch.equal(out.rgb, ref)
    assert float((gV - gV_ref).norm() / gV_ref.norm()) < 1e-5      # float atomics: ulp-level order noise
    st = tr.get_stats()
    assert st["segments"] > 0
    # shrink the object so the next synchronous forward measures a small need, then trace
    # the full object asynchronously: the arena (sized from the small need) overflows
    # (depth 8 makes the full object need more records than the initial 3 per ray)
    ref8 = tr.trace_forward(ds, max_depth=8).rgb.clone()
    small = DeviceScene(sc, torch.device("cuda:0"))
    small.set_vertices(ds.V * 0.05)
    tr2 = Tracer("cuda:0")
    tr2.build_bvh(small.V, small.F)
    tr2.trace_forward(small, max_depth=8)
    tr2.build_bvh(ds.V, ds.F)
    tr2.trace_forward(ds, max_depth=8, async_=True)
    with pytest.raises(DiffTransError, match="RETRY"):
        tr2.get_stats()
    tr2.build_bvh(ds.V, ds.F)
    again = tr2.trace_forward(ds, max_depth=8, async_=True).rgb
    torch.cuda.synchronize()
    tr2.get_stats()
    assert torch.equal(again, ref8)


def test_loss_color_kernel(tracer):
    rgb = torch.tensor([[1.1, 1.1, 1.1]], device="cuda:0")
    tgt = torch.ones((1, 3), device="cuda:0")
    loss, g = tracer.loss_color(rgb, tgt)
    assert abs(float(loss) - 0.03) < 1e-6                              # S: l_color example
    x = torch.rand((1000, 3), device="cuda:0")
    c = torch.rand((1000, 3), device="cuda:0")
    loss, g = tracer.loss_color(x, c)
    ref = (((x - c) * c) ** 2).sum() / 1000
    assert abs(float(loss) - float(ref)) < 1e-5 * float(ref)
    assert torch.allclose(g, 2 * (x - c) * c * c / 1000, atol=1e-7)


def test_context_reuse_across_kinds(tracer):
    """One context serving scenes of different absorption / env kinds in turn (arena lanes for
    the volume moments appear on demand, the sigma snapshot is re-laid out) gives the same
    results as fresh contexts."""
    from paper_2603_00413_b200.tracer import Tracer
    V, F = S.icosphere(2)
    cams = T.one_view(24, 20, (0.5, 0.3, 2.7), fov_deg=55)
    scenes = [T.scene(V, F, cams, env=T.small_grid_env(), D=3),
              T.scene(V, F, cams, env=T.small_volume_env(), absorption=T.small_sigma_grid(V, 6), D=3),
              T.scene(V, F, cams, env=T.lobe_env(), absorption=T.small_hash_grid(V, levels=3, log2_size=6), D=3),
              T.scene(V, F, cams, env=T.small_grid_env(), D=3)]
    pid = np.arange(scenes[0].n_pixels)
    for sc in scenes:
        g = S.upstream_grad(len(pid), 5)
        shared = run_gpu(tracer, sc, pid, grad=g)
        fresh = run_gpu(Tracer("cuda:0"), sc, pid, grad=g)
        np.testing.assert_array_equal(shared["rgb"], fresh["rgb"])
        assert rel_l2(shared["gV"], fresh["gV"]) < 1e-5 and rel_l2(shared["gsig"], fresh["gsig"]) < 1e-5


def test_degenerate_method_cases(tracer):
    """Degenerate cases of the method, each against the oracle: (a) eta = 1 and sigma = 0
    (optical absence: R = 0 everywhere, the reflect child still spawned with weight 0, R5);
    (b) zero-area faces in the mesh (a repeated vertex index and three collinear vertices:
    no hit, no contribution to the vertex normals, R6, R16); (c) the camera inside the object
    (every camera hit is an inside hit: refraction out or TIR, R8)."""
    base = S.config_c1()
    sc = T.scene(base.V, base.F, base.cams, env=base.env, ior=1.0, sigma=(0.0, 0.0, 0.0), D=3)
    pid = np.arange(sc.n_pixels)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    cmp = compare_forward(run_gpu(tracer, sc, pid)["rgb"], run_gpu(tracer, sc, pid)["sig"], orc)
    assert_forward(cmp, "eta1")
    # the exact vertex gradient is 0 here (the radiance no longer depends on the geometry), so
    # rel-L2 has no denominator: the error is measured against the gradient scale of the same
    # scene at eta = 1.5, sigma = 0 (same upstream gradient)
    g = grad_upstream(S.upstream_grad(len(pid), 11), cmp)
    gpu = run_gpu(tracer, sc, pid, grad=g)
    gV, _, _ = O.backward(osc, g, pid)
    ref = T.scene(base.V, base.F, base.cams, env=base.env, ior=1.5, sigma=(0.0, 0.0, 0.0), D=3)
    gref, _, _ = O.backward(O.OracleScene(ref), g, pid)
    assert np.linalg.norm(gV) <= 1e-9 * np.linalg.norm(gref)
    assert np.linalg.norm(gpu["gV"] - gV) <= 1e-3 * np.linalg.norm(gref), np.linalg.norm(gpu["gV"] - gV)
    V, F = S.icosphere(1)
    # exactly collinear in float32 and float64 (A, 1.5 A, 2 A with dyadic A), so the face's cross
    # product is 0 in both and its three vertices are isolated (normal (0, 0, 1), R6)
    A = np.array([0.25, 0.125, 0.0625])
    V = np.concatenate([V, [A, 1.5 * A, 2.0 * A]]).astype(np.float32)
    nv = V.shape[0]
    F = np.concatenate([F, [[0, 0, 5], [nv - 3, nv - 2, nv - 1]]]).astype(np.int32)
    sc = T.scene(V, F, T.one_view(24, 20, (0.3, -0.4, 3.0)), env=T.lobe_env(), D=3)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "zero-area")
    Vt, Ft = torch.as_tensor(V, device="cuda:0"), torch.as_tensor(F, device="cuda:0")
    tracer.build_bvh(Vt, Ft)
    n = tracer.vertex_normals(nv).cpu().numpy()
    osc = O.OracleScene(sc)
    np.testing.assert_allclose(n, O.vertex_normals(osc), atol=1e-5)   # the three extra vertices: (0, 0, 1)
    V, F = S.icosphere(2)
    sc = T.scene(V, F, T.one_view(20, 16, (0.0, 0.0, 0.3), fov_deg=70.0, target=(1.0, 0.2, 0.3)), env=T.lobe_env(), D=4)
    parity_case(tracer, sc, np.arange(sc.n_pixels), "camera-inside")


@pytest.mark.parametrize("quality", [0, 1, 4])
def test_bvh_quality_levels_same_hits(tracer, quality):
    """dt_set_bvh_quality: every treelet-restructuring level gives a valid tree (boxes contain
    their children, every face reached once) and closest hits bit-identical to brute force."""
    from paper_2603_00413_b200.tracer import DeviceScene
    sc = S.config_c2()
    ds = DeviceScene(sc, torch.device("cuda:0"))
    tracer.set_bvh_quality(quality)
    try:
        tracer.build_bvh(ds.V, ds.F)
        chk = tracer.bvh_check()
        assert chk["bad_boxes"] == 0 and chk["leaves"] == sc.F.shape[0] and chk["distinct_faces"] == sc.F.shape[0]
        g = torch.Generator(device="cuda:0")
        g.manual_seed(quality + 5)
        rays = torch.randn(20000, 6, device="cuda:0", generator=g)
        rays[:, :3] *= 0.4
        f1, t1 = tracer.closest_hit(rays, 1e-4, brute_force=False)
        f2, t2 = tracer.closest_hit(rays, 1e-4, brute_force=True)
        assert torch.equal(f1, f2) and torch.equal(t1, t2)
    finally:
        tracer.set_bvh_quality(2)


def test_walk_counters(tracer):
    """Device walk counters behind the texture walks' roofline (bench.py): zero for a constant
    sigma; for a sigma grid the backward replays the forward's walks with the same lane groups,
    so both count the same cell visits, at most nsamp per traced segment."""
    from paper_2603_00413_b200.tracer import DeviceScene
    V, F = S.icosphere(2)
    cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
    for ab, walks in ((None, False), (T.small_sigma_grid(V, 8), True)):
        kw = {} if ab is None else {"absorption": ab}
        sc = T.scene(V, F, cams, env=T.small_grid_env(far_field=1), D=4, **kw)
        ds = DeviceScene(sc, torch.device("cuda:0"))
        tracer.build_bvh(ds.V, ds.F)
        tracer.profile(reset=True)
        tracer.trace_forward(ds, None)
        tracer.trace_backward(torch.ones((sc.n_pixels, 3), dtype=torch.float32, device="cuda:0"))
        torch.cuda.synchronize()
        p = tracer.profile(reset=True)
        if not walks:
            assert p["walk_cells_fwd"] == 0 and p["walk_cells_bwd"] == 0, p
        else:
            assert 0 < p["walk_cells_fwd"] == p["walk_cells_bwd"] <= p["segments"] * sc.absorption.n_samples, p


def test_env_volume_sample_counter(tracer):
    """The volumetric env's backward sample counter (bench.py roofline): every exterior segment
    replays env_nsamp samples, so the count is a positive multiple of env_nsamp, at most
    segments * env_nsamp; zero for the shell env."""
    from paper_2603_00413_b200.tracer import DeviceScene
    V, F = S.icosphere(2)
    cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
    for env, vol in ((T.small_grid_env(far_field=1), False), (T.small_volume_env(), True)):
        sc = T.scene(V, F, cams, env=env, D=3)
        ds = DeviceScene(sc, torch.device("cuda:0"))
        tracer.build_bvh(ds.V, ds.F)
        tracer.profile(reset=True)
        tracer.trace_forward(ds, None)
        tracer.trace_backward(torch.ones((sc.n_pixels, 3), dtype=torch.float32, device="cuda:0"))
        torch.cuda.synchronize()
        p = tracer.profile(reset=True)
        if not vol:
            assert p["env_samples_bwd"] == 0, p
        else:
            m = sc.env.n_samples
            assert 0 < p["env_samples_bwd"] <= p["segments"] * m and p["env_samples_bwd"] % m == 0, p
