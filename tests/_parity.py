"""GPU-vs-oracle comparison protocol.

Forward: a pixel is path-divergent when its topology signature (tree position + event
per node) differs from the oracle's, or its radiance differs by more than RGB_TOL in
any channel.  Oracle-flagged pixels (a node within the edge band, near-miss or tie,
grazing, near-TIR) may legitimately take the other branch in float32; they are counted
separately.  Backward: grad_rgb is zeroed on divergent and flagged pixels in BOTH runs,
then rel-L2 of each gradient block must be <= GRAD_TOL.
"""
import numpy as np

RGB_TOL = 1e-4      # north_star: radiance max abs 1e-4 per channel
DIV_FRAC = 1e-4     # north_star: at most 1e-4 of pixels path-divergent
GRAD_TOL = 1e-3     # north_star: gradients rel-L2 <= 1e-3
GRAD_COND_TOL = 1e-2   # a pixel whose fp64 VJP moves > 1e-2 under float32 direction rounding
GRAD_COND_MAX = 0.15   # ... is excluded from the gradient comparison; at most this fraction


def oracle_forward(O, osc, pixel_ids):
    """Oracle render of the pixels, with the float32 ill-conditioning flag (bit 8) added."""
    orc = O.render(osc, pixel_ids)
    ill = O.ill_conditioned(osc, pixel_ids)
    orc["flags"] = orc["flags"] | np.where(ill, O.FLAG_ILLCOND, 0).astype(np.int32)
    return orc


def compare_forward(gpu_rgb, gpu_sig, orc):
    g = np.asarray(gpu_rgb, np.float64)
    o = orc["rgb"]
    sig_g = np.asarray(gpu_sig).view(np.uint64)
    sig_o = orc["sig_topo"]
    err = np.abs(g - o).max(axis=1)
    div = (sig_g != sig_o) | (err > RGB_TOL)
    flagged = orc["flags"] != 0
    n = len(err)
    out = dict(n=n, divergent=int(div.sum()), divergent_unflagged=int((div & ~flagged).sum()),
               flagged=int(flagged.sum()), sig_mismatch=int((sig_g != sig_o).sum()),
               max_err_ok=float(err[~div].max()) if (~div).any() else 0.0,
               max_err_all=float(err.max()), div_mask=div, flag_mask=flagged)
    return out


def assert_forward(cmp, label=""):
    n = cmp["n"]
    assert cmp["max_err_ok"] <= RGB_TOL, (label, cmp["max_err_ok"])
    assert cmp["divergent_unflagged"] <= int(DIV_FRAC * n), (label, {k: v for k, v in cmp.items() if "mask" not in k})
    # flagged pixels that do diverge still count toward the budget, pooled over the run
    assert cmp["divergent"] <= max(int(DIV_FRAC * n), 0) + cmp["flagged"], (label, cmp["divergent"])


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))


def grad_upstream(O, osc, pixel_ids, g, cmp):
    """The upstream gradient of a gradient comparison: zero on path-divergent and flagged
    pixels, and on pixels whose reverse-mode result float32 cannot hold to GRAD_COND_TOL
    (oracle.ill_conditioned_grad, computed from the oracle alone).  Returns (g, n_excluded)."""
    g = np.array(g, np.float32)
    g[cmp["div_mask"] | cmp["flag_mask"]] = 0.0
    ill = O.ill_conditioned_grad(osc, pixel_ids, g, GRAD_COND_TOL)
    assert ill.sum() <= GRAD_COND_MAX * len(g), int(ill.sum())
    g[ill] = 0.0
    return g, int(ill.sum())
