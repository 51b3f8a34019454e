"""GPU-vs-oracle comparison protocol.

Forward: a pixel is path-divergent when its topology signature (tree position + event per
node) differs from the oracle's, or its radiance differs by more than RGB_TOL in any channel.
Every divergent pixel counts toward the north_star budget (at most DIV_FRAC of the compared
pixels), flagged or not.  The oracle's flags (a node within the edge band min beta < 1e-5,
a near miss or t-tie, grazing cos < 1e-3, near-TIR |q| < 1e-4) are only REPORTED: how many
pixels are flagged, how many of those diverge, and the largest error on them.
Backward: grad_rgb is zeroed on the divergent pixels only (in both runs), then rel-L2 of each
gradient block must be <= GRAD_TOL.

Every comparison appends its counts to PARITY_REPORT (a JSON-lines file, default
gpurun_out/parity_report.jsonl) so the pooled totals over a run can be checked and cited.
"""
import json
import os

import numpy as np

RGB_TOL = 1e-4      # north_star: radiance max abs 1e-4 per channel
DIV_FRAC = 1e-4     # north_star: at most 1e-4 of pixels path-divergent
GRAD_TOL = 1e-3     # north_star: gradients rel-L2 <= 1e-3
FLAG_MAX = 0.10     # sanity bound on the oracle-flagged fraction of a sample (reported only)

REPORT = os.environ.get("PARITY_REPORT", os.path.join(os.path.dirname(os.path.dirname(__file__)), "gpurun_out",
                                                      "parity_report.jsonl"))
POOL = {"n": 0, "divergent": 0}


def oracle_forward(O, osc, pixel_ids):
    """Oracle render of the pixels (flags: edge / grazing / near-TIR bands, reported only)."""
    return O.render(osc, pixel_ids)


def compare_forward(gpu_rgb, gpu_sig, orc):
    g = np.asarray(gpu_rgb, np.float64)
    o = orc["rgb"]
    sig_g = np.asarray(gpu_sig).view(np.uint64)
    sig_o = orc["sig_topo"]
    err = np.abs(g - o).max(axis=1)
    topo = sig_g != sig_o
    div = topo | ~(err <= RGB_TOL)
    flagged = orc["flags"] != 0
    n = len(err)
    out = dict(n=n, divergent=int(div.sum()), divergent_flagged=int((div & flagged).sum()),
               divergent_unflagged=int((div & ~flagged).sum()), flagged=int(flagged.sum()),
               sig_mismatch=int(topo.sum()),
               max_err=float(err.max()) if n else 0.0,
               max_err_ok=float(err[~div].max()) if (~div).any() else 0.0,
               max_err_flagged=float(err[flagged].max()) if flagged.any() else 0.0,
               p99_err=float(np.quantile(err, 0.99)) if n else 0.0,
               div_mask=div, flag_mask=flagged)
    return out


def report(label, cmp, extra=None):
    rec = {k: v for k, v in cmp.items() if "mask" not in k}
    rec["label"] = label
    if extra:
        rec.update(extra)
    try:
        os.makedirs(os.path.dirname(REPORT), exist_ok=True)
        with open(REPORT, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass
    return rec


def assert_forward(cmp, label=""):
    """Every divergent pixel (flagged or not) counts toward the budget int(DIV_FRAC n) of this
    comparison; the pooled total over the run is checked against the pooled budget too."""
    n = cmp["n"]
    rec = report(label, cmp)
    POOL["n"] += n
    POOL["divergent"] += cmp["divergent"]
    assert cmp["flagged"] <= max(FLAG_MAX * n, 1), (label, rec)
    assert cmp["divergent"] <= int(DIV_FRAC * n), (label, rec)
    assert POOL["divergent"] <= int(DIV_FRAC * POOL["n"]), (label, POOL)
    assert cmp["max_err_ok"] <= RGB_TOL, (label, rec)


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))


def grad_upstream(g, cmp):
    """The upstream gradient of a gradient comparison: zero on the path-divergent pixels only
    (they are inside the forward budget); every other pixel, flagged or not, is compared."""
    g = np.array(g, np.float32)
    g[cmp["div_mask"]] = 0.0
    return g
