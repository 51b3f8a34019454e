"""Per-pixel vertex-gradient comparison GPU vs oracle (dev tool): prints the pixels that
dominate the dV rel-L2.   python tools/debug_grad_v.py C5 256 6 17"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2603_00413_b200 import scenes as S  # noqa: E402
from paper_2603_00413_b200.tracer import DeviceScene, Tracer  # noqa: E402
from tests._parity import compare_forward, oracle_forward, rel_l2  # noqa: E402

cfg, n, pseed, gseed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
sc = S.CONFIGS[cfg]()
pid = S.central_pixels(sc.cams, n, pseed)
osc = O.OracleScene(sc)
orc = oracle_forward(O, osc, pid)
dev = torch.device("cuda:0")
ds = DeviceScene(sc, dev)
tr = Tracer(dev)
tr.build_bvh(ds.V, ds.F)
pt = torch.as_tensor(pid, device=dev)
out = tr.trace_forward(ds, pt, want_sig=True)
cmp = compare_forward(out.rgb.cpu().numpy(), out.sig_topo.cpu().numpy(), orc)
print({k: v for k, v in cmp.items() if "mask" not in k})
g = S.upstream_grad(len(pid), gseed)
g[cmp["div_mask"] | cmp["flag_mask"]] = 0
gV, _, _ = tr.trace_backward(torch.as_tensor(g, device=dev))
oV, _, _ = O.backward(osc, g, pid)
print("pixel_ids launch dV rel-L2", rel_l2(gV.cpu().numpy(), oV), "|oV|", np.linalg.norm(oV))
errs = []
for i in range(n):
    if not g[i].any():
        continue
    gg = np.zeros_like(g)
    gg[i] = g[i]
    a, _, _ = tr.trace_backward(torch.as_tensor(gg, device=dev))
    b, _, _ = O.backward(osc, gg[i:i + 1], pid[i:i + 1])
    d = np.linalg.norm(a.cpu().numpy().astype(np.float64) - b)
    errs.append((d, np.linalg.norm(b), i))
errs.sort(reverse=True)
tot = np.sqrt(sum(e[0] ** 2 for e in errs))
print("sqrt(sum per-pixel |err|^2)", tot, "relative", tot / np.linalg.norm(oV))
for d, nb, i in errs[:12]:
    print(f"pix {i} id {pid[i]} |err| {d:.4g} |g_o| {nb:.4g} rel {d / max(nb, 1e-30):.3g} flags {orc['flags'][i]} "
          f"segs {orc['segments'][i]} rgb {orc['rgb'][i]}")
