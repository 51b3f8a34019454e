"""Per-pixel gradient comparison GPU vs oracle (dev tool): prints the worst pixels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2603_00413_b200 import scenes as S
from paper_2603_00413_b200.tracer import DeviceScene, Tracer
from tests._parity import oracle_forward, compare_forward

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
sc = S.CONFIGS[cfg]()
pid = S.central_pixels(sc.cams, n, 4)
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
g = S.upstream_grad(len(pid), 11)
g[cmp["div_mask"] | cmp["flag_mask"]] = 0
gi_gpu = np.zeros(n); gi_orc = np.zeros(n)
for i in range(n):
    gg = np.zeros_like(g); gg[i] = g[i]
    _, gi, _ = tr.trace_backward(torch.as_tensor(gg, device=dev))
    gi_gpu[i] = float(gi.cpu()[0])
    _, oi, _ = O.backward(osc, gg[i:i+1], pid[i:i+1])
    gi_orc[i] = oi
err = np.abs(gi_gpu - gi_orc)
print("total", gi_gpu.sum(), gi_orc.sum(), "rel", abs(gi_gpu.sum()-gi_orc.sum())/abs(gi_orc.sum()))
for i in np.argsort(-err)[:10]:
    print(i, pid[i], gi_gpu[i], gi_orc[i], err[i], orc["flags"][i], orc["segments"][i])
