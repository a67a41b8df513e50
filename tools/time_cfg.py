"""Time forward / inverse of a config with CUDA events (no ncu): python tools/time_cfg.py C3 [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = get_config(name)
nlim = int(os.environ.get("NLIM", "0"))
if nlim:
    cfg = cfg.with_(N=min(cfg.N, nlim))
x = torch.from_numpy(generate(cfg)).cuda()
g, gd = P.gaussian_window(cfg.L, cfg.sigma)
plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom,
              gamma=1e-6 * float(np.sum(g)) * float(x.abs().max()))
T = torch.empty((plan.frames, plan.bins), dtype=torch.complex64, device="cuda")
y = torch.empty(cfg.N, dtype=torch.float32, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for _ in range(2):
    plan.forward(x, out=T)
    plan.inverse(T, out=y)
torch.cuda.synchronize()
tf = ti = 0.0
for _ in range(iters):
    a, b, c = ev(), ev(), ev()
    a.record()
    plan.forward(x, out=T)
    b.record()
    plan.inverse(T, out=y)
    c.record()
    torch.cuda.synchronize()
    tf += a.elapsed_time(b)
    ti += b.elapsed_time(c)
cnt = plan.counters()
calls = iters + 2
print(f"{os.environ.get('SST_LIB_PATH', 'libsst.so')} {name} N={cfg.N}: fwd {tf/iters:.3f} ms  inv {ti/iters:.3f} ms  "
      f"-> {cfg.N / ((tf + ti) / iters * 1e-3) / 1e6:.1f} MS/s; R23 re-decided {cnt['redecided'] / calls / plan.frames:.4f}"
      f"/frame, changed {cnt['changed'] / calls / plan.frames:.2e}/frame")
