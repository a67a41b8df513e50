"""f3b timing: the filter-bank forward against the fused forward on full records with
SST_SOURCE_TRUNCATE (CUDA events): python tools/time_fb.py [C2 C3 C4]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402

for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    cfg = get_config(name)
    x = torch.from_numpy(generate(cfg)).cuda()
    g, gd = P.gaussian_window(cfg.L, cfg.sigma)
    gamma = 1e-6 * float(np.sum(g)) * float(x.abs().max())
    res = {}
    for mode in ("1", "0"):
        os.environ["SST_FILTERBANK"] = mode
        plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=gamma,
                      flags=P.SST_SOURCE_TRUNCATE)
        T = torch.empty((plan.frames, plan.bins), dtype=torch.complex64, device="cuda")
        for _ in range(2):
            plan.forward(x, out=T)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            plan.forward(x, out=T)
        b.record()
        torch.cuda.synchronize()
        res[mode] = (a.elapsed_time(b) / 5, plan.forward_path, plan.counters())
        if mode == "1":
            T1 = T[::97].clone()
        else:
            T0 = T[::97]
            d = float((T0 - T1).abs().pow(2).sum().sqrt() / T1.abs().pow(2).sum().sqrt())
        plan.close()
        del T
    print(f"{name} truncate forward: filter bank {res['1'][0]:.3f} ms (path {res['1'][1]}, R23 {res['1'][2]}); "
          f"fused {res['0'][0]:.3f} ms; T rel diff {d:.2e}", flush=True)
    del x, T1
    torch.cuda.empty_cache()
