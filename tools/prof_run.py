"""Small driver for ncu captures: forward + inverse on a shortened config record.

    python tools/prof_run.py [--cfg C3] [--n-log2 21] [--iters 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C3")
ap.add_argument("--n-log2", type=int, default=21)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--no-inverse", action="store_true")
args = ap.parse_args()
cfg = get_config(args.cfg)
N = min(cfg.N, 1 << args.n_log2)
cfg = cfg.with_(N=N)
x = torch.from_numpy(generate(cfg, 0, N)).cuda()
g, gd = P.gaussian_window(cfg.L, cfg.sigma)
gamma = 1e-6 * float(np.sum(g)) * float(x.abs().max())
plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=gamma)
T = torch.empty((plan.frames, plan.bins), dtype=torch.complex64, device="cuda")
y = torch.empty(N, dtype=torch.float32, device="cuda")
for _ in range(args.iters):
    plan.forward(x, out=T)
    if not args.no_inverse:
        plan.inverse(T, out=y)
torch.cuda.synchronize()
print("ok", cfg.name, N, plan.frames, plan.bins)
