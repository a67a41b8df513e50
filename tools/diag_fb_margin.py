"""R23 margin calibration of the filter-bank forward (f3b): the fp32 error of r from the filter
bank's S, S' (sst_stft_band, truncate plans) against the fp64 oracle, in units of the plan's error
model eta_S = 8 u sqrt(log2(Ns P)) ||x_b|| ||g|| / sqrt(Ns) (see sst_api.cu setup_filterbank).
    python tools/diag_fb_margin.py [frames]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SST_FILTERBANK", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402

nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
for name in ["C2", "C3", "C4"]:
    cfg = get_config(name)
    f0 = cfg.frames // 3
    fe = f0 + nfr
    L, H, Nf, c = cfg.L, cfg.hop, cfg.nfft, cfg.L // 2
    ns = 1
    while ns < 4 * L:
        ns <<= 1
    ns = max(ns, Nf)
    Pn = ns // H
    Fb = (ns - L) // H + 1
    b0, b1 = f0 // Fb, (fe - 1) // Fb
    lo = max(0, b0 * Fb * H - c)
    hi = min(cfg.N, (b1 + 1) * Fb * H - c + ns)
    x = generate(cfg, lo, hi)
    g, gd, cc = O.gaussian_window(L, cfg.sigma)
    plan = P.Plan(cfg.N, cfg.fs, L, cfg.sigma, H, Nf, cfg.f1, cfg.f2, cfg.zoom, gamma=1e-6,
                  flags=P.SST_SOURCE_TRUNCATE)
    assert plan.forward_path == P.SST_PATH_FILTERBANK, name
    xd = torch.from_numpy(x).cuda()
    S, Sd = plan.stft_band(xd, f0, fe, x_off=lo)
    S = S.cpu().numpy().astype(np.complex128)
    Sd = Sd.cpu().numpy().astype(np.complex128)
    xg = np.zeros(hi)
    xg[lo:hi] = x
    fr = np.arange(f0, fe)
    k1, k2 = cfg.k1, cfg.k2
    So = O.stft(xg, g, c, H, Nf, frames=fr)[:, k1:k2]
    Sdo = O.stft(xg, gd, c, H, Nf, frames=fr)[:, k1:k2]
    alpha = plan.layout["alpha"]
    r64 = -np.imag(Sdo / So) * Nf / (2 * np.pi)
    r32 = -np.imag(Sd / S) * Nf / (2 * np.pi)
    err = np.abs(r32 - r64) * cfg.zoom
    # eta per frame: ||x_b|| of its block
    blocks = fr // Fb
    nb = np.zeros(len(fr))
    for b in np.unique(blocks):
        s0 = b * Fb * H - c
        seg = xg[max(0, s0):max(0, s0 + ns)]
        nb[blocks == b] = np.sqrt(np.sum(seg.astype(np.float64) ** 2))
    gn = np.sqrt(np.sum(g ** 2)) * max(1.0, alpha * np.sqrt(np.sum(gd ** 2) / np.sum(g ** 2)))
    etaS = 8 * 2.0 ** -24 * np.sqrt(np.log2(ns * Pn)) * nb[:, None] * gn / np.sqrt(ns)
    zr_scale = cfg.zoom * Nf / (2 * np.pi * alpha)
    aS = np.abs(S)
    UV = np.abs(2 * alpha * Sd.real) + np.abs(2 * alpha * Sd.imag)
    model = zr_scale * etaS * (1 / aS + UV / (2 * aS ** 2))
    ratio = err / model
    eS = np.abs(S - So) / etaS
    print(f"{name}: Ns {ns} P {Pn} Fb {Fb}: r ratio max {ratio.max():.3f} p1e-5 {np.quantile(ratio, 1 - 1e-5):.3f}; "
          f"|dS|/eta_S max {eS.max():.3f}; S rel {np.linalg.norm(S - So) / np.linalg.norm(So):.2e}", flush=True)
    plan.close()
