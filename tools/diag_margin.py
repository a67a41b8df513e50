"""R23 margin calibration on the GPU: the fp32 error of the GPU's own reassignment frequency
(sst_stft, re-decision off) against the fp64 oracle, in units of the R21 error model the kernel
uses, for sampled frame windows of C1-C5.  Reports the error/model ratio distribution and how
many in-band kept bins a margin of M x model would flag, per frame.
    python tools/diag_margin.py [frames_per_window]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402
from tests._helpers import config_gamma  # noqa: E402

nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
for name in ["C1", "C2", "C3", "C4", "C5"]:
    cfg = get_config(name)
    f0 = 0 if name == "C1" else cfg.frames // 3
    fe = min(cfg.frames, f0 + nfr)
    lo = max(0, f0 * cfg.hop - cfg.L)
    hi = min(cfg.N, fe * cfg.hop + cfg.L)
    x = generate(cfg, lo, hi)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    xfull = generate(cfg) if name == "C1" else None
    gamma = config_gamma(cfg, xfull) if name == "C1" else 1e-6 * float(np.sum(g)) * float(np.abs(x).max())
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=gamma)
    xd = torch.from_numpy(x).cuda()
    S, Sd = plan.stft(xd, f0, fe, x_off=lo)
    S = S.cpu().numpy().astype(np.complex128)
    Sd = Sd.cpu().numpy().astype(np.complex128)
    # oracle on a local record: local frame m = global frame f0 + m when the local x starts at f0*H - ...
    xl = np.zeros(cfg.N, np.float64) if False else None
    fr = np.arange(f0, fe)
    # oracle frames need global sample indexing: build a view record
    xg = np.zeros(hi, np.float64)
    xg[lo:hi] = x
    So = O.stft(xg, g, c, cfg.hop, cfg.nfft, frames=fr)
    Sdo = O.stft(xg, gd, c, cfg.hop, cfg.nfft, frames=fr)
    alpha = plan.layout["alpha"]
    z, N = cfg.zoom, cfg.nfft
    k = np.arange(N // 2 + 1)
    r64 = -np.imag(Sdo / So) * N / (2 * np.pi)
    r32 = -np.imag(Sd / S) * N / (2 * np.pi)
    err = np.abs(r32 - r64) * z
    # packed-input norm of each frame (what the kernel accumulates in its gather)
    idx = fr[:, None] * cfg.hop - c + np.arange(cfg.L)[None, :]
    u = np.where((idx >= 0) & (idx < hi), xg[np.clip(idx, 0, hi - 1)], 0.0)
    nrm = np.sqrt(np.sum(u ** 2 * (g ** 2 + alpha ** 2 * gd ** 2)[None, :], axis=1, keepdims=True))
    mag4 = 4 * np.abs(S) ** 2
    rs = 1 / np.sqrt(mag4)
    UV = np.abs(2 * alpha * Sd.real) + np.abs(2 * alpha * Sd.imag)
    uv2 = np.abs(2 * alpha * Sd)
    zr_scale = z * N / (2 * np.pi * alpha)
    eta = 4 * 2.0 ** -24 * np.sqrt(np.log2(N)) * nrm
    model = zr_scale * eta * (rs + UV * rs ** 2)
    model2 = zr_scale * eta * (rs + uv2 * rs ** 2)
    ratio = err / model
    mask = np.abs(So) > gamma
    pos = z * (np.abs(k[None, :] + r64) - cfg.k1) + 0.5
    inb = mask & (pos > -1) & (pos < plan.bins + 1)
    fpos = pos - np.floor(pos)
    d = np.minimum(fpos, 1 - fpos)
    amax = np.abs(So).max()
    big = np.abs(So) >= 1e-2 * amax
    out = [f"{name}: frames {len(fr)} ratio max {np.nanmax(ratio[inb]):.3f} p1e-6 {np.nanquantile(ratio[inb], 1 - 1e-6):.3f} "
           f"(exact |UV|: {np.nanmax((err / model2)[inb]):.3f})"]
    for M in (1, 2, 4, 8):
        fl = inb & (d < M * model)
        flb = fl & big
        out.append(f"M={M}: {fl.sum() / len(fr):.3f}/frame (|S|>=1e-2max: {flb.sum() / len(fr):.3f})")
    print("  ".join(out), flush=True)
    plan.close()
