"""Shared helpers for the GPU parity tests (test-side only)."""

from __future__ import annotations

import numpy as np

import oracle as O
from gen import generate, get_config


def oracle_window(cfg):
    return O.gaussian_window(cfg.L, cfg.sigma)


def config_gamma(cfg, x32: np.ndarray) -> float:
    """Threshold of reading R6: C1 -> 1e-6 * max|S| (oracle fp64, whole record);
    C2-C5 -> 1e-6 * sum(g) * max|x| (a bound on max|S| computable from x alone)."""
    g, gd, c = oracle_window(cfg)
    if cfg.name == "C1":
        S = O.stft(x32.astype(np.float64), g, c, cfg.hop, cfg.nfft)
        return 1e-6 * float(np.abs(S).max())
    return 1e-6 * float(np.sum(g)) * float(np.abs(x32).max())


def make_plan(P, cfg, gamma, flags=0, device=0):
    return P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom,
                  gamma=gamma, flags=flags, device=device)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def flip_stats(l_gpu, l_orc, S_orc, fhat_orc, k1, zoom):
    """Target-index disagreement between GPU and oracle (BASELINE north_star):
    fraction of above-threshold coefficients whose target differs, and the largest distance
    (coarse bins) of a flipped coefficient with |S| >= 1e-2 max from a rounding boundary."""
    above = l_orc != -1
    flips = (l_gpu != l_orc) & above
    n_above = int(above.sum())
    frac = flips.sum() / max(1, n_above)
    amax = np.abs(S_orc).max()
    big = flips & (np.abs(S_orc) >= 1e-2 * amax)
    if big.any():
        pos = zoom * (fhat_orc[big] - k1) + 0.5
        dist = np.abs(pos - np.round(pos)) / zoom
        far = float(dist.max())
    else:
        far = 0.0
    mask_flips = int(((l_gpu == -1) != (l_orc == -1)).sum())
    return {"flips": int(flips.sum()), "above": n_above, "frac": float(frac), "far_big": far,
            "mask_flips": mask_flips}


def decision_stats(l_gpu, S_gpu, Sd_gpu, gamma, nfft, k1, B, zoom):
    """Target decisions re-taken by the oracle in fp64 from the kernel's own fp32 spectra
    (``sst_stft`` output): the kernel's integer decision may differ from the fp64 one only where
    the fp64 position lies within 1e-4 coarse bins of a rounding boundary (reading R21:
    where floating point decides an integer, both sides decide in the same precision -- the
    paper's fp64 -- from the same inputs).  Mask decisions may differ only where |S| is within
    1e-6 relative of gamma.  Returns the largest boundary distance of a disagreement (bins) and
    the count of unexplained mask disagreements."""
    S = np.asarray(S_gpu, dtype=np.complex128)
    Sd = np.asarray(Sd_gpu, dtype=np.complex128)
    mask, r, fhat = O.if_estimate(S, Sd, nfft, gamma)
    l_ref = O.targets(fhat, mask, k1, B, zoom)
    diff = l_gpu != l_ref
    mdiff = diff & ((l_gpu == -1) != (l_ref == -1))
    bad_mask = int((mdiff & (np.abs(np.abs(S) - gamma) > 1e-6 * max(gamma, 1e-30))).sum())
    tdiff = diff & ~mdiff
    if tdiff.any():
        pos = zoom * (fhat[tdiff] - k1) + 0.5
        far = float((np.abs(pos - np.round(pos)) / zoom).max())
    else:
        far = 0.0
    return {"disagree": int(diff.sum()), "far": far, "bad_mask": bad_mask}


def signal(cfg_name, start=0, stop=None):
    return generate(cfg_name, start, stop)


__all__ = ["oracle_window", "config_gamma", "make_plan", "rel", "flip_stats", "decision_stats", "signal", "get_config"]
