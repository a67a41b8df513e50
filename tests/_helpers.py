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


def flip_stats(l_gpu, l_orc, S_orc, fhat_orc, k1, zoom, Sd_orc=None, nfft=None, alpha=None, gamma=None):
    """Target-index disagreement between the GPU and the oracle (BASELINE north_star), computed
    from oracle quantities only (the oracle never sees GPU data):
      frac      flipped / above-threshold coefficients;
      far_big   largest rounding-boundary distance (coarse bins, oracle's fp64 position) of a flip
                with |S| >= 1e-2 max (reported);
      far       the same over flips of *resolvable* coefficients -- those whose reassignment
                frequency an fp32 STFT fixes to better than 1e-5 fine bins (reading R21):
                delta_r = N_f/(2 pi) eta/2 (1/(alpha |S|) + |S'|/|S|^2),
                eta = 4 u sqrt(log2 N_f) ||z_m||_2 the packed-FFT error of one bin of frame m,
                ||z_m||_2^2 = (2/N_f) sum_k (|S|^2 + alpha^2 |S'|^2), u = 2^-24;
      bad_mask  mask disagreements farther from the threshold than max(1e-5 gamma, eta/2), the
                fp32 STFT's resolution of |S| in the same error model (R21)."""
    above = l_orc != -1
    flips = (l_gpu != l_orc) & above
    n_above = int(above.sum())
    frac = flips.sum() / max(1, n_above)
    amax = np.abs(S_orc).max()
    pos = zoom * (fhat_orc - k1) + 0.5
    with np.errstate(invalid="ignore"):
        dist = np.abs(pos - np.round(pos)) / zoom
    big = flips & (np.abs(S_orc) >= 1e-2 * amax)
    far_big = float(dist[big].max()) if big.any() else 0.0
    out = {"flips": int(flips.sum()), "above": n_above, "frac": float(frac), "far_big": far_big}
    if Sd_orc is not None:
        aS = np.abs(S_orc)
        zn2 = 2.0 / nfft * np.sum(aS ** 2 + alpha ** 2 * np.abs(Sd_orc) ** 2, axis=1, keepdims=True)
        eta = 4.0 * 2.0 ** -24 * np.sqrt(np.log2(nfft)) * np.sqrt(zn2)
        with np.errstate(divide="ignore", invalid="ignore"):
            dr = nfft / (2 * np.pi) * eta / 2 * (1.0 / (alpha * aS) + np.abs(Sd_orc) / aS ** 2)
        res = flips & (zoom * dr < 1e-5)
        out["far"] = float(dist[res].max()) if res.any() else 0.0
        out["unresolvable_flips"] = int((flips & ~res).sum())
        mdiff = (l_gpu == -1) != (l_orc == -1)
        g = max(gamma or 0.0, 1e-30)
        # a mask disagreement is legitimate when |S| lies within what an fp32 STFT resolves of the
        # threshold: eta/2 (the same per-bin error model, R21) or 1e-5 gamma, whichever is larger
        out["bad_mask"] = int((mdiff & (np.abs(aS - g) > np.maximum(1e-5 * g, eta / 2))).sum())
    return out


def signal(cfg_name, start=0, stop=None):
    return generate(cfg_name, start, stop)


__all__ = ["oracle_window", "config_gamma", "make_plan", "rel", "flip_stats", "signal", "get_config"]
