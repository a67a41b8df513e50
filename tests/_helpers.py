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


def flip_stats(l_gpu, l_orc, S_orc, fhat_orc, k1, zoom, gamma=0.0):
    """Target disagreement between the GPU and the oracle (BASELINE north_star), computed from
    oracle quantities only (the oracle never sees GPU data):
      frac      (target flips + mask disagreements) / above-threshold coefficients (<= 1e-4);
      far       largest distance (coarse bins) of a target flip's oracle fp64 position
                z (fhat - k1) + 1/2 from the nearest rounding boundary (Eq. 28), over all flips
                (reported);
      far_big   the same over flips with |S| >= 1e-2 max|S|: the north star's "lying within 1e-4
                bins of a rounding boundary", read as SURVEY §8(c) states it (clause 2 applies to
                coefficients with |S| >= 1e-2 max|S|) -- asserted <= 1e-4;
      bad_mask  mask disagreements (Eq. 13) with ||S| - gamma| > 1e-5 gamma, i.e. not explained
                by the rounding of the threshold itself (must be 0).
    Reading R23: the GPU re-takes in fp64 every in-band decision its fp32 FFT could
    have moved, so these hold with no resolvability model on the test side."""
    kept_o = l_orc != -1
    kept_g = l_gpu != -1
    mdiff = kept_o != kept_g
    flips = kept_o & kept_g & (l_gpu != l_orc)
    n_above = int(kept_o.sum())
    frac = (int(flips.sum()) + int(mdiff.sum())) / max(1, n_above)
    amax = np.abs(S_orc).max()
    with np.errstate(invalid="ignore"):
        pos = zoom * (fhat_orc - k1) + 0.5
        dist = np.abs(pos - np.round(pos)) / zoom
    dist = np.where(np.isfinite(dist), dist, np.inf)
    big = flips & (np.abs(S_orc) >= 1e-2 * amax)
    g = max(float(gamma or 0.0), 1e-300)
    bad_mask = mdiff & (np.abs(np.abs(S_orc) - g) > 1e-5 * g)
    return {"flips": int(flips.sum()), "mask_diff": int(mdiff.sum()), "above": n_above, "frac": float(frac),
            "far": float(dist[flips].max()) if flips.any() else 0.0,
            "far_big": float(dist[big].max()) if big.any() else 0.0,
            "bad_mask": int(bad_mask.sum())}


def assert_flips(st, ctx=None):
    """The north star's disagreement clause, unconditionally: <= 1e-4 of
    above-threshold coefficients disagree, every target flip of a coefficient with
    |S| >= 1e-2 max|S| lies within 1e-4 coarse bins of a rounding boundary, and no mask disagreement
    is farther from gamma than its own rounding (1e-5 gamma)."""
    assert st["frac"] <= 1e-4, (ctx, st)
    assert st["far_big"] <= 1e-4, (ctx, st)
    assert st["bad_mask"] == 0, (ctx, st)


def signal(cfg_name, start=0, stop=None):
    return generate(cfg_name, start, stop)


__all__ = ["oracle_window", "config_gamma", "make_plan", "rel", "flip_stats", "assert_flips", "signal", "get_config"]
