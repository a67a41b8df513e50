"""Deterministic, block-addressable synthetic signals for configs C1-C5.

Any sample range [start, stop) can be generated on its own and is bit-identical to the
same range of the whole record, so every rank of a sharded run (and the oracle) sees the
same samples without communication:

* tonal parts use closed-form phases (integral of the IF), never a cumulative sum;
* random parts are drawn per block of ``BLOCK`` samples from
  ``numpy.random.Generator(PCG64(SeedSequence([seed, stream, block])))``;
* parameters (phases, speed profiles, FM laws) come from stream 0.

Noise level: SNR is relative to the *nominal* clean tonal power sum(a^2)/2 (a record-
independent constant, so it does not depend on which range is generated).
"""

from __future__ import annotations

import numpy as np

from .configs import Config, get_config

BLOCK = 1 << 16
_STREAM_PARAMS, _STREAM_NOISE, _STREAM_IMPULSE = 0, 1, 2


def _rng(seed: int, stream: int, block: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, block])))


# --------------------------------------------------------------------------------------- noise
def _white_block(seed: int, b: int) -> np.ndarray:
    return _rng(seed, _STREAM_NOISE, b).standard_normal(BLOCK)


def _pink_block(seed: int, b: int) -> np.ndarray:
    """White noise of one block shaped by f^(-1/2) in an rfft (DC zeroed), unit variance."""
    w = _white_block(seed, b)
    W = np.fft.rfft(w)
    f = np.arange(W.shape[0], dtype=np.float64)
    shape = np.zeros_like(f)
    shape[1:] = f[1:] ** -0.5
    p = np.fft.irfft(W * shape, n=BLOCK)
    return p / p.std()


def _noise(seed: int, start: int, stop: int, kind: str) -> np.ndarray:
    out = np.empty(stop - start, dtype=np.float64)
    b0, b1 = start // BLOCK, (stop - 1) // BLOCK
    for b in range(b0, b1 + 1):
        blk = _white_block(seed, b) if kind == "white" else _pink_block(seed, b)
        lo, hi = max(start, b * BLOCK), min(stop, (b + 1) * BLOCK)
        out[lo - start:hi - start] = blk[lo - b * BLOCK:hi - b * BLOCK]
    return out


def _impulses(seed: int, fs: float, start: int, stop: int, rate: float = 20.0,
              amp: float = 0.5, f_res: float = 1200.0, tau: float = 5e-3, trunc: float = 0.05):
    """Resonance driven by Poisson(rate) impulses: amp e^{-t/tau} sin(2 pi f_res t), 0 <= t < trunc.
    Arrivals are drawn per block; blocks whose impulses can reach [start, stop) are included."""
    out = np.zeros(stop - start, dtype=np.float64)
    reach = int(np.ceil(trunc * fs))
    b0, b1 = max(0, (start - reach) // BLOCK), (stop - 1) // BLOCK
    for b in range(b0, b1 + 1):
        rng = _rng(seed, _STREAM_IMPULSE, b)
        n_imp = rng.poisson(rate * BLOCK / fs)
        t0 = (b * BLOCK + rng.uniform(0.0, BLOCK, size=n_imp)) / fs   # arrival times (s)
        for ti in np.sort(t0):
            s0 = int(np.ceil(ti * fs))
            s1 = s0 + reach
            lo, hi = max(s0, start), min(s1, stop)
            if lo >= hi:
                continue
            t = np.arange(lo, hi, dtype=np.float64) / fs - ti
            out[lo - start:hi - start] += amp * np.exp(-t / tau) * np.sin(2 * np.pi * f_res * t)
    return out


# --------------------------------------------------------------------------------------- tonal
def _c1_clean(t):
    tone = np.cos(2 * np.pi * 100.0 * t)
    chirp = 0.5 * np.cos(2 * np.pi * (200.0 * t + 25.0 * t * t))      # 200 -> 400 Hz over 4 s
    return tone, chirp


_C2_AMPS = (1.0, 0.6, 0.4, 0.2)
_C3_ORDERS = (1, 2, 3, 5, 8)
_C3_AMPS = (1.0, 0.5, 0.3, 0.2, 0.1)


def _c2_clean(seed, t):
    psi = _rng(seed, _STREAM_PARAMS).uniform(0.0, 2 * np.pi, size=4)
    theta = 2 * np.pi * 150.0 * t - 20.0 * np.cos(np.pi * t)          # f0 = 150 + 10 sin(pi t)
    am = 1.0 + 0.05 * np.sin(2 * np.pi * 2.0 * t)
    x = np.zeros_like(t)
    for h, (a, p) in enumerate(zip(_C2_AMPS, psi), start=1):
        x += a * np.cos(h * theta + p)
    return x * am


def _runup_theta(seed, cfg, t):
    """Shaft angle for C3 (one linear run-up 50->250 Hz over the record) and C4 (16 seeded
    run-ups f_a~U[45,55] -> f_b~U[240,260], phase continuous across joins)."""
    if cfg.name == "C4":
        nseg = 16
        rng = _rng(seed, _STREAM_PARAMS, 1)
        fa = rng.uniform(45.0, 55.0, size=nseg)
        fb = rng.uniform(240.0, 260.0, size=nseg)
        Tseg = cfg.N / nseg / cfg.fs
        seg = np.minimum((t // Tseg).astype(np.int64), nseg - 1)
        start_phase = np.concatenate([[0.0], np.cumsum(2 * np.pi * Tseg * (fa + fb) / 2.0)])
        tl = t - seg * Tseg
        return start_phase[seg] + 2 * np.pi * (fa[seg] * tl + (fb[seg] - fa[seg]) * tl * tl / (2 * Tseg))
    Trec = cfg.N / cfg.fs
    return 2 * np.pi * (50.0 * t + 100.0 * t * t / Trec)


def _runup_clean(seed, cfg, t):
    psi = _rng(seed, _STREAM_PARAMS).uniform(0.0, 2 * np.pi, size=len(_C3_ORDERS))
    theta = _runup_theta(seed, cfg, t)
    x = np.zeros_like(t)
    for o, a, p in zip(_C3_ORDERS, _C3_AMPS, psi):
        x += a * np.cos(o * theta + p)
    return x


def c5_laws(seed: int, fs: float = 25600.0, sigma: float = 64.0):
    """8 crossing-free FM laws IF_k = c_k + a_k sin(2 pi b_k t): redraw until every pair has
    |c_i - c_j| >= a_i + a_j + 8 sigma_f (sigma_f = fs / (2 pi sigma) Hz)."""
    rng = _rng(seed, _STREAM_PARAMS, 1)
    sig_f = fs / (2 * np.pi * sigma)
    while True:
        c = rng.uniform(500.0, 10000.0, size=8)
        a = rng.uniform(0.0, 50.0, size=8)
        b = rng.uniform(0.1, 2.0, size=8)
        ok = all(abs(c[i] - c[j]) >= a[i] + a[j] + 8 * sig_f for i in range(8) for j in range(i + 1, 8))
        if ok:
            psi = rng.uniform(0.0, 2 * np.pi, size=8)
            return c, a, b, psi


def _c5_clean(seed, t):
    c, a, b, psi = c5_laws(seed)
    x = np.zeros_like(t)
    for k in range(8):
        x += np.cos(2 * np.pi * (c[k] * t - a[k] * np.cos(2 * np.pi * b[k] * t) / (2 * np.pi * b[k])) + psi[k])
    return x


_NOMINAL_POWER = {
    "C2": sum(a * a for a in _C2_AMPS) / 2.0,
    "C3": sum(a * a for a in _C3_AMPS) / 2.0,
    "C4": sum(a * a for a in _C3_AMPS) / 2.0,
    "C5": 8 * 0.5,
}
_SNR_DB = {"C2": 10.0, "C3": 5.0, "C4": 5.0, "C5": 20.0}


def _cfg(name_or_cfg):
    return name_or_cfg if isinstance(name_or_cfg, Config) else get_config(name_or_cfg)


def clean_components(name, start: int = 0, stop: int | None = None):
    """Noise-free parts of a config's signal on [start, stop), fp64 (dict name -> array).
    ``name`` is a config name or a Config (e.g. C3 with N scaled for weak scaling)."""
    cfg = _cfg(name)
    name = cfg.name
    stop = cfg.N if stop is None else stop
    t = np.arange(start, stop, dtype=np.float64) / cfg.fs
    if name == "C1":
        tone, chirp = _c1_clean(t)
        return {"tone": tone, "chirp": chirp}
    if name == "C2":
        return {"harmonics": _c2_clean(cfg.seed, t)}
    if name in ("C3", "C4"):
        return {"orders": _runup_clean(cfg.seed, cfg, t),
                "resonance": _impulses(cfg.seed, cfg.fs, start, stop)}
    if name == "C5":
        return {"fm": _c5_clean(cfg.seed, t)}
    raise KeyError(name)


def generate(name, start: int = 0, stop: int | None = None, dtype=np.float32) -> np.ndarray:
    """Samples [start, stop) of config ``name``'s record (default: whole record) as ``dtype``.
    ``name`` is a config name or a Config.  fp32 is the GPU input; the oracle takes the same
    fp32 samples upcast to fp64."""
    cfg = _cfg(name)
    name = cfg.name
    stop = cfg.N if stop is None else stop
    if not (0 <= start <= stop <= cfg.N):
        raise ValueError("range outside record")
    if start == stop:
        return np.zeros(0, dtype=dtype)
    parts = clean_components(cfg, start, stop)
    x = sum(parts.values())
    if name == "C1":
        x = x + 0.1 * _noise(cfg.seed, start, stop, "white")
    else:
        sd = np.sqrt(_NOMINAL_POWER[name] / 10.0 ** (_SNR_DB[name] / 10.0))
        kind = "pink" if name in ("C3", "C4") else "white"
        x = x + sd * _noise(cfg.seed, start, stop, kind)
    return np.ascontiguousarray(x, dtype=dtype)


# --------------------------------------------------------------------------------------- paper
def eq30_signal(N: int = 8192, fs: float = 1024.0):
    """The three AM-FM components of Eq. (30), fp64; returns (x1, x2, x3)."""
    t = np.arange(N, dtype=np.float64) / fs
    x1 = (1 - 0.1 * np.cos(0.25 * np.pi * t)) * np.cos(100 * np.pi * t)
    x2 = np.where(t < 4,
                  np.cos(500 * np.pi * t - 25 * np.pi * t ** 2),
                  np.cos(500 * np.pi * t - 50 * np.pi * t ** 2 + 25.0 / 6.0 * np.pi * t ** 3 + 4.0 / 3.0 * np.pi))
    x3 = (1 - 0.2 * np.cos(0.125 * np.pi * t)) * np.cos(740 * np.pi * t + 400.0 / 3.0 * np.sin(0.75 * np.pi * t)
                                                       - 200 * np.sin(0.5 * np.pi * t))
    return x1, x2, x3


def eq30_true_ifs(N: int = 8192, fs: float = 1024.0):
    """True IFs of Eq. (31), Hz."""
    t = np.arange(N, dtype=np.float64) / fs
    f1 = np.full_like(t, 50.0)
    f2 = np.where(t < 4, 250 - 25 * t, 250 - 50 * t + 6.25 * t ** 2)
    f3 = 370 + 50 * np.cos(0.75 * np.pi * t) - 50 * np.cos(0.5 * np.pi * t)
    return f1, f2, f3


def eq30_noisy(snr_db: float, seed: int, N: int = 8192, fs: float = 1024.0):
    """Eq. (30) sum plus white Gaussian noise at `snr_db` relative to its mean power (the §3.3
    reconstruction experiments); returns (x fp32, (x1, x2, x3) fp64)."""
    x1, x2, x3 = eq30_signal(N, fs)
    x = x1 + x2 + x3
    p = np.mean(x ** 2)
    w = np.random.default_rng(seed).standard_normal(N) * np.sqrt(p / 10 ** (snr_db / 10))
    return (x + w).astype(np.float32), (x1, x2, x3)


def s52_milling(seed: int = 52, N: int = 573440, fs: float = 10240.0):
    """Stand-in for the §5.2 milling vibration record (fs = 10240 Hz, 56 s,
    N = 573440, spindle 9600 r/min, chatter near 1200-1400 Hz from about 28 s).  Synthetic and
    invented -- not the dataset: harmonics 1-6 of a 160 Hz spindle whose speed fluctuates weakly
    and quickly (the 4th harmonic stays inside 630-640 Hz, the paper's Fig. 16(e) band), a chatter
    component whose IF drifts 1310 -> 1345 Hz and whose amplitude rises smoothly around 28 s, and
    white noise at 10 dB below the clean power.  Returns fp32 x."""
    rng = np.random.default_rng(seed)
    t = np.arange(N, dtype=np.float64) / fs
    a1, a2 = 0.08 * rng.uniform(0.8, 1.2), 0.05 * rng.uniform(0.8, 1.2)
    f1, f2 = rng.uniform(2.0, 3.0), rng.uniform(6.0, 8.0)
    # spindle IF 158.9 + a1 sin + a2 sin (Hz); phase = closed-form integral
    th = 2 * np.pi * (158.9 * t - a1 / (2 * np.pi * f1) * np.cos(2 * np.pi * f1 * t)
                      - a2 / (2 * np.pi * f2) * np.cos(2 * np.pi * f2 * t))
    x = np.zeros(N)
    for h, amp in zip(range(1, 7), (1.0, 0.5, 0.3, 0.4, 0.15, 0.1)):
        x += amp * np.cos(h * th + rng.uniform(0, 2 * np.pi))
    T_rec = N / fs
    ch_phase = 2 * np.pi * (1310.0 * t + 35.0 * t ** 2 / (2 * T_rec))
    ch_amp = 0.6 / (1.0 + np.exp(-(t - 28.0) / 1.5))
    x += ch_amp * np.cos(ch_phase + rng.uniform(0, 2 * np.pi))
    p = np.mean(x ** 2)
    x += rng.standard_normal(N) * np.sqrt(p / 10.0)
    return x.astype(np.float32)
