"""Plain fp64 numpy oracle of the downsampled STFT-based SST (He & Cao, arXiv 2003.07065).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Imported by tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs only.

Every function follows one passage of PAPER.md (cited as ``P:Lnnn``, with the
section / equation).  Where the paper is silent or garbled the function applies
the DESIGN.md reading ``Rnn`` it names.  No blocking, fusion or reordering of
the arithmetic beyond what the equation states: frames are processed in
independent chunks only to bound memory (frames are independent, Eq. 7-9).

Units: frequencies are in *coarse bins* of width df = fs/N_f unless a name ends
in ``_hz``; sigma and all window quantities are in samples (R1).
"""

from __future__ import annotations

import numpy as np

_CHUNK_ELEMS = 1 << 22  # memory bound for one chunk of frames (complex128 elements)


# --------------------------------------------------------------------------------------
# Window model -- P:L55 (§2.1, Gaussian window), P:L110 (§2.2, g'), reading R1/R3.
# --------------------------------------------------------------------------------------
def gaussian_window(L: int, sigma: float, center: int | None = None):
    """Unit-energy Gaussian g and its analytic derivative g'.

    g[j]  = (pi sigma^2)^(-1/4) exp(-(j-c)^2 / (2 sigma^2))      (sigma in samples, R1)
    g'[j] = -(pi sigma^2)^(-1/4) exp(-(j-c)^2/(2 sigma^2)) (j-c)/sigma^2
    c = (L-1)/2 for odd L (M=(L-1)/2); c = L/2 for even L (R3).  Both are L//2.
    Returns (g, gd, c).
    """
    if L < 1 or not (sigma > 0):
        raise ValueError("L >= 1 and sigma > 0 required")
    c = L // 2 if center is None or center < 0 else int(center)
    t = np.arange(L, dtype=np.float64) - c
    g = (np.pi * sigma * sigma) ** -0.25 * np.exp(-(t * t) / (2.0 * sigma * sigma))
    gd = -(np.pi * sigma * sigma) ** -0.25 * np.exp(-(t * t) / (2.0 * sigma * sigma)) * t / (sigma * sigma)
    return g, gd, c


def frame_count(N: int, hop: int) -> int:
    """Frames m = 0..floor((N-1)/H_t), frame m centred on sample m*H_t (R4)."""
    return (N - 1) // hop + 1


def _frame_rows(x, hop, c, L, frames):
    """u[m, n] = x[n + m H_t - M] for n = 0..L-1, zero outside [0, N)  (Eq. 8 summand, R4)."""
    N = x.shape[0]
    idx = frames[:, None] * hop - c + np.arange(L)[None, :]
    ok = (idx >= 0) & (idx < N)
    u = np.zeros(idx.shape, dtype=np.float64)
    u[ok] = x[idx[ok]]
    return u


def _chunks(frames, per_frame):
    step = max(1, _CHUNK_ELEMS // max(1, per_frame))
    for i in range(0, len(frames), step):
        yield frames[i:i + step]


# --------------------------------------------------------------------------------------
# Downsampled STFT -- Eq. 7-9, P:L81-93 (§2.1).
# --------------------------------------------------------------------------------------
def stft(x, w, c: int, hop: int, nfft: int, frames=None, full: bool = False):
    """S_x^w[m, k] by Eq. (9): the N_f-point DFT of the buffer
    b[n] = x[n + m H_t - M] w[n - M] (n = 0..L-1, zero-padded to N_f), times the
    phase e^{+i 2 pi k M / N_f}.  Returns k = 0..N_f/2 (R7) unless ``full``.

    ``w`` is the tap array w[0..L-1] with centre c (so w[n] is the paper's g[n-M]).
    The DFT is numpy's FFT, "setting N_f to the power of 2 and using FFT".
    """
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    L = w.shape[0]
    if L > nfft:
        raise ValueError("Eq. 9 needs L <= N_f (P:L89)")
    F = frame_count(x.shape[0], hop)
    frames = np.arange(F) if frames is None else np.asarray(frames, dtype=np.int64)
    K = nfft if full else nfft // 2 + 1
    k = np.arange(K)
    phase = np.exp(2j * np.pi * k * c / nfft)                      # e^{i 2 pi k M / N_f}
    out = np.empty((len(frames), K), dtype=np.complex128)
    pos = 0
    for fr in _chunks(frames, nfft):
        buf = np.zeros((len(fr), nfft), dtype=np.float64)
        buf[:, :L] = _frame_rows(x, hop, c, L, fr) * w[None, :]   # x[n+mH-M] g[n-M]
        spec = np.fft.fft(buf, axis=1)[:, :K]                       # sum_n ... e^{-i2pi kn/N_f}
        out[pos:pos + len(fr)] = spec * phase[None, :]
        pos += len(fr)
    return out


def stft_direct(x, w, c: int, hop: int, nfft: int, frames, bins):
    """Brute-force Eq. (8): S[m,k] = sum_{n=0}^{L-1} x[n+mH-M] g[n-M] e^{-i2pi k(n-M)/N_f}.
    Python loops; tiny inputs only (pin P1)."""
    x = np.asarray(x, dtype=np.float64)
    N, L = x.shape[0], len(w)
    out = np.zeros((len(frames), len(bins)), dtype=np.complex128)
    for a, m in enumerate(frames):
        for b, k in enumerate(bins):
            acc = 0j
            for n in range(L):
                s = n + m * hop - c
                if 0 <= s < N:
                    acc += x[s] * w[n] * np.exp(-2j * np.pi * k * (n - c) / nfft)
            out[a, b] = acc
    return out


def frame_diagonal(g, c: int, hop: int, N: int, n0: int = 0, n1: int | None = None):
    """d[n] = sum_m g[n - m H_t + M]^2 over the frames m = 0..F-1 that cover n
    (the normaliser of Eq. 11 / Eq. 26, "sum_m |g[n - mH]|^2 = 1"; R2)."""
    n1 = N if n1 is None else n1
    g = np.asarray(g, dtype=np.float64)
    L = g.shape[0]
    F = frame_count(N, hop)
    n = np.arange(n0, n1)
    d = np.zeros(n.shape, dtype=np.float64)
    m_lo = max(0, (n0 + c - L) // hop)
    m_hi = min(F - 1, (n1 - 1 + c) // hop + 1)
    for m in range(m_lo, m_hi + 1):
        j = n - m * hop + c
        ok = (j >= 0) & (j < L)
        d[ok] += g[j[ok]] ** 2
    return d


def stft_inverse(S_full, g, c: int, hop: int, nfft: int, N: int):
    """Downsampled STFT synthesis, Eq. (10)-(11): undo the phase
    e^{-i2pi kM/N_f}, N_f-point inverse DFT, keep n = 0..L-1, multiply by g[n],
    overlap-add at n + mH - M, divide by the frame diagonal d[n] (R2).
    ``S_full`` is the two-sided [F, N_f] STFT (all frames)."""
    g = np.asarray(g, dtype=np.float64)
    L = g.shape[0]
    F = S_full.shape[0]
    k = np.arange(nfft)
    unphase = np.exp(-2j * np.pi * k * c / nfft)
    y = np.zeros(N, dtype=np.float64)
    for fr in _chunks(np.arange(F), nfft):
        s_t = np.fft.ifft(S_full[fr] * unphase[None, :], axis=1)[:, :L]   # s~[m, n]
        contrib = np.real(s_t) * g[None, :]
        idx = fr[:, None] * hop - c + np.arange(L)[None, :]
        ok = (idx >= 0) & (idx < N)
        y += np.bincount(idx[ok], weights=contrib[ok], minlength=N)
    d = frame_diagonal(g, c, hop, N)
    return y / d


# --------------------------------------------------------------------------------------
# IF estimate -- Eq. 12-13, RF Eq. 36.
# --------------------------------------------------------------------------------------
def if_estimate(S, Sd, nfft: int, gamma: float):
    """Discrete IF estimator, Eq. (13):
        omega_hat[m,k] = | xi[k] - Im{S^{g'}/S^g} |   where |S^g| > gamma  (strict, R6)
    with xi[k] = k * 2 pi fs / N_f (Eq. 12).  Returned in coarse bins
    (omega * N_f / (2 pi fs) with Im(.) in rad/sample, R1), together with the
    reassignment frequency r = -Im{S^{g'}/S^g} N_f/(2 pi) of Eq. (36).
    Returns (mask, r, fhat).  Entries outside the mask are NaN."""
    S = np.asarray(S)
    k = np.arange(S.shape[-1], dtype=np.float64)
    mask = np.abs(S) > gamma
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        r = -np.imag(Sd / S) * nfft / (2.0 * np.pi)
        fhat = np.abs(k[None, :] + r)
    r = np.where(mask, r, np.nan)
    fhat = np.where(mask, fhat, np.nan)
    return mask, r, fhat


# --------------------------------------------------------------------------------------
# Selective reassignment + frequency subdivision -- Eq. 27-29.
# --------------------------------------------------------------------------------------
def band_grid(fs: float, nfft: int, f1: float, f2: float, zoom: int):
    """Band of interest snapped to the coarse grid (R9): k1 = round(f1/df), k2 = round(f2/df),
    N_r = k2 - k1, output grid xi*[l] = 2pi[f1 + l (f2-f1)/(z N_r)] (Eq. 29),
    B = z N_r bins (half-open, R10), spacing df* = df/z."""
    df = fs / nfft
    k1f, k2f = f1 / df, f2 / df
    k1, k2 = int(round(k1f)), int(round(k2f))
    if abs(k1f - k1) > 1e-9 or abs(k2f - k2) > 1e-9:
        raise ValueError("band edges must lie on the coarse grid fs/N_f (R9)")
    if not (0 <= k1 < k2 <= nfft // 2) or zoom < 1:
        raise ValueError("need 0 <= f1 < f2 <= fs/2 and z >= 1")
    return {"k1": k1, "k2": k2, "Nr": k2 - k1, "B": zoom * (k2 - k1), "zoom": zoom,
            "df_hz": df, "dfz_hz": df / zoom, "f0_hz": k1 * df}


def targets(fhat, mask, k1: int, B: int, zoom: int):
    """Target bin of Eq. (28): coefficient (m,k) goes to the l with
    |omega_hat - xi*[l]| <= dxi*/2, i.e. l = floor(z (fhat - k1) + 1/2) (ties go up, R10);
    kept iff 0 <= l < B (half-open band, out-of-band dropped, R10).
    Returns int64 l with -1 = masked (|S| <= gamma), -2 = out of band / non-finite (R17)."""
    with np.errstate(invalid="ignore", over="ignore"):
        pos = zoom * (fhat - k1) + 0.5
        ok = mask & np.isfinite(pos) & (pos >= 0.0) & (pos < B)
        l = np.full(fhat.shape, -2, dtype=np.int64)
        l[ok] = np.floor(pos[ok]).astype(np.int64)
    l[~mask] = -1
    return l


def targets_bruteforce(fhat, mask, f1_bins: float, f2_bins: float, Nr: int, zoom: int):
    """Eq. (28)/(29) membership written out: for each masked coefficient test every
    l in [0, z N_r) for |omega_hat - xi*[l]| <= dxi*/2 with xi*[l] = f1 + l (f2-f1)/(z N_r)
    (all in bins).  Where two l qualify (exact tie) take the upper one (R10).  Loops; tiny only."""
    B = zoom * Nr
    half = 0.5 * (f2_bins - f1_bins) / (zoom * Nr)
    out = np.full(fhat.shape, -2, dtype=np.int64)
    for idx in np.ndindex(fhat.shape):
        if not mask[idx]:
            out[idx] = -1
            continue
        f = fhat[idx]
        if not np.isfinite(f):
            continue
        for l in range(B):
            xi = f1_bins + l * (f2_bins - f1_bins) / (zoom * Nr)
            if abs(f - xi) <= half:
                out[idx] = l        # keeps the last (upper) qualifying bin
    return out


def squeeze(S, l, B: int):
    """T[m, l] = sum over kept k of S^g[m, k]  (Eq. 14 / 27 / 28; reading R11: S[m,k], the
    complex coefficient is moved, not its magnitude).  Sums in ascending k per frame."""
    F = S.shape[0]
    keep = l >= 0
    rows = np.broadcast_to(np.arange(F)[:, None], l.shape)
    flat = (rows[keep] * B + l[keep]).astype(np.int64)
    re = np.bincount(flat, weights=S.real[keep], minlength=F * B)
    im = np.bincount(flat, weights=S.imag[keep], minlength=F * B)
    return (re + 1j * im).reshape(F, B)


def sst_forward(x, g, gd, c: int, hop: int, nfft: int, fs: float, f1: float, f2: float,
                zoom: int, gamma: float, truncate: bool = False, frames=None, debug: bool = False):
    """Downsampled SST with selective reassignment and subdivision:
    two STFTs by Eq. (9) with g and g', omega_hat by Eq. (13), target by Eq. (28)/(29),
    squeeze into the band.  ``truncate`` restricts source bins to [k1, k2) (R12).
    Returns T [frames, B] complex128 (and S, Sd, l when ``debug``)."""
    band = band_grid(fs, nfft, f1, f2, zoom)
    S = stft(x, g, c, hop, nfft, frames)
    Sd = stft(x, gd, c, hop, nfft, frames)
    mask, r, fhat = if_estimate(S, Sd, nfft, gamma)
    if truncate:
        k = np.arange(S.shape[1])
        mask = mask & ((k >= band["k1"]) & (k < band["k2"]))[None, :]
    l = targets(fhat, mask, band["k1"], band["B"], zoom)
    T = squeeze(S, l, band["B"])
    if debug:
        return T, S, Sd, l
    return T


# --------------------------------------------------------------------------------------
# Approximate direct inverse -- Eq. 22-26, zero padding / zN_f IFFT.
# --------------------------------------------------------------------------------------
def discrete_constant(g, c: int) -> float:
    """C_d = g[M] sum g / sum g^2: the discrete counterpart of Eq. (22)/(24)'s C = sqrt 2
    (R15; used only with the DISCRETE_CONSTANT flag)."""
    g = np.asarray(g, dtype=np.float64)
    return float(g[c] * g.sum() / np.sum(g * g))


def sst_inverse(T, g, c: int, hop: int, nfft: int, zoom: int, k1: int, N: int,
                frame_begin: int = 0, n0: int = 0, n1: int | None = None,
                constant: str = "sqrt2"):
    """Reconstruction from the downsampled SST, Eq. (25)-(26) with P:L222:
    per frame, zero-pad T into a two-sided z N_f spectrum (bin z k1 + l gets T[m,l], bin
    z N_f - (z k1 + l) gets conj T[m,l]; DC and Nyquist not doubled, R14), multiply by the
    phase e^{-i 2 pi j M/(z N_f)} (R13), z N_f-point inverse DFT, real part, times z (R14),
    keep n = 0..L-1; overlap-add g[n] r~[m,n] at n + m H_t - M (Eq. 26) and divide by
    C d[n] (C = sqrt 2, Eq. 24, R15; d = frame diagonal, R2).

    T holds rows for frames [frame_begin, frame_begin + len(T)); the result covers the
    output window [n0, n1) and is exact there only if those rows include every frame
    touching the window (the caller guarantees it)."""
    g = np.asarray(g, dtype=np.float64)
    L = g.shape[0]
    n1 = N if n1 is None else n1
    Fr, B = T.shape
    zN = zoom * nfft
    j_band = zoom * k1 + np.arange(B)
    j_mirr = (zN - j_band) % zN
    own = (j_mirr != j_band)                 # DC / Nyquist are not mirrored (not doubled)
    phase = np.exp(-2j * np.pi * np.arange(zN) * c / zN)
    y = np.zeros(n1 - n0, dtype=np.float64)
    for fr in _chunks(np.arange(Fr), zN):
        Hs = np.zeros((len(fr), zN), dtype=np.complex128)
        Hs[:, j_band] = T[fr]
        Hs[:, j_mirr[own]] = np.conj(T[fr][:, own])
        rt = zoom * np.real(np.fft.ifft(Hs * phase[None, :], axis=1))[:, :L]   # r~[m, n]
        contrib = rt * g[None, :]
        idx = (fr[:, None] + frame_begin) * hop - c + np.arange(L)[None, :]
        ok = (idx >= n0) & (idx < n1)
        y += np.bincount(idx[ok] - n0, weights=contrib[ok], minlength=n1 - n0)
    d = frame_diagonal(g, c, hop, N, n0, n1)
    C = np.sqrt(2.0) if constant == "sqrt2" else discrete_constant(g, c)
    return y / (C * d)


# --------------------------------------------------------------------------------------
# Analysis formulas (§3-4).  Not on the hot path; pinned by printed paper values.
# --------------------------------------------------------------------------------------
def sigma_f_hz(sigma_s: float) -> float:
    """Frequency diffusion sigma_f = 1/(2 pi sigma) (Eq. 35), sigma in seconds."""
    return 1.0 / (2.0 * np.pi * sigma_s)


def hf_bound_eq38(N: int, sigma_s: float, fs: float) -> float:
    """Upper limit H_f < 3N / (4 pi sigma f_s) (Eq. 38)."""
    return 3.0 * N / (4.0 * np.pi * sigma_s * fs)


def hf_bound_eq46(N: int, sigma_s: float, fs: float) -> float:
    """H_f bound from Delta f < sqrt 2 sigma_f (Eq. 46) with Delta f = H_f fs / N (Eq. 12)."""
    return np.sqrt(2.0) * sigma_f_hz(sigma_s) * N / fs


def renyi_entropy(P, alpha: float = 3.0) -> float:
    """Renyi entropy of order alpha of a TFR P (Eq. 32), discrete sums."""
    P = np.asarray(P, dtype=np.float64)
    p = P / P.sum()
    return float(np.log2(np.sum(p ** alpha)) / (1.0 - alpha))


# --------------------------------------------------------------------------------------
# Mode retrieval: ridge, zone, Eq. 15 and the zone-masked inverse.
# P:L126-130 (§2.2) names "extracting TF ridges" without an algorithm; the ridge here is the
# penalised dynamic programme of SPEC.md's reading (reading R22 of DESIGN.md):
#   maximise  sum_m E[m, l_m] - lambda sum_m (l_{m+1} - l_m)^2,  E = log(|T| + eps),
#   eps = 1e-12 max|T|, ties -> the lowest bin index.
# --------------------------------------------------------------------------------------
def ridge_emission(T):
    """E[m, l] = log(|T[m, l]| + eps), eps = 1e-12 max|T| (R22)."""
    A = np.abs(np.asarray(T))
    eps = 1e-12 * A.max()
    return np.log(A + eps)


def ridge_dp(E, lam: float):
    """Viterbi for the R22 objective on emissions E[F, B], written as the plain recurrence
    V_0[l] = E[0, l],  V_m[l] = E[m, l] + max_{l'} (V_{m-1}[l'] - lam (l - l')^2)  (smallest
    maximising l'), then traceback from the smallest l maximising V_{F-1}.  O(F B^2)."""
    E = np.asarray(E, dtype=np.float64)
    F, B = E.shape
    l = np.arange(B)
    pen = lam * (l[:, None] - l[None, :]).astype(np.float64) ** 2     # pen[l, l']
    V = E[0].copy()
    back = np.zeros((F, B), dtype=np.int64)
    for m in range(1, F):
        cand = V[None, :] - pen                                         # [l, l']
        back[m] = np.argmax(cand, axis=1)                               # first maximiser
        V = E[m] + cand[l, back[m]]
    path = np.empty(F, dtype=np.int64)
    path[-1] = int(np.argmax(V))
    for m in range(F - 1, 0, -1):
        path[m - 1] = back[m, path[m]]
    return path


def ridge_suppress(E, path, half: int, floor: float):
    """After a ridge is found its zone +-half bins is suppressed (set to the floor emission
    log(eps)) before the next one."""
    E = np.array(E, dtype=np.float64, copy=True)
    B = E.shape[1]
    for m, c in enumerate(path):
        E[m, max(0, c - half):min(B, c + half + 1)] = floor
    return E


def extract_ridges(T, lam: float, count: int, suppress: int = 3):
    """`count` ridges found one after another by ridge_dp with zone suppression (R22)."""
    E = ridge_emission(T)
    floor = float(np.log(1e-12 * np.abs(np.asarray(T)).max()))
    paths = []
    for _ in range(count):
        p = ridge_dp(E, lam)
        paths.append(p)
        E = ridge_suppress(E, p, suppress, floor)
    return np.array(paths)


def zone_mask(path, half: int, B: int):
    """M_q[m] = {l : |l - path[m]| <= half} clipped to [0, B) ('offsetting the IFs in
    both directions to form a banded area')."""
    l = np.arange(B)
    return np.abs(l[None, :] - np.asarray(path)[:, None]) <= half


def mode_full(T, zone, g, c: int, nfft: int, k1: int, zoom: int):
    """Eq. (15): x_q[m] = 1/(2 pi g(0)) Re sum_{l in M_q[m]} T[m, l], H_t = 1.  The sum
    over the discrete band stands for the integral over omega with d omega = 2 pi / N_f per
    source bin (T sums S coefficients), and the one-sided band counts twice except DC (R14):
    x_q[m] = (2 / (N_f g[c])) Re sum_l w_l T[m, l],  w_l = 1/2 at z k1 + l = 0."""
    T = np.asarray(T)
    w = np.ones(T.shape[1])
    j = zoom * k1 + np.arange(T.shape[1])
    w[j == 0] = 0.5
    return 2.0 / (nfft * g[c]) * np.real(np.sum(np.where(zone, T, 0) * w[None, :], axis=1))


def retrieve_mode(T, zone, g, c: int, hop: int, nfft: int, zoom: int, k1: int, N: int):
    """§2.3: T outside the zone set to zero, then the downsampled inverse Eq. (25)-(26)."""
    return sst_inverse(np.where(zone, T, 0), g, c, hop, nfft, zoom, k1, N)
