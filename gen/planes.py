"""Seeded synthetic band planes T[F, B] (complex64) for the isolated inverse parity test (K4).

No SST arithmetic here: only random numbers with a ridge-like structure, generated per block of
``ROWS`` rows from ``PCG64(SeedSequence([seed, 7, block]))`` so any row range [r0, r1) is produced on
its own, bit-identical to the same rows of the whole plane (the GPU test uploads the whole plane;
the oracle regenerates only the rows of the frames it checks).

Each row holds a dense complex Gaussian floor (scale ``floor``) plus ``ridges`` narrow bumps whose
centres wander slowly with the row index (a stand-in for squeezed components: a few large
coefficients per row over a weak background).  Bin 0 and bin B-1 carry values like any other bin,
so the inverse's DC / Nyquist handling (R14) is exercised when the band touches them.
"""

from __future__ import annotations

import numpy as np

ROWS = 1024
_STREAM = 7


def _block(seed: int, b: int, B: int, ridges: int, floor: float) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _STREAM, b])))
    T = (rng.standard_normal((ROWS, B)) + 1j * rng.standard_normal((ROWS, B))) * floor
    rows = b * ROWS + np.arange(ROWS)
    cols = np.arange(B)
    prm = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, _STREAM, 1 << 40])))
    for _ in range(ridges):
        c0, amp, per, width = prm.uniform(0.1, 0.9) * B, prm.uniform(0.5, 1.0), prm.uniform(2e3, 2e4), prm.uniform(0.6, 2.0)
        ph = prm.uniform(0, 2 * np.pi)
        centre = c0 + 0.05 * B * np.sin(2 * np.pi * rows / per)
        bump = amp * np.exp(-0.5 * ((cols[None, :] - centre[:, None]) / width) ** 2)
        T += bump * np.exp(1j * (ph + 0.01 * rows))[:, None]
    return T.astype(np.complex64)


def band_plane(seed: int, B: int, r0: int, r1: int, ridges: int = 3, floor: float = 0.05) -> np.ndarray:
    """Rows [r0, r1) of the seeded plane with B bins, complex64 [r1 - r0, B]."""
    out = np.empty((r1 - r0, B), dtype=np.complex64)
    for b in range(r0 // ROWS, (r1 - 1) // ROWS + 1):
        blk = _block(seed, b, B, ridges, floor)
        lo, hi = max(r0, b * ROWS), min(r1, (b + 1) * ROWS)
        out[lo - r0:hi - r0] = blk[lo - b * ROWS:hi - b * ROWS]
    return out
