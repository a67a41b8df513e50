"""fp64 CPU oracle for the downsampled STFT-based SST of He & Cao (arXiv 2003.07065).

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2003_07065_b200`` + ``libsst.so``) never imports, links or calls it and
fails loudly when its CUDA library is missing.

The oracle shares no code with the CUDA path: it is plain numpy written from
PAPER.md, one function per equation, each citing the passage it follows
(``P:Lnnn`` = PAPER.md line nnn).  Readings where the paper is silent or garbled
are the R-numbered readings of DESIGN.md §3.

Pinning: every function here is pinned by a ``-m "not gpu"``
test against something other than itself (brute force, closed forms, paper
values, invariants).  Parity unpinned: the numeric value of the threshold
gamma (any gamma >= 0 is valid, Eq. 13 never quantifies it) and the tie-break at
exact half-bin targets (measure-zero; frozen by reading R10).
"""

from .sst import (  # noqa: F401
    gaussian_window,
    frame_count,
    stft,
    stft_direct,
    stft_inverse,
    if_estimate,
    band_grid,
    targets,
    targets_bruteforce,
    squeeze,
    sst_forward,
    sst_inverse,
    frame_diagonal,
    discrete_constant,
    sigma_f_hz,
    hf_bound_eq38,
    hf_bound_eq46,
    renyi_entropy,
    ridge_emission,
    ridge_dp,
    ridge_suppress,
    extract_ridges,
    zone_mask,
    mode_full,
    retrieve_mode,
)
