"""Narrow-band inverse path (inv_nb_kernel.cuh, SST_IPATH_NARROWBAND, incl. its full-band form for C5's
shape): isolated parity against the
oracle's sst_inverse (Eq. 25-26, with P:L222's zero-padded z N_f IDFT) on seeded synthetic
band planes from gen.planes (no SST arithmetic), at relative L2 <= 1e-4 (north star), plus agreement
with the residue-split kernel (SST_IPATH_RESIDUE, forced by SST_INV_NB=0 at plan creation) on the
same plane.  Cases cover both N_f instantiations (1024, 2048), z in {1, 2, 4, 8}, bands from DC and
with k1 > 0, band/mirror row counts RM <= 5 and 6..8, the full band (N_f = 512, z = 4, 8), hops
8-40 and 3, 5, 12, an odd frame
count (last pair without frame B), frame sub-ranges through sst_inverse_accumulate, and C2 / C3 at
full size in the bench's launch configuration (sampled output windows of the whole record).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle as O  # noqa: E402
from gen import get_config  # noqa: E402
from gen.planes import band_plane  # noqa: E402
from tests._helpers import rel  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


# (N, fs, L = N_f, sigma, hop, N_f, f1, f2, z)
NB = [
    (60000, 51200.0, 2048, 256.0, 16, 2048, 0.0, 4000.0, 4),       # C3 shape, band from DC, RM = 5
    (60000, 51200.0, 2048, 256.0, 16, 2048, 1000.0, 4000.0, 4),    # k1 > 0
    (50000, 51200.0, 2048, 256.0, 8, 2048, 0.0, 6400.0, 1),        # z = 1, RM = 8
    (40000, 51200.0, 2048, 256.0, 24, 2048, 2000.0, 5000.0, 2),    # z = 2, hop 24, RM = 5
    (30000, 51200.0, 2048, 256.0, 32, 2048, 0.0, 3000.0, 8),       # z = 8
    (70001, 25600.0, 1024, 128.0, 8, 1024, 0.0, 2000.0, 2),        # C2 shape, odd N
    (50000, 25600.0, 1024, 128.0, 16, 1024, 400.0, 3200.0, 4),     # N_f = 1024, z = 4, RM = 8
    (30000, 25600.0, 1024, 128.0, 40, 1024, 0.0, 1200.0, 8),       # N_f = 1024, z = 8, hop 40
    (20000, 25600.0, 1024, 128.0, 8, 1024, 100.0, 1500.0, 1),      # N_f = 1024, z = 1
    (50000, 51200.0, 2048, 256.0, 12, 2048, 0.0, 4000.0, 4),       # hop 12 (not a multiple of 8)
    (30000, 25600.0, 1024, 128.0, 5, 1024, 0.0, 2000.0, 2),        # hop 5
    (40000, 25600.0, 512, 64.0, 4, 512, 0.0, 12800.0, 8),          # C5 shape: full band (k1 = 0, B = z N/2)
    (30001, 25600.0, 512, 64.0, 3, 512, 0.0, 12800.0, 4),          # full band, z = 4, hop 3, odd N
]


def _ids(s):
    return f"nf{s[5]}_h{s[4]}_z{s[8]}_f{int(s[6])}-{int(s[7])}_N{s[0]}"


def _plan(P, spec, nb=True):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    old = os.environ.get("SST_INV_NB")
    os.environ["SST_INV_NB"] = "1" if nb else "0"
    try:
        return P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    finally:
        if old is None:
            del os.environ["SST_INV_NB"]
        else:
            os.environ["SST_INV_NB"] = old


@pytest.mark.parametrize("spec", NB, ids=[_ids(s) for s in NB])
def test_nb_inverse_isolated(P, spec):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    plan = _plan(P, spec)
    assert plan.inverse_path == P.SST_IPATH_NARROWBAND
    ref = _plan(P, spec, nb=False)
    assert ref.inverse_path == P.SST_IPATH_RESIDUE
    g, gd, c = O.gaussian_window(L, sigma)
    T = band_plane(23, plan.bins, 0, plan.frames)
    Td = torch.from_numpy(T).to(DEV)
    y = plan.inverse(Td).cpu().numpy()
    yo = O.sst_inverse(T.astype(np.complex128), g, c, hop, nfft, z, plan.layout["k1"], N)
    e = rel(y, yo)
    assert e <= 1e-4, e
    yr = ref.inverse(Td).cpu().numpy()
    assert rel(y, yr) <= 2e-5


def test_nb_accumulate_subranges(P):
    """sst_inverse_accumulate over ragged frame sub-ranges (odd counts: pairs without frame B, CTA seams
    inside each launch) + finalize equals the whole-record inverse."""
    spec = NB[0]
    plan = _plan(P, spec)
    assert plan.inverse_path == P.SST_IPATH_NARROWBAND
    T = torch.from_numpy(band_plane(5, plan.bins, 0, plan.frames)).to(DEV)
    y_whole = plan.inverse(T)
    y = torch.zeros(plan.n, dtype=torch.float32, device=DEV)
    cuts = [0, 1, 778, 779, 2001, plan.frames]
    for a, b in zip(cuts[:-1], cuts[1:]):
        plan.inverse_accumulate(T[a:b], a, b, y)
    plan.inverse_finalize(y)
    assert rel(y.cpu().numpy(), y_whole.cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_nb_config_full(P, name):
    """C2 / C3 at full size through the whole-record sst_inverse (the bench's launch configuration) on a
    seeded band plane; sampled output windows (start, middle, end, CTA borders) against the oracle's
    inverse of the frames that reach them."""
    cfg = get_config(name)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=0.0, device=0)
    assert plan.inverse_path == P.SST_IPATH_NARROWBAND
    F, B = plan.frames, plan.bins
    T = band_plane(77, B, 0, F)
    y = plan.inverse(torch.from_numpy(T).to(DEV)).cpu().numpy()
    W = 4 * cfg.L
    rng = np.random.default_rng(3)
    # windows at both record edges, random positions and CTA borders of the launch
    fpc = -(-F // (148 * 4))
    borders = [k * fpc * cfg.hop - c - W // 2 for k in (1, 97, 301)]
    starts = [0, cfg.N - W] + [int(v) for v in rng.integers(0, cfg.N - W, size=5)] + borders
    for n0 in sorted(set(min(max(0, s), cfg.N - W) for s in starts)):
        n1 = n0 + W
        fb = max(0, (n0 + c - cfg.L) // cfg.hop)
        fe = min(F, (n1 - 1 + c) // cfg.hop + 1)
        yo = O.sst_inverse(T[fb:fe].astype(np.complex128), g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N,
                           frame_begin=fb, n0=n0, n1=n1)
        assert rel(y[n0:n1], yo) <= 1e-4, n0
