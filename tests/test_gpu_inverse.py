"""Isolated inverse (K4) parity: a seeded synthetic band plane T from gen.planes (no SST arithmetic)
fed to BOTH the GPU inverse (Eq. 25-26 with P:L222's zero-padded z N_f IDFT, through the C ABI)
and the oracle's sst_inverse, so the inverse is checked on its own, not through forward flips
(SURVEY §8(c) "Reconstruction" check 1).  Tolerance: relative L2 <= 1e-4 (north star).

Cases: small records with z in {1, 2, 3, 4, 8, 20} and k1 > 0 (plus bands touching DC and
Nyquist, R14), the multi-pass path (N_f > 8192, both inverse formulations), C3 at full size in
the bench's launch configuration (whole-record sst_inverse, sampled output windows), and C5 at full
size through sst_inverse_accumulate + sst_inverse_finalize on output windows (its whole T is
256 GiB), including the windows around the P = 8 rank seams.
"""

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


# (N, fs, L, sigma, hop, nfft, f1, f2, z)
SMALL = [
    (30000, 1024.0, 257, 32.0, 4, 512, 100.0, 300.0, 1),
    (40000, 2048.0, 200, 25.0, 7, 256, 256.0, 768.0, 2),
    (30011, 25600.0, 512, 64.0, 4, 512, 1000.0, 9000.0, 3),
    (60000, 51200.0, 2048, 256.0, 16, 2048, 1000.0, 4000.0, 4),
    (30000, 25600.0, 512, 64.0, 4, 512, 50.0, 12800.0, 8),        # band up to Nyquist
    (20000, 1024.0, 301, 40.0, 10, 512, 100.0, 140.0, 20),
    (50000, 51200.0, 4096, 512.0, 32, 4096, 0.0, 6400.0, 2),       # band from DC
    (60000, 44100.0, 5745, 882.0, 1149, 8192, 1282 * 44100.0 / 8192, 1765 * 44100.0 / 8192, 8),
]


def _inverse_case(P, spec, seed):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    g, gd, c = O.gaussian_window(L, sigma)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    T = band_plane(seed, plan.bins, 0, plan.frames)
    y = plan.inverse(torch.from_numpy(T).to(DEV)).cpu().numpy()
    yo = O.sst_inverse(T.astype(np.complex128), g, c, hop, nfft, z, plan.layout["k1"], N)
    return rel(y, yo)


@pytest.mark.parametrize("spec", SMALL, ids=[f"nf{s[5]}_z{s[8]}_k1_{int(s[6] * s[5] / s[1])}" for s in SMALL])
def test_inverse_isolated_small(P, spec):
    e = _inverse_case(P, spec, seed=11)
    assert e <= 1e-4, e


@pytest.mark.parametrize("path", ["fft", "direct"])
def test_inverse_isolated_multipass(P, path, monkeypatch):
    monkeypatch.setenv("SST_MP_INVERSE", path)
    e = _inverse_case(P, (120000, 16384.0, 4001, 500.0, 256, 16384, 1000.0, 2000.0, 3), seed=12)
    assert e <= 1e-4, (path, e)


def _out_windows(N, W, count, seed, extra=()):
    rng = np.random.default_rng(seed)
    starts = [0, N - W] + [int(v) for v in rng.integers(0, N - W, size=count)] + [int(v) for v in extra]
    return sorted(set(min(max(0, s), N - W) for s in starts))


def test_inverse_isolated_c3_full(P):
    """C3 (N = 2^24, F = 2^20 frames, B = 640): the whole synthetic plane through sst_inverse in the
    bench's launch configuration; sampled output windows (both record edges) against the oracle."""
    cfg = get_config("C3")
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=0.0, device=0)
    T = band_plane(33, plan.bins, 0, plan.frames)
    y = plan.inverse(torch.from_numpy(T).to(DEV)).cpu().numpy()
    W = 4 * cfg.L
    for n0 in _out_windows(cfg.N, W, 6, 3):
        n1 = n0 + W
        fb = max(0, (n0 + c - cfg.L) // cfg.hop)
        fe = min(plan.frames, (n1 - 1 + c) // cfg.hop + 1)
        yo = O.sst_inverse(T[fb:fe].astype(np.complex128), g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N,
                           frame_begin=fb, n0=n0, n1=n1)
        assert rel(y[n0:n1], yo) <= 1e-4, n0


def test_inverse_isolated_c5_windows(P):
    """C5 (N = 2^26, z = 8, B = 2048; whole T = 256 GiB): frames covering each output window
    accumulated with sst_inverse_accumulate into a window buffer and finalised, against the oracle;
    windows at both record edges, random positions and the P = 8 rank seams."""
    cfg = get_config("C5")
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=0.0, device=0)
    F = plan.frames
    W = 8 * cfg.L
    seams = [(F * r // 8) * cfg.hop - c - W // 2 for r in range(1, 8)]
    for n0 in _out_windows(cfg.N, W, 4, 5, seams):
        n1 = n0 + W
        fb = max(0, (n0 + c - cfg.L) // cfg.hop)
        fe = min(F, (n1 - 1 + c) // cfg.hop + 1)
        T = band_plane(55, plan.bins, fb, fe)
        lo = max(0, fb * cfg.hop - c)
        hi = min(cfg.N, (fe - 1) * cfg.hop - c + cfg.L)
        y = torch.zeros(hi - lo, dtype=torch.float32, device=DEV)
        plan.inverse_accumulate(torch.from_numpy(T).to(DEV), fb, fe, y, y_off=lo)
        plan.inverse_finalize(y[n0 - lo:n1 - lo], y_off=n0)
        yo = O.sst_inverse(T.astype(np.complex128), g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N,
                           frame_begin=fb, n0=n0, n1=n1)
        assert rel(y[n0 - lo:n1 - lo].cpu().numpy(), yo) <= 1e-4, n0
