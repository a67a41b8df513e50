"""f3b: the frequency-domain filter-bank forward (§6) that plans choose
for SST_SOURCE_TRUNCATE (R12) with a narrow band, against the fp64 oracle with truncate=True:
  - S, S' of the band's source bins from the filter bank (sst_stft_band): relative Frobenius <= 1e-5;
  - T: relative L2 <= 1e-3 against the oracle, and against the fused path's T of the same plan
    parameters (SST_FILTERBANK=0) to fp32 rounding of S (both take every decision like the oracle,
    R23);
  - frame sub-ranges with offset x slices reproduce the rows of the whole-record forward (the same
    blocks on the global frame grid; values to fp32 rounding: the zero fill outside a slice changes
    the rounding, not the exact value, of a block's transform);
  - the inverse of the filter-bank T against the oracle's inverse (<= 1e-4)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle as O  # noqa: E402
from tests._helpers import rel  # noqa: E402

DEV = torch.device("cuda:0")

# (N, fs, L, sigma, hop, nfft, f1, f2, z): C3-, C2-, C4-like shapes and an offset band with z = 3
FB = [
    (200000, 51200.0, 2048, 256.0, 16, 2048, 0.0, 4000.0, 4),
    (100000, 25600.0, 1024, 128.0, 8, 1024, 0.0, 2000.0, 2),
    (300000, 51200.0, 4096, 512.0, 32, 4096, 0.0, 6400.0, 2),
    (120000, 25600.0, 1024, 128.0, 8, 1024, 3000.0, 5000.0, 3),
]
IDS = ["c3like", "c2like", "c4like", "offset_z3"]


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


def _sig(N, fs, seed):
    rng = np.random.default_rng(seed)
    t = np.arange(N) / fs
    x = np.zeros(N)
    for h, a in zip((1, 2, 3, 5), (1.0, 0.5, 0.3, 0.2)):
        x += a * np.cos(2 * np.pi * h * (60 * t + 20 * t * t / t[-1]) + rng.uniform(0, 6.28))
    x += 0.4 * np.cos(2 * np.pi * 0.05 * fs * t + 1.0)
    x += 0.2 * rng.standard_normal(N)
    return x.astype(np.float32)


def _plan(P, spec, gamma):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    return P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, flags=P.SST_SOURCE_TRUNCATE, device=0)


def test_filterbank_choice(P, monkeypatch):
    """SST_FILTER_BANK selects the filter bank for a truncated band; without it the plan's cost model
    (calibrated on B200, where the fused forward is faster on C2-C4) keeps the fused path; never
    without SST_SOURCE_TRUNCATE."""
    monkeypatch.delenv("SST_FILTERBANK", raising=False)
    N, fs, L, sigma, hop, nfft, f1, f2, z = FB[0]
    for spec in FB[:3]:
        assert _plan(P, spec, 1e-4).forward_path == P.SST_PATH_FUSED
    fl = P.SST_SOURCE_TRUNCATE | P.SST_FILTER_BANK
    assert P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, flags=fl, device=0).forward_path == \
        P.SST_PATH_FILTERBANK
    assert P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, flags=P.SST_FILTER_BANK,
                  device=0).forward_path == P.SST_PATH_FUSED


@pytest.mark.parametrize("spec", FB, ids=IDS)
def test_filterbank_forward(P, spec, monkeypatch):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _sig(N, fs, N)
    g, gd, c = O.gaussian_window(L, sigma)
    gamma = 1e-6 * float(np.sum(g)) * float(np.abs(x).max())
    monkeypatch.setenv("SST_FILTERBANK", "1")                 # every shape here, C4-like included
    plan = _plan(P, spec, gamma)
    assert plan.forward_path == P.SST_PATH_FILTERBANK
    xd = torch.from_numpy(x).to(DEV)
    k1, k2 = plan.layout["k1"], plan.layout["k2"]
    # band STFT of the filter bank vs Eq. 9 (oracle)
    fr = np.arange(plan.frames)
    S, Sd = plan.stft_band(xd)
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)[:, k1:k2]
    Sdo = O.stft(x.astype(np.float64), gd, c, hop, nfft)[:, k1:k2]
    assert rel(S.cpu().numpy(), So) <= 1e-5
    assert rel(Sd.cpu().numpy(), Sdo) <= 1e-5
    # T vs the oracle (truncate) and vs the fused path
    T = plan.forward(xd)
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, truncate=True, frames=fr)
    e = rel(T.cpu().numpy(), To)
    assert e <= 1e-3, e
    monkeypatch.setenv("SST_FILTERBANK", "0")
    plan_f = _plan(P, spec, gamma)
    assert plan_f.forward_path == P.SST_PATH_FUSED
    Tf = plan_f.forward(xd)
    assert rel(T.cpu().numpy(), Tf.cpu().numpy()) <= 1e-5
    # inverse of the filter-bank T
    y = plan.inverse(T).cpu().numpy()
    yo = O.sst_inverse(To, g, c, hop, nfft, z, k1, N)
    assert rel(y, yo) <= 1e-4
    print(spec, "T", e, "vs fused", rel(T.cpu().numpy(), Tf.cpu().numpy()), "counters", plan.counters())


def test_filterbank_frame_ranges(P):
    spec = FB[0]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _sig(N, fs, 3)
    plan = _plan(P, spec, 1e-4)
    xd = torch.from_numpy(x).to(DEV)
    full = plan.forward(xd)
    F = plan.frames
    c = L // 2
    for fb, fe in [(0, 7), (383, 1200), (F - 9, F), (5000, 5001)]:
        lo = max(0, fb * hop - c)
        hi = min(N, (fe - 1) * hop - c + L)
        part = plan.forward(xd[lo:hi].contiguous(), fb, fe, x_off=lo)
        assert rel(part.cpu().numpy(), full[fb:fe].cpu().numpy()) <= 1e-5, (fb, fe)
        # same launch twice: bitwise identical (deterministic)
        assert torch.equal(part, plan.forward(xd[lo:hi].contiguous(), fb, fe, x_off=lo))
