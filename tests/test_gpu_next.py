"""GPU parity of the SURVEY §8(f) rows built so far, through the C ABI, against the fp64 oracle.

* f2 -- plain downsampled STFT synthesis, Eq. (10)-(11): ``sst_istft`` of the GPU's own
  ``sst_stft`` spectrum reproduces x (exact identity up to fp32 rounding, pin P4) and equals the
  oracle's ``stft_inverse`` of the oracle's STFT.
* f4 -- Renyi entropy, Eq. (32): ``sst_renyi`` of a GPU plane equals the oracle's
  ``renyi_entropy`` of the same plane.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle as O  # noqa: E402
from gen import get_config  # noqa: E402
from tests._helpers import config_gamma, make_plan, rel, signal  # noqa: E402
from tests.test_gpu_parity import SMALL, _case  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


@pytest.mark.parametrize("spec", SMALL, ids=[f"nf{s[5]}_h{s[4]}_L{s[2]}_N{s[0]}" for s in SMALL])
def test_istft_round_trip(P, spec):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    xd = torch.from_numpy(x).to(DEV)
    S, _ = plan.stft(xd)
    y = plan.istft(S).cpu().numpy()
    # Eq. 10-11 is an exact identity (P4): synthesis of the analysis returns x
    assert rel(y, x.astype(np.float64)) <= 1e-5
    # and the kernel equals the oracle's synthesis of the oracle's STFT
    Sfull = O.stft(x.astype(np.float64), g, c, hop, nfft, full=True)
    yo = O.stft_inverse(Sfull, g, c, hop, nfft, N)
    assert rel(y, yo) <= 1e-5


def test_istft_is_linear_and_padded_rows(P):
    spec = SMALL[3]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    xd = torch.from_numpy(x).to(DEV)
    S, _ = plan.stft(xd)
    Sp = torch.zeros((S.shape[0], S.shape[1] + 5), dtype=torch.complex64, device=DEV)
    Sp[:, :S.shape[1]] = S
    y1 = plan.istft(S)
    y2 = plan.istft(Sp)
    assert torch.equal(y1, y2)
    y3 = plan.istft((2.0 * S).contiguous())
    assert torch.allclose(y3, 2.0 * y1, rtol=0, atol=1e-6 * float(y1.abs().max()))


@pytest.mark.parametrize("alpha", [3.0, 2.0, 0.5])
def test_renyi_matches_oracle(P, alpha):
    cfg = get_config("C1")
    x = signal("C1")
    plan = make_plan(P, cfg, config_gamma(cfg, x))
    T = plan.forward(torch.from_numpy(x).to(DEV))
    out = plan.renyi(T, alpha).cpu().numpy()
    Pn = np.abs(T.cpu().numpy().astype(np.complex128)) ** 2
    assert out[0] == pytest.approx(Pn.sum(), rel=1e-12)
    assert out[1] == pytest.approx((Pn ** alpha).sum(), rel=1e-10)
    assert out[2] == pytest.approx(O.renyi_entropy(Pn, alpha), rel=1e-10, abs=1e-10)
    # reproducible: same bits on a second call
    assert np.array_equal(plan.renyi(T, alpha).cpu().numpy(), out)


def test_renyi_sst_sharper_than_stft(P):
    """The SST plane concentrates energy: its Renyi entropy is below the STFT's."""
    cfg = get_config("C1")
    x = signal("C1")
    plan = make_plan(P, cfg, config_gamma(cfg, x))
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    S, _ = plan.stft(xd)
    h_sst = float(plan.renyi(T)[2])
    Sb = S[:, :plan.bins].contiguous()
    h_stft = float(plan.renyi(Sb)[2])
    assert h_sst < h_stft - 1.0, (h_sst, h_stft)


def test_renyi_errors(P):
    cfg = get_config("C1")
    plan = make_plan(P, cfg, 0.0)
    T = torch.zeros((4, plan.bins), dtype=torch.complex64, device=DEV)
    with pytest.raises(P.SSTError):
        plan.renyi(T, 1.0)
    with pytest.raises(P.SSTError):
        plan.renyi(T, -2.0)
