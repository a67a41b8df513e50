"""GPU parity of the large-N_f multi-pass path (8192 < N_f <= 65536) against the
fp64 oracle.  Shapes: the paper's §5.2 chatter analysis (fs = 10240 Hz, N = 573440,
sigma = 0.1 s, N_f = 2^15, H = 667 with band 1200-1400 Hz, and H = 200 with band 630-640 Hz, z = 20;
reading R19 takes the printed "H_f" as H_t) on the synthetic stand-in gen.signals.s52_milling, an
N_f = 2^14 selective case and an N_f = 2^16 full-band case whose B = 32768 bins exceed one shared-
memory squeeze pass.  Same tolerances as test_gpu_parity.py; the oracle sees only x and its window.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle as O  # noqa: E402
from gen.signals import s52_milling  # noqa: E402
from tests._helpers import assert_flips, flip_stats, rel  # noqa: E402

DEV = torch.device("cuda:0")

S52_N, S52_FS, S52_SIGMA = 573440, 10240.0, 1024.0
S52_L = 8 * 1024 + 1                      # +-4 sigma (the paper's window length is unstated)

# (name, N, fs, L, sigma, hop, nfft, f1, f2, z)
BIG = [
    ("s52_chatter", S52_N, S52_FS, S52_L, S52_SIGMA, 667, 32768, 1200.0, 1400.0, 1),
    ("s52_spindle_z20", S52_N, S52_FS, S52_L, S52_SIGMA, 200, 32768, 630.0, 640.0, 20),
    ("nf16k_sel_z3", 200000, 16384.0, 4001, 500.0, 256, 16384, 1000.0, 3000.0, 3),
    ("nf64k_full", 300000, 65536.0, 20001, 2500.0, 4096, 65536, 0.0, 32768.0, 1),
]


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


def _sig(name, N, fs):
    if name.startswith("s52"):
        return s52_milling(52, N, fs)
    rng = np.random.default_rng(N)
    t = np.arange(N) / fs
    x = 0.5 * np.cos(2 * np.pi * (0.05 * fs * t + 0.01 * fs * t * t / t[-1]))
    for f in rng.uniform(0.03, 0.45, size=5) * fs:
        x += rng.uniform(0.3, 1.0) * np.cos(2 * np.pi * f * t + rng.uniform(0, 6.28))
    x += 0.1 * rng.standard_normal(N)
    return x.astype(np.float32)


def _setup(P, spec, gamma=None):
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _sig(name, N, fs)
    g, gd, c = O.gaussian_window(L, sigma)
    if gamma is None:
        gamma = 1e-6 * float(np.sum(g)) * float(np.abs(x).max())     # reading R6 (bound from x)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, device=0)
    return x, g, gd, c, gamma, plan


def _windows(F, size=24):
    return [(0, min(F, size)), (F // 2 - size // 2, F // 2 + size // 2), (max(0, F - size), F)]


@pytest.mark.parametrize("spec", BIG, ids=[s[0] for s in BIG])
def test_mp_stft_parity(P, spec):
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    for fb, fe in _windows(plan.frames):
        S, Sd = plan.stft(xd, fb, fe)
        fr = np.arange(fb, fe)
        So = O.stft(x.astype(np.float64), g, c, hop, nfft, frames=fr)
        Sdo = O.stft(x.astype(np.float64), gd, c, hop, nfft, frames=fr)
        print(name, "stft", fb, rel(S.cpu().numpy(), So), rel(Sd.cpu().numpy(), Sdo))
        assert rel(S.cpu().numpy(), So) <= 1e-5, (fb, rel(S.cpu().numpy(), So))
        assert rel(Sd.cpu().numpy(), Sdo) <= 1e-5, (fb, rel(Sd.cpu().numpy(), Sdo))


@pytest.mark.parametrize("spec", BIG, ids=[s[0] for s in BIG])
def test_mp_forward_parity_and_flips(P, spec):
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    Tall = plan.forward(xd).cpu().numpy()
    assert Tall.shape == (plan.frames, plan.bins)
    for fb, fe in _windows(plan.frames):
        fr = np.arange(fb, fe)
        lg = plan.targets(xd, fb, fe).cpu().numpy()
        To, S, Sd, lo = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma,
                                      frames=fr, debug=True)
        _, _, fhat = O.if_estimate(S, Sd, nfft, gamma)
        st = flip_stats(lg, lo, S, fhat, plan.layout["k1"], z, gamma)
        assert_flips(st, fb)
        e = rel(Tall[fb:fe], To)
        print(name, "forward", fb, e, st)
        assert e <= 1e-3, (fb, e, st)


@pytest.mark.parametrize("spec", [BIG[0], BIG[2]], ids=[BIG[0][0], BIG[2][0]])
def test_mp_inverse_whole(P, spec):
    """Whole-record forward + inverse vs the oracle's inverse (Eq. 25-26) of the oracle's T; the
    paper reconstructs the 1300-1400 Hz part of the §5.2 record this way (Fig. 17)."""
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    y = plan.inverse(plan.forward(xd)).cpu().numpy()
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma)
    yo = O.sst_inverse(To, g, c, hop, nfft, z, plan.layout["k1"], N)
    print(name, "inverse", rel(y, yo))
    assert rel(y, yo) <= 1e-4, rel(y, yo)


@pytest.mark.parametrize("spec", [BIG[1], BIG[3]], ids=[BIG[1][0], BIG[3][0]])
def test_mp_inverse_windows(P, spec):
    """inverse_accumulate of the frames covering sampled output windows + inverse_finalize,
    against the oracle's forward + inverse of those frames (both record edges)."""
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    W = 2 * L
    for n0 in (0, N // 2, N - W):
        n1 = n0 + W
        fb = max(0, (n0 + c - L) // hop)
        fe = min(plan.frames, (n1 - 1 + c) // hop + 1)
        T = plan.forward(xd, fb, fe)
        lo = max(0, fb * hop - c)
        hi = min(N, (fe - 1) * hop - c + L)
        y = torch.zeros(hi - lo, dtype=torch.float32, device=DEV)
        plan.inverse_accumulate(T, fb, fe, y, y_off=lo)
        plan.inverse_finalize(y[n0 - lo:n1 - lo], y_off=n0)
        To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, frames=np.arange(fb, fe))
        yo = O.sst_inverse(To, g, c, hop, nfft, z, plan.layout["k1"], N, frame_begin=fb, n0=n0, n1=n1)
        e = rel(y[n0 - lo:n1 - lo].cpu().numpy(), yo)
        print(name, "inverse window", n0, e)
        assert e <= 1e-4, (n0, e)


def test_mp_istft_round_trip(P):
    """Eq. 10-11 synthesis of the analysis is exact (pin P4) on the multi-pass path too."""
    spec = BIG[2]
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    S, _ = plan.stft(torch.from_numpy(x).to(DEV))
    y = plan.istft(S).cpu().numpy()
    assert rel(y, x.astype(np.float64)) <= 1e-5


def test_mp_bitwise_chunking_and_repeat(P):
    """The forward is chunked internally (scratch for 512 frames at N_f = 2^15): frame sub-ranges
    and repeated calls give bitwise the same T (exact fixed-point squeeze)."""
    spec = BIG[0]
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    T1 = plan.forward(xd)
    T2 = plan.forward(xd)
    assert torch.equal(T1, T2)
    F = plan.frames
    parts = [plan.forward(xd, a, b) for a, b in ((0, 300), (300, 301), (301, F))]
    assert torch.equal(torch.cat(parts), T1)
    # x slice with an offset
    fb, fe = 500, 560
    lo = fb * spec[5] - c
    hi = min(spec[1], (fe - 1) * spec[5] - c + spec[3])
    Ts = plan.forward(xd[lo:hi].contiguous(), fb, fe, x_off=lo)
    assert torch.equal(Ts, T1[fb:fe])


def test_mp_relative_gamma_and_absmax(P):
    """SST_GAMMA_RELATIVE on the multi-pass path: the absmax pre-pass matches the oracle's max|S|,
    and the forward with gamma = 1e-3 max|S| matches the oracle at its own (fp64) threshold."""
    spec = BIG[2]
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _sig(name, N, fs)
    g, gd, c = O.gaussian_window(L, sigma)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-3, flags=P.SST_GAMMA_RELATIVE, device=0)
    xd = torch.from_numpy(x).to(DEV)
    amax = float(plan.absmax(xd).cpu())
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    ref = float(np.abs(So).max())
    assert abs(amax - ref) <= 1e-5 * ref
    T = plan.forward(xd).cpu().numpy()
    lg = plan.targets(xd).cpu().numpy()
    gamma = 1e-3 * ref
    To, S, Sd, lo = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, debug=True)
    _, _, fhat = O.if_estimate(S, Sd, nfft, gamma)
    st = flip_stats(lg, lo, S, fhat, plan.layout["k1"], z, gamma)
    assert_flips(st)
    e = rel(T, To)
    assert e <= 1e-3, (e, st)


# edge shapes of the multi-pass path: a full-length window (L = N_f, even, c = N_f/2) on a record of
# exactly N_f samples; a short window (L = N_f/8: mostly zero gather) with a non-power-of-two z and a
# band not starting at DC; a 101-tap window zero-padded 160x at z = 7 (r ill-conditioned: the fp32
# decisions there are the ones R23 re-takes in fp64); two frames; a single frame with the window
# centre at tap 0.
EDGE = [
    ("nf16k_fullwin", 16384, 16384.0, 16384, 2048.0, 4096, 16384, 0.0, 8192.0, 1),
    ("nf16k_shortwin_z7", 50000, 16384.0, 2001, 250.0, 37, 16384, 2000.0, 2500.0, 7),
    ("nf16k_101tap_z7", 50000, 16384.0, 101, 12.5, 37, 16384, 2000.0, 2500.0, 7),
    ("nf32k_two_frames", 32768, 32768.0, 32768, 4096.0, 16384, 32768, 1000.0, 5000.0, 2),
    ("nf32k_one_frame_c0", 32768, 32768.0, 32768, 8192.0, 32768, 32768, 1000.0, 5000.0, 2, 0),
]


def _sig_sweep(N, fs, seed):
    """Three crossing-free linear chirps plus noise: every ridge moves from frame to frame, unlike
    a stationary tone, whose ridge coefficient sits at the same distance from a rounding boundary in
    every frame (one unlucky tone then flips a large coefficient in all frames at once)."""
    rng = np.random.default_rng(seed)
    t = np.arange(N) / fs
    x = np.zeros(N)
    for lo, hi in ((0.05, 0.09), (0.12, 0.16), (0.25, 0.40)):
        f0, f1 = lo * fs, hi * fs
        x += rng.uniform(0.5, 1.0) * np.cos(2 * np.pi * (f0 * t + 0.5 * (f1 - f0) * t * t / t[-1]) + rng.uniform(0, 6.28))
    x += 0.05 * rng.standard_normal(N)
    return x.astype(np.float32)


@pytest.mark.parametrize("spec", EDGE, ids=[s[0] for s in EDGE])
def test_mp_edge_shapes(P, spec):
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec[:10]
    center = spec[10] if len(spec) > 10 else None
    x = _sig_sweep(N, fs, N + L)
    g, gd, c = O.gaussian_window(L, sigma, center)
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    Sdo = O.stft(x.astype(np.float64), gd, c, hop, nfft)
    gamma = 1e-6 * float(np.abs(So).max())
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, device=0, center=c)
    xd = torch.from_numpy(x).to(DEV)
    S, Sd = plan.stft(xd)
    assert rel(S.cpu().numpy(), So) <= 1e-5 and rel(Sd.cpu().numpy(), Sdo) <= 1e-5
    T = plan.forward(xd).cpu().numpy()
    lg = plan.targets(xd).cpu().numpy()
    To, S2, Sd2, lo = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, debug=True)
    _, _, fhat = O.if_estimate(S2, Sd2, nfft, gamma)
    st = flip_stats(lg, lo, S2, fhat, plan.layout["k1"], z, gamma)
    assert_flips(st)
    e = rel(T, To)
    assert e <= 1e-3, (e, st)
    y = plan.inverse(plan.forward(xd)).cpu().numpy()
    yo = O.sst_inverse(To, g, c, hop, nfft, z, plan.layout["k1"], N)
    print(name, "T", e, "inverse", rel(y, yo), st)
    assert rel(y, yo) <= 1e-4, rel(y, yo)


@pytest.mark.parametrize("path", ["fft", "direct"])
@pytest.mark.parametrize("spec", [BIG[1], BIG[2]], ids=[BIG[1][0], BIG[2][0]])
def test_mp_inverse_both_paths(P, spec, path, monkeypatch):
    """Both inverse formulations of the multi-pass path (residue-split FFTs, direct band sum; the
    plan picks one by cost) against the oracle on an output window in the middle of the record."""
    monkeypatch.setenv("SST_MP_INVERSE", path)
    name, N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c, gamma, plan = _setup(P, spec)
    xd = torch.from_numpy(x).to(DEV)
    n0 = N // 3
    n1 = n0 + 2 * L
    fb = max(0, (n0 + c - L) // hop)
    fe = min(plan.frames, (n1 - 1 + c) // hop + 1)
    T = plan.forward(xd, fb, fe)
    lo = max(0, fb * hop - c)
    hi = min(N, (fe - 1) * hop - c + L)
    y = torch.zeros(hi - lo, dtype=torch.float32, device=DEV)
    plan.inverse_accumulate(T, fb, fe, y, y_off=lo)
    plan.inverse_finalize(y[n0 - lo:n1 - lo], y_off=n0)
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, frames=np.arange(fb, fe))
    yo = O.sst_inverse(To, g, c, hop, nfft, z, plan.layout["k1"], N, frame_begin=fb, n0=n0, n1=n1)
    e = rel(y[n0 - lo:n1 - lo].cpu().numpy(), yo)
    print(name, path, e)
    assert e <= 1e-4, e
