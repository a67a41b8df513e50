"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star), asserted unconditionally in every test: STFT relative
Frobenius <= 1e-5; squeezed plane relative L2 <= 1e-3 with target disagreement <= 1e-4 of
above-threshold coefficients, every flip lying within 1e-4 coarse bins of a rounding boundary
(tests/_helpers.assert_flips; the GPU re-takes uncertain decisions in fp64, reading R23);
reconstruction relative L2 <= 1e-4.  The oracle only ever receives the same fp32 samples (upcast to
fp64) and its own window -- never GPU output.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle as O  # noqa: E402
from gen import get_config  # noqa: E402
from tests._helpers import assert_flips, config_gamma, flip_stats, make_plan, rel, signal  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


# (N, fs, L, sigma, hop, nfft, f1, f2, z): every N2 instantiation, ragged N / F, L < N_f,
# selective bands, non-power-of-two z, the BIG (chunked) squeeze path
SMALL = [
    (50001, 1000.0, 128, 16.0, 3, 128, 0.0, 500.0, 1),
    (40000, 2048.0, 200, 25.0, 7, 256, 256.0, 768.0, 3),
    (30011, 25600.0, 512, 64.0, 4, 512, 0.0, 12800.0, 8),
    (70000, 25600.0, 1024, 128.0, 8, 1024, 0.0, 2000.0, 2),
    (60000, 51200.0, 2048, 256.0, 16, 2048, 0.0, 4000.0, 4),
    (40960, 1024.0, 257, 32.0, 1, 4096, 0.0, 512.0, 1),
    (50000, 51200.0, 4096, 512.0, 32, 4096, 0.0, 6400.0, 2),
    (20000, 1024.0, 301, 40.0, 10, 512, 100.0, 400.0, 2),
    (30000, 1000.0, 256, 30.0, 6, 256, 0.0, 500.0, 5),
    # N_f = 8192: the paper's §5.1 shape (fs 44.1 kHz, L = 5745, H_t = 1149, band 1282..1765 df, z = 8;
    # P:L427) on a short record, and a full-band L < N_f case
    (60000, 44100.0, 5745, 882.0, 1149, 8192, 1282 * 44100.0 / 8192, 1765 * 44100.0 / 8192, 8),
    (30000, 8192.0, 4001, 500.0, 64, 8192, 0.0, 4096.0, 1),
]


def _sig(N, fs, seed):
    t = np.arange(N) / fs
    rng = np.random.default_rng(seed)
    x = np.zeros(N)
    for f in rng.uniform(0.02, 0.4, size=4) * fs:
        x += rng.uniform(0.3, 1.0) * np.cos(2 * np.pi * f * t + rng.uniform(0, 6.28))
    x += 0.5 * np.cos(2 * np.pi * (0.1 * fs * t + 0.02 * fs * t * t / t[-1]))
    x += 0.1 * rng.standard_normal(N)
    return x.astype(np.float32)


def _case(spec, seed=0):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _sig(N, fs, seed + N)
    g, gd, c = O.gaussian_window(L, sigma)
    return x, g, gd, c


@pytest.mark.parametrize("spec", SMALL, ids=[f"nf{s[5]}_h{s[4]}_z{s[8]}_N{s[0]}" for s in SMALL])
def test_stft_parity(P, spec):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    S, Sd = plan.stft(torch.from_numpy(x).to(DEV))
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    Sdo = O.stft(x.astype(np.float64), gd, c, hop, nfft)
    assert rel(S.cpu().numpy(), So) <= 1e-5
    assert rel(Sd.cpu().numpy(), Sdo) <= 1e-5


@pytest.mark.parametrize("spec", SMALL, ids=[f"nf{s[5]}_h{s[4]}_z{s[8]}_N{s[0]}" for s in SMALL])
def test_forward_parity_and_flips(P, spec):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    gamma = 1e-6 * float(np.abs(So).max())
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd).cpu().numpy()
    lg = plan.targets(xd).cpu().numpy()
    To, S, Sd, lo = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma, debug=True)
    _, _, fhat = O.if_estimate(S, Sd, nfft, gamma)
    st = flip_stats(lg, lo, S, fhat, plan.layout["k1"], z, gamma)
    assert T.shape == To.shape
    assert_flips(st)
    e = rel(T, To)
    assert e <= 1e-3, (e, st)


@pytest.mark.parametrize("spec", SMALL, ids=[f"nf{s[5]}_h{s[4]}_z{s[8]}_N{s[0]}" for s in SMALL])
def test_inverse_parity(P, spec):
    """Forward + inverse end to end vs the oracle's inverse (Eq. 25-26) of the oracle's T."""
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    y = plan.inverse(T).cpu().numpy()
    k1 = plan.layout["k1"]
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 0.0)
    ye = O.sst_inverse(To, g, c, hop, nfft, z, k1, N)
    assert rel(y, ye) <= 1e-4


def test_discrete_constant_flag(P):
    N, fs, L, sigma, hop, nfft, f1, f2, z = SMALL[3]
    x, g, gd, c = _case(SMALL[3])
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, flags=P.SST_DISCRETE_CONSTANT, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    y = plan.inverse(T).cpu().numpy()
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 0.0)
    yo = O.sst_inverse(To, g, c, hop, nfft, z, 0, N, constant="discrete")
    assert rel(y, yo) <= 1e-4


def test_frame_ranges_and_offsets_bitwise(P):
    """Forward over sub-ranges with an offset x slice reproduces rows of the full forward
    exactly (frames are independent, P12), including both record edges."""
    spec = SMALL[4]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
    xd = torch.from_numpy(x).to(DEV)
    full = plan.forward(xd)
    F = plan.frames
    for fb, fe in [(0, 7), (5, 130), (F - 9, F), (1000, 1001)]:
        lo = max(0, fb * hop - c)
        hi = min(N, (fe - 1) * hop - c + L)
        xs = xd[lo:hi].contiguous()
        part = plan.forward(xs, fb, fe, x_off=lo)
        assert torch.equal(part, full[fb:fe])


def test_ldT_padding(P):
    spec = SMALL[3]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
    xd = torch.from_numpy(x).to(DEV)
    full = plan.forward(xd)
    out = torch.full((plan.frames, plan.bins + 7), 123.0 + 0j, dtype=torch.complex64, device=DEV)
    plan.forward(xd, out=out)
    assert torch.equal(out[:, :plan.bins], full)
    assert torch.all(out[:, plan.bins:] == 123.0)
    y1 = plan.inverse(full)
    y2 = plan.inverse(out)
    assert torch.allclose(y1, y2, rtol=0, atol=1e-6 * float(y1.abs().max()))


def test_absmax_and_relative_gamma(P):
    spec = SMALL[1]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.05, flags=P.SST_GAMMA_RELATIVE, device=0)
    xd = torch.from_numpy(x).to(DEV)
    m = float(plan.absmax(xd))
    assert m == pytest.approx(float(np.abs(So).max()), rel=1e-5)
    T = plan.forward(xd).cpu().numpy()
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 0.05 * float(np.abs(So).max()))
    assert rel(T, To) <= 1e-3
    # externally supplied max (as all-reduced over ranks); the oracle's threshold comes from its own
    # max, never from the GPU's
    ref = float(np.abs(So).max())
    ext = torch.tensor(2.0 * ref, dtype=torch.float32, device=DEV)
    plan.set_absmax(ext)
    T2 = plan.forward(xd).cpu().numpy()
    To2 = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 0.1 * ref)
    assert rel(T2, To2) <= 1e-3


def test_truncate_flag(P):
    spec = SMALL[7]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-5, flags=P.SST_SOURCE_TRUNCATE, device=0)
    T = plan.forward(torch.from_numpy(x).to(DEV)).cpu().numpy()
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 1e-5, truncate=True)
    assert rel(T, To) <= 1e-3


def test_sharded_inverse_equals_whole(P):
    """Frame ranges accumulated into overlapping y spans, seams added, then finalised, equal the
    single-call inverse (P13 on one device; ranks emulated sequentially, no cross-waiting)."""
    spec = SMALL[4]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    whole = plan.inverse(T)
    F = plan.frames
    cuts = [0, F // 3, (2 * F) // 3 + 5, F]
    y = torch.zeros(N, dtype=torch.float32, device=DEV)
    for fb, fe in zip(cuts[:-1], cuts[1:]):
        lo = max(0, fb * hop - c)
        hi = min(N, (fe - 1) * hop - c + L)
        part = torch.zeros(hi - lo, dtype=torch.float32, device=DEV)
        plan.inverse_accumulate(T[fb:fe].contiguous(), fb, fe, part, y_off=lo)
        y[lo:hi] += part
    plan.inverse_finalize(y, 0)
    assert rel(y.cpu().numpy(), whole.cpu().numpy()) <= 1e-6


def test_c1_full(P):
    """configs[0] (C1) end to end at full size: STFT, T, flips, reconstruction."""
    cfg = get_config("C1")
    x = signal("C1")
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    gamma = config_gamma(cfg, x)
    plan = make_plan(P, cfg, gamma)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    y = plan.inverse(T)
    lg = plan.targets(xd).cpu().numpy()
    To, S, Sd, lo = O.sst_forward(x.astype(np.float64), g, gd, c, cfg.hop, cfg.nfft, cfg.fs, cfg.f1, cfg.f2,
                                  cfg.zoom, gamma, debug=True)
    _, _, fhat = O.if_estimate(S, Sd, cfg.nfft, gamma)
    st = flip_stats(lg, lo, S, fhat, cfg.k1, cfg.zoom, gamma)
    Tg = T.cpu().numpy()
    assert rel(Tg, To) <= 1e-3, st
    assert_flips(st)
    yo = O.sst_inverse(To, g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N)
    assert rel(y.cpu().numpy(), yo) <= 1e-4


def _windows(F, n, size, seed, seams=0):
    """n frame windows of ``size`` frames: both record edges, the windows centred on the rank
    boundaries F r / P of a P = ``seams`` sharding, the rest at seeded random positions."""
    rng = np.random.default_rng(seed)
    fixed = [0, F - size] + ([F * r // seams - size // 2 for r in range(1, seams)] if seams else [])
    starts = set(fixed)
    while len(starts) < n:
        starts.add(int(rng.integers(0, F - size)))
    return [(int(s), int(s) + size) for s in sorted(starts)]


# windows per config: SURVEY §8(d) asks for 64 windows of 1024 frames on C4-C5 (every P = 8 rank seam
# included); C2 / C3 get the same treatment at their (whole-record) launch
WINDOWS = {"C2": (16, 1024), "C3": (64, 1024), "C4": (64, 1024), "C5": (64, 1024)}


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_config_sampled_frames(P, name):
    """Full-size configs in the bench's launch configuration, compared on sampled frame windows
    (both record edges and the P = 8 rank seams included) that the oracle computes one by one."""
    cfg = get_config(name)
    x = signal(name)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    gamma = config_gamma(cfg, x)
    plan = make_plan(P, cfg, gamma)
    xd = torch.from_numpy(x).to(DEV)
    F = cfg.frames
    n, size = WINDOWS[name]
    wins = _windows(F, n, size, 5, seams=8)
    if name in ("C4", "C5"):
        Tw = None                          # T of C4 / C5 is 64 / 256 GiB: forward the windows only
    else:
        T = plan.forward(xd)
        Tw = {w: T[w[0]:w[1]].cpu().numpy() for w in wins}
        del T
    x64 = x.astype(np.float64)
    worst = 0.0
    for w in wins:
        Tg = plan.forward(xd, *w).cpu().numpy() if Tw is None else Tw[w]
        fr = np.arange(*w)
        To, S, Sd, lo = O.sst_forward(x64, g, gd, c, cfg.hop, cfg.nfft, cfg.fs, cfg.f1, cfg.f2, cfg.zoom,
                                      gamma, frames=fr, debug=True)
        e = rel(Tg, To)
        worst = max(worst, e)
        assert e <= 1e-3, (name, w, e)
        lg = plan.targets(xd, *w).cpu().numpy()
        _, _, fhat = O.if_estimate(S, Sd, cfg.nfft, gamma)
        st = flip_stats(lg, lo, S, fhat, cfg.k1, cfg.zoom, gamma)
        assert_flips(st, (name, w))
    print(name, "windows", len(wins), "worst T rel L2", worst)


@pytest.mark.parametrize("name", ["C3"])
def test_config_inverse_sampled(P, name):
    """Full-size forward + inverse (bench launch config) vs the oracle's forward + inverse of the
    frames covering sampled output windows."""
    cfg = get_config(name)
    x = signal(name)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    plan = make_plan(P, cfg, config_gamma(cfg, x))
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    y = plan.inverse(T).cpu().numpy()
    rng = np.random.default_rng(3)
    for n0 in [0, cfg.N - 4000] + list(rng.integers(0, cfg.N - 4000, size=3)):
        n0 = int(n0)
        n1 = n0 + 4000
        fb = max(0, (n0 + c - cfg.L) // cfg.hop)
        fe = min(cfg.frames, (n1 - 1 + c) // cfg.hop + 1)
        To = O.sst_forward(x.astype(np.float64), g, gd, c, cfg.hop, cfg.nfft, cfg.fs, cfg.f1, cfg.f2, cfg.zoom,
                           config_gamma(cfg, x), frames=np.arange(fb, fe))
        yo = O.sst_inverse(To, g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N, frame_begin=fb, n0=n0, n1=n1)
        assert rel(y[n0:n1], yo) <= 1e-4, n0


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_config_inverse_windows(P, name):
    """C4 / C5 at full size (T of the whole record is 64 / 256 GiB): the forward of the frames
    covering sampled output windows, sst_inverse_accumulate of those frames into a window buffer and
    sst_inverse_finalize, against the oracle's forward + inverse of those frames; both record edges."""
    cfg = get_config(name)
    x = signal(name)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    plan = make_plan(P, cfg, config_gamma(cfg, x))
    xd = torch.from_numpy(x).to(DEV)
    rng = np.random.default_rng(4)
    W = 8 * cfg.L
    for n0 in [0, cfg.N - W] + list(rng.integers(0, cfg.N - W, size=2)):
        n0 = int(n0)
        n1 = n0 + W
        fb = max(0, (n0 + c - cfg.L) // cfg.hop)
        fe = min(cfg.frames, (n1 - 1 + c) // cfg.hop + 1)
        T = plan.forward(xd, fb, fe)
        lo = max(0, fb * cfg.hop - c)
        hi = min(cfg.N, (fe - 1) * cfg.hop - c + cfg.L)
        y = torch.zeros(hi - lo, dtype=torch.float32, device=DEV)
        plan.inverse_accumulate(T, fb, fe, y, y_off=lo)
        plan.inverse_finalize(y[n0 - lo:n1 - lo], y_off=n0)
        To = O.sst_forward(x.astype(np.float64), g, gd, c, cfg.hop, cfg.nfft, cfg.fs, cfg.f1, cfg.f2, cfg.zoom,
                           config_gamma(cfg, x), frames=np.arange(fb, fe))
        yo = O.sst_inverse(To, g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, cfg.N, frame_begin=fb, n0=n0, n1=n1)
        assert rel(y[n0 - lo:n1 - lo].cpu().numpy(), yo) <= 1e-4, (name, n0)


EXTREME = [
    # (N, fs, L, sigma, hop, nfft, f1, f2, z): smallest N_f with z = 64 (z N_f = 8192), a short
    # window far below N_f, hop = L (no overlap), hop = 1 with a narrow band at the top edge
    (3000, 1024.0, 96, 12.0, 5, 128, 0.0, 512.0, 64),
    (20000, 4096.0, 9, 1.5, 2, 512, 0.0, 2048.0, 2),
    (16256, 2048.0, 256, 32.0, 256, 256, 256.0, 768.0, 3),
    (6000, 1000.0, 128, 16.0, 1, 128, 437.5, 500.0, 7),
]


@pytest.mark.parametrize("spec", EXTREME, ids=[f"nf{s[5]}_L{s[2]}_h{s[4]}_z{s[8]}" for s in EXTREME])
def test_extreme_parameters(P, spec):
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-5, device=0)
    xd = torch.from_numpy(x).to(DEV)
    S, Sd = plan.stft(xd)
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    assert rel(S.cpu().numpy(), So) <= 1e-5
    T = plan.forward(xd)
    To, So64, Sdo64, lo = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 1e-5, debug=True)
    lg = plan.targets(xd).cpu().numpy()
    _, _, fhat = O.if_estimate(So64, Sdo64, nfft, 1e-5)
    st = flip_stats(lg, lo, So64, fhat, plan.layout["k1"], z, 1e-5)
    e = rel(T.cpu().numpy(), To)
    assert_flips(st)
    assert e <= 1e-3, (e, st)
    y = plan.inverse(T).cpu().numpy()
    yo = O.sst_inverse(To, g, c, hop, nfft, z, plan.layout["k1"], N)
    assert rel(y, yo) <= 1e-4


def test_error_codes(P):
    spec = SMALL[3]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=0.0, device=0)
    xd = torch.from_numpy(x).to(DEV)
    with pytest.raises(P.SSTError) as e:
        plan.forward(xd, 5, 5)
    assert e.value.status == P.SST_E_INVALID_ARGUMENT
    with pytest.raises(P.SSTError):
        plan.forward(xd, 0, plan.frames + 1)
    with pytest.raises(P.SSTError):
        plan.forward(xd[100:], 0, 10, x_off=100)       # slice does not cover frame 0
    bad = torch.empty((plan.frames, plan.bins - 1), dtype=torch.complex64, device=DEV)
    with pytest.raises(P.SSTError):
        plan.forward(xd, out=bad)
    with pytest.raises(TypeError):
        plan.forward(xd.double())


@pytest.mark.parametrize("kind", ["zeros", "dc", "nyquist"])
def test_degenerate_signals(P, kind):
    """Degenerate inputs: an all-zero record (every coefficient masked at gamma = 0: T = 0, x_hat = 0
    exactly), a constant (DC only) and an alternating (fs/2) record, against the oracle."""
    N, fs, L, sigma, hop, nfft, f1, f2, z = (5000, 1000.0, 128, 16.0, 3, 128, 0.0, 500.0, 2)
    if kind == "zeros":
        x = np.zeros(N, np.float32)
    elif kind == "dc":
        x = np.full(N, 0.75, np.float32)
    else:
        x = (0.5 * (-1.0) ** np.arange(N)).astype(np.float32)
    g, gd, c = O.gaussian_window(L, sigma)
    gamma = 0.0 if kind == "zeros" else 1e-6
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = plan.forward(xd)
    y = plan.inverse(T).cpu().numpy()
    Tn = T.cpu().numpy()
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, gamma)
    if kind == "zeros":
        assert not np.any(Tn) and not np.any(y)
        return
    assert rel(Tn, To) <= 1e-3
    yo = O.sst_inverse(To, g, c, hop, nfft, z, 0, N)
    assert rel(y, yo) <= 1e-4


def test_cuda_graph_capture_replays_bitwise(P):
    """The forward + inverse launch sequence is stream-ordered with no host synchronisation, so it
    can be captured into a CUDA graph and replayed (launch-bound small configs); the replay equals
    the eager result bit for bit (the squeeze sums are exact, the OLA order fixed)."""
    spec = SMALL[4]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T = torch.empty((plan.frames, plan.bins), dtype=torch.complex64, device=DEV)
    y = torch.empty(N, dtype=torch.float32, device=DEV)
    plan.forward(xd, out=T)
    plan.inverse(T, out=y)
    T0, y0 = T.clone(), y.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.forward(xd, out=T)
        plan.inverse(T, out=y)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        plan.forward(xd, out=T)
        plan.inverse(T, out=y)
    T.zero_()
    y.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(T, T0) and torch.equal(y, y0)


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_pipelined_host_roundtrip(P, chunks):
    """pipeline.RoundTrip (chunked H2D / forward / inverse_accumulate / finalize / D2H on three
    streams) equals the device-resident single calls: T bitwise, x_hat to fp32 re-association."""
    from paper_2003_07065_b200.pipeline import RoundTrip
    spec = SMALL[4]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
    xd = torch.from_numpy(x).to(DEV)
    T_ref = plan.forward(xd)
    y_ref = plan.inverse(T_ref).cpu().numpy()
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.zeros(N, dtype=torch.float32).pin_memory()
    T = torch.empty_like(T_ref)
    rt = RoundTrip(plan, chunks=chunks)
    for _ in range(2):                    # reuse of buffers and streams
        rt.run(xh, yh, T)
        torch.cuda.synchronize()
        assert torch.equal(T, T_ref)
        assert rel(yh.numpy(), y_ref) <= 1e-6
    y_run = yh.clone()
    # the same round trip captured once as a CUDA graph and replayed: identical results
    graph = rt.capture(xh, yh, T)
    for _ in range(2):
        yh.zero_()
        T.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(T, T_ref)
        assert torch.equal(yh, y_run)


def test_pipelined_roundtrip_relative_gamma(P):
    """RoundTrip under SST_GAMMA_RELATIVE: refused until the record's max|S| is supplied (chunks would
    otherwise threshold against their own maxima); with plan.set_absmax(plan.absmax(x)) it equals the
    single-call forward + inverse (T bitwise, x_hat to re-association)."""
    from paper_2003_07065_b200.pipeline import RoundTrip
    spec = SMALL[4]
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x, g, gd, c = _case(spec)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-3, flags=P.SST_GAMMA_RELATIVE, device=0)
    xd = torch.from_numpy(x).to(DEV)
    with pytest.raises(ValueError):
        RoundTrip(plan, chunks=4)
    amax = plan.absmax(xd)
    plan.set_absmax(amax)
    T_ref = plan.forward(xd)
    y_ref = plan.inverse(T_ref).cpu().numpy()
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.zeros(N, dtype=torch.float32).pin_memory()
    T = torch.empty_like(T_ref)
    RoundTrip(plan, chunks=4).run(xh, yh, T)
    torch.cuda.synchronize()
    assert torch.equal(T, T_ref)
    assert rel(yh.numpy(), y_ref) <= 1e-6
    # and the threshold really is the record's: the oracle at 1e-3 * its own max|S|
    So = O.stft(x.astype(np.float64), g, c, hop, nfft)
    To = O.sst_forward(x.astype(np.float64), g, gd, c, hop, nfft, fs, f1, f2, z, 1e-3 * float(np.abs(So).max()))
    assert rel(T.cpu().numpy(), To) <= 1e-3
