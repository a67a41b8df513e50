"""Diagnostic (GPU box): where do target flips far from a rounding boundary come from?

Compares, on the C1-like parity case, the r (reassignment frequency, Eq. 36) error of
  (a) our sst_stft spectra (fp32 packed FFT),
  (b) cuFFT complex64 of the separately windowed frames (torch.fft; yardstick only),
  (c) our kernel's fp32 target arithmetic (sst_targets),
against the fp64 oracle, for coefficients with |S| >= 1e-2 max.
    python tests/diag_flip.py [frames]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))   # repo root (tests/ -> ..)
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2003_07065_b200 as P  # noqa: E402
from tests.test_gpu_parity import _case  # noqa: E402

spec = (40960, 1024.0, 257, 32.0, 1, 4096, 0.0, 512.0, 1)
if len(sys.argv) > 2:
    spec = tuple(type(v)(a) for v, a in zip(spec, sys.argv[2].split(",")))
N, fs, L, sigma, hop, nfft, f1, f2, z = spec
nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
x, g, gd, c = _case(spec)
frames = np.arange(nfr)
So = O.stft(x.astype(np.float64), g, c, hop, nfft)
amax = np.abs(So).max()
gamma = 1e-6 * amax
So = So[:nfr]
Sdo = O.stft(x.astype(np.float64), gd, c, hop, nfft, frames=frames)
plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=gamma, device=0)
xd = torch.from_numpy(x).cuda()
S, Sd = plan.stft(xd, 0, nfr)
S = S.cpu().numpy().astype(np.complex128)
Sd = Sd.cpu().numpy().astype(np.complex128)
lg = plan.targets(xd, 0, nfr).cpu().numpy()

# cuFFT yardstick: frames placed circularly (tau mod N_f), complex64
idx = frames[:, None] * hop - c + np.arange(L)[None, :]
u = np.where((idx >= 0) & (idx < N), x[np.clip(idx, 0, N - 1)], 0).astype(np.float32)
buf = np.zeros((nfr, nfft), np.float32)
bufd = np.zeros((nfr, nfft), np.float32)
tau = np.arange(L) - c
buf[:, tau % nfft] = u * g.astype(np.float32)
bufd[:, tau % nfft] = u * gd.astype(np.float32)
K = nfft // 2 + 1
Sc = torch.fft.fft(torch.from_numpy(buf).cuda().to(torch.complex64), dim=1)[:, :K].cpu().numpy().astype(np.complex128)
Sdc = torch.fft.fft(torch.from_numpy(bufd).cuda().to(torch.complex64), dim=1)[:, :K].cpu().numpy().astype(np.complex128)


def rF(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def rf(S_, Sd_):
    return -np.imag(Sd_ / S_) * nfft / (2 * np.pi)


print(f"S rel: ours {rF(S, So):.2e} cufft {rF(Sc, So):.2e};  S' rel: ours {rF(Sd, Sdo):.2e} cufft {rF(Sdc, Sdo):.2e}")
big = np.abs(So) >= 1e-2 * amax
ro = rf(So, Sdo)
for name, (a, b) in {"ours": (S, Sd), "cufft": (Sc, Sdc)}.items():
    e = np.abs(rf(a, b) - ro)[big]
    print(f"{name:6s} |r err| on |S|>=1e-2max: max {e.max():.2e} p99.99 {np.quantile(e, 0.9999):.2e} "
          f"p99 {np.quantile(e, 0.99):.2e} median {np.median(e):.2e}")
    # where is the worst one
    ii = np.argmax(np.abs(rf(a, b) - ro) * big)
    m, k = np.unravel_index(ii, ro.shape)
    print(f"       worst at m={m} k={k} |S|/max={abs(So[m, k]) / amax:.3e} r={ro[m, k]:.2f}")
mask, _, fhat = O.if_estimate(So, Sdo, nfft, gamma)
k1 = plan.layout["k1"]
lo = O.targets(fhat, mask, k1, plan.bins, z)
flips = (lg != lo) & (lo != -1)
bigf = flips & big
pos = z * (fhat - k1) + 0.5
dist = np.abs(pos - np.round(pos)) / z
print(f"kernel flips {flips.sum()} of {(lo != -1).sum()}; big flips {bigf.sum()}, their boundary distance max "
      f"{dist[bigf].max() if bigf.any() else 0:.2e}")
for m, k in zip(*np.nonzero(bigf)):
    print(f"   m={m} k={k} |S|/max={abs(So[m, k]) / amax:.3e} r={ro[m, k]:.3f} dist={dist[m, k]:.2e} "
          f"r_ours={rf(S[m, k], Sd[m, k]):.5f} r_cufft={rf(Sc[m, k], Sdc[m, k]):.5f} r_orc={ro[m, k]:.5f}")
