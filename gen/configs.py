"""Workload definitions C1-C5 (BASELINE.json ``configs``).

Pure parameter records.  Band edges are in Hz and lie exactly on the coarse grid
fs/N_f for every config (checked in tests/test_gen.py).
"""

from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class Config:
    name: str
    N: int            # samples
    fs: float         # Hz
    L: int            # window length (taps)
    sigma: float      # Gaussian sigma in samples
    hop: int          # H_t
    nfft: int         # N_f
    f1: float         # band [f1, f2) in Hz
    f2: float
    zoom: int         # subdivision z
    seed: int
    inverse: bool     # does BASELINE.json ask for the inverse on this config
    gamma_rel: float = 1e-6   # gamma = gamma_rel * (bound or max of |S|), R6
    desc: str = ""

    @property
    def frames(self) -> int:
        return (self.N - 1) // self.hop + 1

    @property
    def df(self) -> float:
        return self.fs / self.nfft

    @property
    def k1(self) -> int:
        return int(round(self.f1 / self.df))

    @property
    def k2(self) -> int:
        return int(round(self.f2 / self.df))

    @property
    def bins(self) -> int:
        return self.zoom * (self.k2 - self.k1)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]: tiny standard SST, forward + inverse
    "C1": Config("C1", N=4096, fs=1024.0, L=257, sigma=32.0, hop=1, nfft=4096,
                 f1=0.0, f2=512.0, zoom=1, seed=1, inverse=True,
                 desc="100 Hz tone + 200->400 Hz chirp (0.5) + white noise (0.1)"),
    # configs[1]: spindle-like
    "C2": Config("C2", N=1 << 20, fs=25600.0, L=1024, sigma=128.0, hop=8, nfft=1024,
                 f1=0.0, f2=2000.0, zoom=2, seed=2, inverse=False,
                 desc="spindle harmonics 1-4 of 150+10 sin(pi t) Hz, 5% AM at 2 Hz, SNR 10 dB"),
    # configs[2]: aero-engine run-up
    "C3": Config("C3", N=1 << 24, fs=51200.0, L=2048, sigma=256.0, hop=16, nfft=2048,
                 f1=0.0, f2=4000.0, zoom=4, seed=3, inverse=True,
                 desc="run-up 50->250 Hz, orders 1,2,3,5,8, 1.2 kHz resonance impulses, pink SNR 5 dB"),
    # configs[3]: multi-GPU long record
    "C4": Config("C4", N=1 << 28, fs=51200.0, L=4096, sigma=512.0, hop=32, nfft=4096,
                 f1=0.0, f2=6400.0, zoom=2, seed=4, inverse=False,
                 desc="16 concatenated seeded run-ups, continuous phase"),
    # configs[4]: reconstruction-heavy dense grid
    "C5": Config("C5", N=1 << 26, fs=25600.0, L=512, sigma=64.0, hop=4, nfft=512,
                 f1=0.0, f2=12800.0, zoom=8, seed=5, inverse=True,
                 desc="8 crossing-free FM components, SNR 20 dB"),
}


def get_config(name: str) -> Config:
    try:
        return CONFIGS[name]
    except KeyError:
        raise KeyError(f"unknown config {name!r}; have {sorted(CONFIGS)}") from None
