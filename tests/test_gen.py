"""Input generators (gen/): determinism, block addressability, config geometry.  CPU only."""

import numpy as np
import pytest

from gen import CONFIGS, generate, get_config
from gen.signals import BLOCK, c5_laws


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_config_geometry(name):
    """Band edges on the coarse grid (R9), frame count, B as in SURVEY §8(a)."""
    cfg = get_config(name)
    assert abs(cfg.f1 / cfg.df - cfg.k1) < 1e-9 and abs(cfg.f2 / cfg.df - cfg.k2) < 1e-9
    assert 0 <= cfg.k1 < cfg.k2 <= cfg.nfft // 2
    assert cfg.L <= cfg.nfft <= cfg.N and cfg.hop <= cfg.L
    expect = {"C1": (4096, 2048), "C2": (131072, 160), "C3": (1048576, 640),
              "C4": (8388608, 1024), "C5": (16777216, 2048)}[name]
    assert (cfg.frames, cfg.bins) == expect


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_range_generation_is_consistent(name):
    """Any [start, stop) equals the same slice of a larger range (block-addressable, so ranks and
    the oracle see identical samples)."""
    cfg = get_config(name)
    n = min(cfg.N, 3 * BLOCK)
    big = generate(name, 0, n)
    for a, b in [(0, 100), (BLOCK - 50, BLOCK + 70), (n - 333, n), (1234, 1234)]:
        if b > n:
            continue
        assert np.array_equal(generate(name, a, b), big[a:b])
    again = generate(name, 0, n)
    assert np.array_equal(big, again)
    assert big.dtype == np.float32 and np.all(np.isfinite(big))


def test_c4_range_far_into_record():
    cfg = get_config("C4")
    a = cfg.N - 5000
    x = generate("C4", a, cfg.N)
    assert np.array_equal(x[100:300], generate("C4", a + 100, a + 300))


def test_c5_crossing_free():
    c, a, b, _ = c5_laws(5)
    sf = 25600.0 / (2 * np.pi * 64.0)
    for i in range(8):
        for j in range(i + 1, 8):
            assert abs(c[i] - c[j]) >= a[i] + a[j] + 8 * sf


def test_snr_roughly_as_specified():
    """Noise power relative to the nominal tonal power: C2 10 dB, C5 20 dB."""
    from gen.signals import clean_components
    for name, snr in (("C2", 10.0), ("C5", 20.0)):
        n = 2 * BLOCK
        x = generate(name, 0, n, dtype=np.float64)
        clean = sum(clean_components(name, 0, n).values())
        noise = x - clean
        nominal = {"C2": (1 + .36 + .16 + .04) / 2, "C5": 4.0}[name]
        got = 10 * np.log10(nominal / np.mean(noise ** 2))
        assert abs(got - snr) < 0.2
