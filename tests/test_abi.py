"""The C-ABI library: loads, exports every symbol include/sst.h declares, host-only entry points
(window, validation, layout) behave as documented.  No GPU needed (no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from gen import CONFIGS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import paper_2003_07065_b200 as P
    return P


def _declared():
    src = open(os.path.join(ROOT, "include", "sst.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sst_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(P):
    from paper_2003_07065_b200 import _lib
    names = _declared()
    assert len(names) >= 17
    for n in names:
        assert hasattr(_lib.lib, n), n
        assert n in _lib.SIGNATURES, n
    assert _lib.lib.sst_abi_version() == _lib.ABI_VERSION == 4


def test_status_strings(P):
    from paper_2003_07065_b200 import _lib
    for s, name in [(0, "SST_OK"), (1, "SST_E_INVALID_ARGUMENT"), (2, "SST_E_COVERAGE"), (3, "SST_E_UNSUPPORTED"),
                    (4, "SST_E_CUDA"), (5, "SST_E_OUT_OF_MEMORY"), (6, "SST_E_INTERNAL")]:
        assert _lib.lib.sst_status_str(s).decode() == name


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_window_matches_oracle(P, name):
    """sst_gaussian_window (C++) and the oracle's window (numpy) are independent implementations of
    P:L55 / P:L110; they agree to rounding."""
    cfg = CONFIGS[name]
    g, gd = P.gaussian_window(cfg.L, cfg.sigma)
    go, gdo, c = O.gaussian_window(cfg.L, cfg.sigma)
    assert np.allclose(g, go, rtol=1e-14, atol=0)
    assert np.allclose(gd, gdo, rtol=1e-13, atol=1e-300)


def test_window_errors(P):
    from paper_2003_07065_b200 import _lib
    g = np.zeros(4)
    dp = g.ctypes.data_as(_lib._dp)
    assert _lib.lib.sst_gaussian_window(0, 1.0, -1, dp, dp) == P.SST_E_INVALID_ARGUMENT
    assert _lib.lib.sst_gaussian_window(4, -1.0, -1, dp, dp) == P.SST_E_INVALID_ARGUMENT
    assert _lib.lib.sst_gaussian_window(4, 1.0, 4, dp, dp) == P.SST_E_INVALID_ARGUMENT
    assert _lib.lib.sst_gaussian_window(4, 1.0, -1, None, dp) == P.SST_E_INVALID_ARGUMENT


BASE = dict(n=4096, fs=1024.0, win_len=257, sigma=32.0, hop=1, nfft=4096, f1=0.0, f2=512.0, zoom=1)


@pytest.mark.parametrize("change,status", [
    ({}, 0),
    ({"hop": 0}, 1),
    ({"zoom": 0}, 1),
    ({"gamma": -1.0}, 1),
    ({"gamma": float("nan")}, 1),
    ({"nfft": 128}, 1),                       # L > N_f
    ({"n": 2048}, 1),                         # N_f > N
    ({"f1": 100.0, "f2": 50.0}, 1),           # f2 <= f1
    ({"f2": 600.0}, 1),                       # f2 > fs/2
    ({"f1": 0.1}, 1),                         # off-grid (R9)
    ({"fs": 0.0}, 1),
    ({"flags": 64}, 1),                       # unknown flag
    ({"flags": 2 | 16}, 0),                   # SST_SOURCE_TRUNCATE | SST_FILTER_BANK
    ({"nfft": 3000}, 3),                      # not a power of two
    ({"nfft": 131072, "n": 131072}, 3),       # outside this build's N_f range (<= 65536)
    ({"nfft": 32768, "n": 573440, "fs": 10240.0, "win_len": 8193, "sigma": 1024.0, "hop": 667,
      "f1": 1200.0, "f2": 1400.0}, 0),        # §5.2 shape: multi-pass path
    ({"zoom": 65}, 3),
    ({"flags": 4}, 0),                        # DETERMINISTIC accepted (always reproducible)
    ({"hop": 258}, 2),                        # H_t > L -> gaps (R20)
    ({"win_len": 4096, "sigma": 512.0, "hop": 4096, "n": 4097 * 4096}, 3),   # tiles beyond 227 KB smem
    ({"nfft": 8192, "n": 8192, "win_len": 5745, "sigma": 882.0, "hop": 1149}, 0),   # §5.1 shape
    ({"win_len": 64, "sigma": 8.0, "hop": 64, "nfft": 4096, "n": 4136}, 2),   # tail uncovered
])
def test_validation_codes(P, change, status):
    kw = dict(BASE)
    kw.update(change)
    assert P.validate(**kw) == status


def test_coverage_matches_oracle_diagonal(P):
    """SST_E_COVERAGE exactly when the oracle's frame diagonal has a zero on [0, N) (R20)."""
    for (N, L, hop) in [(600, 32, 32), (592, 32, 32), (1000, 40, 30), (1000, 40, 21), (999, 64, 40), (1001, 64, 33)]:
        g, gd, c = O.gaussian_window(L, L / 6.0)
        d = O.frame_diagonal(g, c, hop, N)
        st = P.validate(n=N, fs=1000.0, win_len=L, sigma=L / 6.0, hop=hop, nfft=128, f1=0.0, f2=500.0,
                        g=g, gd=gd)
        assert (st == P.SST_E_COVERAGE) == bool(np.any(d <= 0)), (N, L, hop, st)


def test_layout_values(P):
    lay = P.layout(**BASE)
    assert (lay["frames"], lay["bins"], lay["k1"], lay["k2"], lay["src_bins"]) == (4096, 2048, 0, 2048, 2049)
    assert lay["alpha"] == pytest.approx(32.0 * np.sqrt(2.0))
    lay = P.layout(n=1 << 24, fs=51200.0, win_len=2048, sigma=256.0, hop=16, nfft=2048, f1=0.0, f2=4000.0, zoom=4)
    assert (lay["frames"], lay["bins"], lay["k2"]) == (1048576, 640, 160)
    assert lay["dfz_hz"] == pytest.approx(6.25)
    # Eq. 38 bound with sigma in seconds = sigma_samples / fs (golden: P:L359 'H_f < 64')
    lay = P.layout(n=8192, fs=1024.0, win_len=187, sigma=0.03 * 1024, hop=20, nfft=1024, f1=0.0, f2=512.0)
    assert int(np.ceil(lay["hf_bound"])) == 64


def test_eq37_eq46_warnings(P):
    """Eq. 35/37/46 limits in the layout (host only) and the warning bits, pinned to the paper's
    printed values for its simulation (sigma = 0.03 s, N = 8192, fs = 1024): sigma_f = 5.31 Hz
    (P:L335), H_f < 64 (Eq. 38) and H_f < 60 (Eq. 46)."""
    import json
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_values.json")))
    base = dict(n=8192, fs=1024.0, win_len=187, sigma=0.03 * 1024, hop=20, f1=0.0, f2=512.0)
    lay = P.layout(nfft=1024, **base)                         # H_f = 8: inside both intervals
    assert lay["sigma_f_hz"] == pytest.approx(5.305, abs=5e-3)
    assert int(np.ceil(lay["hf_bound"])) == gold["hf_bound_eq38"]["value"] == 64
    assert int(np.round(lay["hf_bound46"])) == gold["hf_bound_eq46"]["value"] == 60
    assert lay["df_eq37_hz"] == pytest.approx(1.5 * lay["sigma_f_hz"])
    assert lay["df_eq46_hz"] == pytest.approx(np.sqrt(2.0) * lay["sigma_f_hz"])
    assert lay["warnings"] == 0
    # H_f = 64 = N / N_f with N_f = 128: df = 8 Hz >= 1.5 sigma_f = 7.96 Hz and >= sqrt 2 sigma_f
    lay = P.layout(nfft=256, **dict(base, win_len=187))        # H_f = 32: still fine
    assert lay["warnings"] == 0
    lay = P.layout(nfft=128, **dict(base, win_len=127, hop=20))
    assert lay["warnings"] == P.SST_WARN_EQ37 | P.SST_WARN_EQ46
    # between the two limits: df in [sqrt 2 sigma_f, 1.5 sigma_f) -> only the Eq. 46 bit
    sig = 1024.0 / (2 * np.pi * 8.0 / 1.45)                      # sigma_f = 8 / 1.45 Hz with df = 8 Hz
    lay = P.layout(n=8192, fs=1024.0, win_len=127, sigma=sig, hop=20, nfft=128, f1=0.0, f2=512.0)
    assert lay["warnings"] == P.SST_WARN_EQ46


def test_istft_shared_memory_checked_by_validate(P):
    """A window / hop whose z = 1 inverse (run by sst_istft) needs more shared memory than the plan's
    z: rejected by validation (SST_E_UNSUPPORTED), not at launch."""
    assert P.validate(n=1 << 20, fs=1000.0, win_len=4096, sigma=512.0, hop=2048, nfft=4096, f1=0.0, f2=500.0,
                      zoom=2) == P.SST_E_UNSUPPORTED


def test_plan_create_without_gpu_fails_cleanly(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2003_07065_b200 import _lib
    p, keep = P.make_params(**BASE)
    h = ctypes.c_void_p()
    st = _lib.lib.sst_plan_create(ctypes.byref(p), 0, ctypes.byref(h))
    assert st in (P.SST_E_CUDA, P.SST_E_INVALID_ARGUMENT)
    assert not h.value
    with pytest.raises(RuntimeError):
        P.Plan(**BASE)
