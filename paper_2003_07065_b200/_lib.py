"""ctypes binding of include/sst.h -- argument marshalling only.

Every transform step runs in ``libsst.so`` (hand-written sm_100a CUDA).  There is no CPU
fallback: importing this module raises if the library is missing, and compute calls need CUDA
tensors on the plan's device.
"""

from __future__ import annotations

import ctypes
import os

ABI_VERSION = 4                  # SST_ABI_VERSION of include/sst.h this binding mirrors
_HERE = os.path.dirname(os.path.abspath(__file__))
# SST_LIB=bounds loads the -DSST_BOUNDS debug build (device-side bounds asserts); SST_LIB_PATH
# overrides the path (dev A/B builds only)
_VARIANT = {"": "libsst.so", "release": "libsst.so", "bounds": "libsst_bounds.so"}[os.environ.get("SST_LIB", "")]
LIB_PATH = os.environ.get("SST_LIB_PATH") or os.path.join(_HERE, _VARIANT)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; g.build()'`. "
        "There is no fallback implementation.")

lib = ctypes.CDLL(LIB_PATH)
if lib.sst_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI version {lib.sst_abi_version()}, this binding needs {ABI_VERSION}: rebuild it")

# ---------------------------------------------------------------- constants (sst.h)
SST_OK = 0
SST_E_INVALID_ARGUMENT = 1
SST_E_COVERAGE = 2
SST_E_UNSUPPORTED = 3
SST_E_CUDA = 4
SST_E_OUT_OF_MEMORY = 5
SST_E_INTERNAL = 6

SST_GAMMA_RELATIVE = 1
SST_SOURCE_TRUNCATE = 2
SST_DETERMINISTIC = 4
SST_DISCRETE_CONSTANT = 8
SST_FILTER_BANK = 16

SST_WARN_EQ37 = 1
SST_WARN_EQ46 = 2

SST_PATH_FUSED = 0
SST_PATH_MULTIPASS = 1
SST_PATH_FILTERBANK = 2
SST_IPATH_RESIDUE = 0
SST_IPATH_NARROWBAND = 1
SST_IPATH_MULTIPASS = 2

_i32, _i64, _u32, _dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)


class sst_params(ctypes.Structure):
    _fields_ = [("n", _i64), ("fs", _dbl), ("win_len", _i32), ("win_center", _i32),
                ("g", _dp), ("gd", _dp), ("sigma", _dbl), ("hop", _i32), ("nfft", _i32),
                ("f1", _dbl), ("f2", _dbl), ("zoom", _i32), ("gamma", _dbl), ("flags", _u32)]


class sst_layout(ctypes.Structure):
    _fields_ = [("n", _i64), ("frames", _i64), ("bins", _i32), ("k1", _i32), ("k2", _i32),
                ("nfft", _i32), ("zoom", _i32), ("hop", _i32), ("center", _i32), ("win_len", _i32),
                ("src_bins", _i32), ("fs", _dbl), ("f0_hz", _dbl), ("df_hz", _dbl), ("dfz_hz", _dbl),
                ("gamma_abs", _dbl), ("alpha", _dbl), ("hf", _dbl), ("hf_bound", _dbl),
                ("sigma_f_hz", _dbl), ("df_eq37_hz", _dbl), ("df_eq46_hz", _dbl), ("hf_bound46", _dbl),
                ("warnings", _u32), ("forward_path", _i32), ("inverse_path", _i32)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = ctypes.POINTER(sst_params)
_L = ctypes.POINTER(sst_layout)

# name -> (restype, argtypes); every symbol declared in include/sst.h
SIGNATURES = {
    "sst_gaussian_window": (_i32, [_i32, _dbl, _i32, _dp, _dp]),
    "sst_params_validate": (_i32, [_P]),
    "sst_params_layout": (_i32, [_P, _L]),
    "sst_status_str": (ctypes.c_char_p, [_i32]),
    "sst_last_error": (ctypes.c_char_p, [_vp]),
    "sst_abi_version": (_i32, []),
    "sst_plan_create": (_i32, [_P, ctypes.c_int, ctypes.POINTER(_vp)]),
    "sst_plan_layout": (_i32, [_vp, _L]),
    "sst_plan_set_gamma": (_i32, [_vp, _dbl]),
    "sst_plan_set_absmax": (_i32, [_vp, _vp]),
    "sst_plan_destroy": (None, [_vp]),
    "sst_plan_counters": (_i32, [_vp, ctypes.POINTER(ctypes.c_uint64)]),
    "sst_forward": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _i64, _vp]),
    "sst_inverse": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "sst_inverse_accumulate": (_i32, [_vp, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp]),
    "sst_inverse_finalize": (_i32, [_vp, _vp, _i64, _i64, _vp]),
    "sst_inverse_finalize_seam": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp]),
    "sst_istft": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "sst_renyi": (_i32, [_vp, _vp, _i64, _i64, _dbl, _vp, _vp]),
    "sst_ridge_emission": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "sst_ridge": (_i32, [_vp, _vp, _i64, _dbl, _i32, _i32, _vp, _vp, _vp]),
    "sst_zone_mask": (_i32, [_vp, _vp, _i64, _i64, _vp, _i32, _i32, _vp]),
    "sst_mode_full": (_i32, [_vp, _vp, _i64, _i64, _vp, _i32, _vp, _vp]),
    "sst_inverse_zone": (_i32, [_vp, _vp, _i64, _vp, _i32, _i32, _vp, _vp]),
    "sst_stft": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sst_targets": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
    "sst_stft_band": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]),
    "sst_absmax": (_i32, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class SSTError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        name = lib.sst_status_str(status).decode()
        super().__init__(f"{name}: {message}")


def check(status: int, plan=None):
    if status != SST_OK:
        msg = lib.sst_last_error(plan)
        raise SSTError(status, msg.decode() if msg else "")
    return status
