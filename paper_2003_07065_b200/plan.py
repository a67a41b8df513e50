"""Python face of the SST library: a ``Plan`` over the C ABI (include/sst.h).

Marshalling only: tensors are checked for device/dtype/contiguity and their pointers passed
to libsst.so; all compute runs in its sm_100a kernels on the caller's current CUDA stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib as L


def gaussian_window(win_len: int, sigma: float, center: int = -1):
    """Unit-energy Gaussian window and analytic derivative (sst_gaussian_window, R1)."""
    g = np.zeros(win_len, dtype=np.float64)
    gd = np.zeros(win_len, dtype=np.float64)
    L.check(L.sst_gaussian_window(win_len, float(sigma), center,
                                  g.ctypes.data_as(L._dp), gd.ctypes.data_as(L._dp)))
    return g, gd


def make_params(n, fs, win_len, sigma, hop, nfft, f1, f2, zoom=1, gamma=0.0, flags=0,
                g=None, gd=None, center=-1):
    """Build an ``sst_params`` (plus the window arrays it points at, kept alive by the caller)."""
    if g is None or gd is None:
        g, gd = gaussian_window(win_len, sigma, center)
    g = np.ascontiguousarray(g, dtype=np.float64)
    gd = np.ascontiguousarray(gd, dtype=np.float64)
    if g.shape != (win_len,) or gd.shape != (win_len,):
        raise ValueError("window arrays must have win_len taps")
    p = L.sst_params(n=int(n), fs=float(fs), win_len=int(win_len), win_center=int(center),
                     g=g.ctypes.data_as(L._dp), gd=gd.ctypes.data_as(L._dp), sigma=float(sigma),
                     hop=int(hop), nfft=int(nfft), f1=float(f1), f2=float(f2), zoom=int(zoom),
                     gamma=float(gamma), flags=int(flags))
    return p, (g, gd)


def validate(**kw) -> int:
    """sst_params_validate (no GPU needed).  Returns the status code."""
    p, keep = make_params(**kw)
    return L.sst_params_validate(ctypes.byref(p))


def layout(**kw) -> dict:
    """sst_params_layout (no GPU needed); raises SSTError on invalid parameters."""
    p, keep = make_params(**kw)
    out = L.sst_layout()
    L.check(L.sst_params_layout(ctypes.byref(p), ctypes.byref(out)))
    return out.as_dict()


def _ptr(t: torch.Tensor, device: torch.device, dtype, name: str) -> int:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _rows(T: torch.Tensor, rows: int, bins: int, name: str):
    """T must be a 2-D [>= rows, ldT >= B] plane (the C ABI cannot see tensor extents)."""
    if not isinstance(T, torch.Tensor) or T.dim() != 2:
        raise ValueError(f"{name} must be a 2-D [rows, ldT] tensor")
    if rows < 0 or T.shape[0] < rows:
        raise ValueError(f"{name} has {T.shape[0]} rows, need {rows}")
    if T.shape[1] < bins:
        raise ValueError(f"{name} has ldT = {T.shape[1]} < B = {bins}")


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_DEFERRED: list = []        # plan handles whose destruction was requested during a graph capture


def _capturing() -> bool:
    try:
        return torch.cuda.is_available() and torch.cuda.is_current_stream_capturing()
    except Exception:
        return False


def _flush_deferred():
    while _DEFERRED and not _capturing():
        L.sst_plan_destroy(_DEFERRED.pop())


class Plan:
    """sst_plan wrapper.  Parameters follow sst_params (include/sst.h); sigma in samples."""

    def __init__(self, n, fs, win_len, sigma, hop, nfft, f1, f2, zoom=1, gamma=0.0, flags=0,
                 g=None, gd=None, center=-1, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2003_07065_b200.Plan needs a CUDA device (no CPU fallback)")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           (device if isinstance(device, int) else torch.device(device).index or 0))
        self.device = dev
        p, keep = make_params(n, fs, win_len, sigma, hop, nfft, f1, f2, zoom, gamma, flags, g, gd, center)
        self._keep = keep
        _flush_deferred()
        h = ctypes.c_void_p()
        L.check(L.sst_plan_create(ctypes.byref(p), dev.index, ctypes.byref(h)))
        self._h = h
        warn = L.sst_last_error(h)
        self.warning = warn.decode() if warn else ""
        lay = L.sst_layout()
        L.check(L.sst_plan_layout(h, ctypes.byref(lay)), h)
        self.layout = lay.as_dict()
        self.flags = flags
        self._absmax_ref = None

    # ------------------------------------------------------------------ properties
    @property
    def frames(self) -> int:
        return self.layout["frames"]

    @property
    def bins(self) -> int:
        return self.layout["bins"]

    @property
    def n(self) -> int:
        return self.layout["n"]

    @property
    def src_bins(self) -> int:
        return self.layout["src_bins"]

    def _frames(self, fb, fe):
        fe = self.frames if fe is None else fe
        return int(fb), int(fe)

    # ------------------------------------------------------------------ threshold
    def set_gamma(self, gamma_abs: float):
        L.check(L.sst_plan_set_gamma(self._h, float(gamma_abs)), self._h)

    def set_absmax(self, t: torch.Tensor | None):
        """RELATIVE mode: use this device float32 scalar as max|S| (e.g. all-reduced over ranks)."""
        ptr = None if t is None else _ptr(t, self.device, torch.float32, "absmax")
        self._absmax_ref = t
        L.check(L.sst_plan_set_absmax(self._h, ptr), self._h)

    def counters(self) -> dict:
        """sst_plan_counters: R23 fp64 re-decisions so far (synchronous)."""
        out = (ctypes.c_uint64 * 2)()
        L.check(L.sst_plan_counters(self._h, out), self._h)
        return {"redecided": int(out[0]), "changed": int(out[1])}

    # ------------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor, frame_begin: int = 0, frame_end: int | None = None,
                x_off: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
        """sst_forward: T[frames, B] complex64 for frames [frame_begin, frame_end)."""
        fb, fe = self._frames(frame_begin, frame_end)
        if out is None:
            out = torch.empty((max(0, fe - fb), self.bins), dtype=torch.complex64, device=self.device)
        if out.dim() != 2 or out.shape[0] < fe - fb:
            raise ValueError("out must be [frames, ldT]")
        L.check(L.sst_forward(self._h, _ptr(x, self.device, torch.float32, "x"), int(x_off), x.numel(), fb, fe,
                              _ptr(out, self.device, torch.complex64, "T"), out.shape[1], _stream(self.device)), self._h)
        return out

    # ------------------------------------------------------------------ inverse
    def inverse(self, T: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """sst_inverse: x_hat[N] float32 from the whole-record T (Eq. 25-26)."""
        if T.dim() != 2 or T.shape[0] != self.frames:
            raise ValueError("T must be [F, ldT] with all frames")
        _rows(T, self.frames, self.bins, "T")
        if out is None:
            out = torch.empty(self.n, dtype=torch.float32, device=self.device)
        if out.numel() < self.n:
            raise ValueError("out must hold N samples")
        L.check(L.sst_inverse(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1],
                              _ptr(out, self.device, torch.float32, "y"), _stream(self.device)), self._h)
        return out

    def inverse_accumulate(self, T: torch.Tensor, frame_begin: int, frame_end: int, y: torch.Tensor,
                           y_off: int = 0) -> torch.Tensor:
        """sst_inverse_accumulate: y += unnormalised OLA of frames [frame_begin, frame_end)."""
        _rows(T, int(frame_end) - int(frame_begin), self.bins, "T")
        L.check(L.sst_inverse_accumulate(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1],
                                         int(frame_begin), int(frame_end),
                                         _ptr(y, self.device, torch.float32, "y"), int(y_off), y.numel(),
                                         _stream(self.device)), self._h)
        return y

    def inverse_finalize(self, y: torch.Tensor, y_off: int = 0) -> torch.Tensor:
        """sst_inverse_finalize: y /= C d[n] on its global span."""
        L.check(L.sst_inverse_finalize(self._h, _ptr(y, self.device, torch.float32, "y"), int(y_off), y.numel(),
                                       _stream(self.device)), self._h)
        return y

    def inverse_finalize_seam(self, y: torch.Tensor, y_off: int, seam: torch.Tensor | None,
                              seam_off: int = 0) -> torch.Tensor:
        """sst_inverse_finalize_seam: y = (y + seam) / (C d[n]) in one pass (seam over global samples
        [seam_off, seam_off + seam.numel()), inside y's span); seam None -> plain finalize."""
        if seam is None or seam.numel() == 0:
            return self.inverse_finalize(y, y_off)
        L.check(L.sst_inverse_finalize_seam(self._h, _ptr(y, self.device, torch.float32, "y"), int(y_off), y.numel(),
                                            _ptr(seam, self.device, torch.float32, "seam"), int(seam_off), seam.numel(),
                                            _stream(self.device)), self._h)
        return y

    # ------------------------------------------------------------------ plain STFT synthesis / analysis
    def istft(self, S: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """sst_istft: Eq. 10-11 synthesis of the one-sided STFT S[F, >= N_f/2+1] (from stft())."""
        if S.dim() != 2 or S.shape[0] != self.frames:
            raise ValueError("S must be [F, ldS] with all frames")
        if out is None:
            out = torch.empty(self.n, dtype=torch.float32, device=self.device)
        L.check(L.sst_istft(self._h, _ptr(S, self.device, torch.complex64, "S"), S.shape[1],
                            _ptr(out, self.device, torch.float32, "y"), _stream(self.device)), self._h)
        return out

    def renyi(self, T: torch.Tensor, alpha: float = 3.0) -> torch.Tensor:
        """sst_renyi: device float64 [3] = (sum |T|^2, sum |T|^(2 alpha), H_alpha) (Eq. 32)."""
        _rows(T, T.shape[0] if T.dim() == 2 else -1, self.bins, "T")
        out = torch.empty(3, dtype=torch.float64, device=self.device)
        L.check(L.sst_renyi(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[0], T.shape[1],
                            float(alpha), out.data_ptr(), _stream(self.device)), self._h)
        return out

    # ------------------------------------------------------------------ mode retrieval (f1, R22)
    def ridge_emission(self, T: torch.Tensor):
        """sst_ridge_emission: (E float64 [rows, B], floor float64 scalar) on the device."""
        _rows(T, T.shape[0] if T.dim() == 2 else -1, self.bins, "T")
        E = torch.empty((T.shape[0], self.bins), dtype=torch.float64, device=self.device)
        fl = torch.empty((), dtype=torch.float64, device=self.device)
        L.check(L.sst_ridge_emission(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1], T.shape[0],
                                     E.data_ptr(), fl.data_ptr(), _stream(self.device)), self._h)
        return E, fl

    def ridge(self, E: torch.Tensor, floor: torch.Tensor, lam: float = 0.01, count: int = 1, suppress: int = 3):
        """sst_ridge: int32 [count, rows] ridge paths (E is modified: suppressed zones)."""
        if E.dim() != 2 or E.shape[1] != self.bins:
            raise ValueError(f"E must be [rows, B={self.bins}]")
        paths = torch.empty((count, E.shape[0]), dtype=torch.int32, device=self.device)
        L.check(L.sst_ridge(self._h, _ptr(E, self.device, torch.float64, "E"), E.shape[0], float(lam), int(count),
                            int(suppress), _ptr(floor, self.device, torch.float64, "floor"), paths.data_ptr(),
                            _stream(self.device)), self._h)
        return paths

    def ridges(self, T: torch.Tensor, lam: float = 0.01, count: int = 1, suppress: int = 3):
        E, fl = self.ridge_emission(T)
        return self.ridge(E, fl, lam, count, suppress)

    def zone_mask(self, T: torch.Tensor, path: torch.Tensor, half: int, keep_inside: bool = True) -> torch.Tensor:
        """sst_zone_mask, in place on T."""
        _rows(T, T.shape[0] if T.dim() == 2 else -1, self.bins, "T")
        if path.numel() < T.shape[0]:
            raise ValueError("path must have one bin per row of T")
        L.check(L.sst_zone_mask(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1], T.shape[0],
                                _ptr(path, self.device, torch.int32, "path"), int(half), int(bool(keep_inside)),
                                _stream(self.device)), self._h)
        return T

    def retrieve_mode(self, T: torch.Tensor, path: torch.Tensor, half: int, keep_inside: bool = True,
                      out: torch.Tensor | None = None) -> torch.Tensor:
        """§2.3 mode retrieval: the downsampled inverse (Eq. 25-26) of T restricted to the zone
        |l - path[m]| <= half (sst_inverse_zone: the zone is applied inside the inverse's T loads,
        T is not copied or modified)."""
        _rows(T, self.frames, self.bins, "T")
        if path.numel() < self.frames:
            raise ValueError("path must have one bin per frame")
        if out is None:
            out = torch.empty(self.n, dtype=torch.float32, device=self.device)
        L.check(L.sst_inverse_zone(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1],
                                   _ptr(path, self.device, torch.int32, "path"), int(half), int(bool(keep_inside)),
                                   _ptr(out, self.device, torch.float32, "y"), _stream(self.device)), self._h)
        return out

    def mode_full(self, T: torch.Tensor, path: torch.Tensor, half: int) -> torch.Tensor:
        """sst_mode_full: Eq. 15 (H_t = 1), float32 [rows]."""
        _rows(T, T.shape[0] if T.dim() == 2 else -1, self.bins, "T")
        if path.numel() < T.shape[0]:
            raise ValueError("path must have one bin per row of T")
        x = torch.empty(T.shape[0], dtype=torch.float32, device=self.device)
        L.check(L.sst_mode_full(self._h, _ptr(T, self.device, torch.complex64, "T"), T.shape[1], T.shape[0],
                                _ptr(path, self.device, torch.int32, "path"), int(half), x.data_ptr(),
                                _stream(self.device)), self._h)
        return x

    # ------------------------------------------------------------------ debug / parity
    def stft(self, x: torch.Tensor, frame_begin: int = 0, frame_end: int | None = None, x_off: int = 0):
        fb, fe = self._frames(frame_begin, frame_end)
        S = torch.empty((fe - fb, self.src_bins), dtype=torch.complex64, device=self.device)
        Sd = torch.empty_like(S)
        L.check(L.sst_stft(self._h, _ptr(x, self.device, torch.float32, "x"), int(x_off), x.numel(), fb, fe,
                           S.data_ptr(), Sd.data_ptr(), _stream(self.device)), self._h)
        return S, Sd

    def stft_band(self, x: torch.Tensor, frame_begin: int = 0, frame_end: int | None = None, x_off: int = 0):
        """sst_stft_band: S, S' of the band's source bins [k1, k2) by the filter bank (f3b plans)."""
        fb, fe = self._frames(frame_begin, frame_end)
        kb = self.layout["k2"] - self.layout["k1"]
        S = torch.empty((fe - fb, kb), dtype=torch.complex64, device=self.device)
        Sd = torch.empty_like(S)
        L.check(L.sst_stft_band(self._h, _ptr(x, self.device, torch.float32, "x"), int(x_off), x.numel(), fb, fe,
                                S.data_ptr(), Sd.data_ptr(), _stream(self.device)), self._h)
        return S, Sd

    @property
    def forward_path(self) -> int:
        return self.layout["forward_path"]

    @property
    def inverse_path(self) -> int:
        return self.layout["inverse_path"]

    def targets(self, x: torch.Tensor, frame_begin: int = 0, frame_end: int | None = None, x_off: int = 0):
        fb, fe = self._frames(frame_begin, frame_end)
        out = torch.empty((fe - fb, self.src_bins), dtype=torch.int32, device=self.device)
        L.check(L.sst_targets(self._h, _ptr(x, self.device, torch.float32, "x"), int(x_off), x.numel(), fb, fe,
                              out.data_ptr(), _stream(self.device)), self._h)
        return out

    def absmax(self, x: torch.Tensor, frame_begin: int = 0, frame_end: int | None = None, x_off: int = 0):
        fb, fe = self._frames(frame_begin, frame_end)
        out = torch.empty((), dtype=torch.float32, device=self.device)
        L.check(L.sst_absmax(self._h, _ptr(x, self.device, torch.float32, "x"), int(x_off), x.numel(), fb, fe,
                             out.data_ptr(), _stream(self.device)), self._h)
        return out

    # ------------------------------------------------------------------ lifetime
    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            if _capturing():
                # sst_plan_destroy frees device memory, which would invalidate a CUDA graph being
                # captured (e.g. a finaliser run by the garbage collector mid-capture): defer it
                _DEFERRED.append(h)
            else:
                L.sst_plan_destroy(h)
        _flush_deferred()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def gamma_bound(x_absmax: float, g) -> float:
    """R6 for C2-C5: 1e-6 * sum(g) * max|x| bounds 1e-6 * max|S| from above; callers use it as the
    absolute threshold so both sides can compute it from x alone."""
    return 1e-6 * float(np.sum(g)) * float(x_absmax)


__all__ = ["Plan", "gaussian_window", "make_params", "validate", "layout", "gamma_bound"]
