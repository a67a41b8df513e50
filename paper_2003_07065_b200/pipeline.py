"""Host-to-host SST round trip with copy/compute overlap (public API helper).

``roundtrip(plan, x_host, y_host, T)`` takes a pinned host record x, runs the forward (T stays in
HBM) and the inverse, and leaves x_hat in the pinned host buffer y_host.  The record is cut into
`chunks` frame ranges; three CUDA streams overlap, chunk by chunk,
  copy-in (H2D of the chunk's new samples) -> sst_forward + sst_inverse_accumulate of the chunk ->
  sst_inverse_finalize of the samples no later frame touches -> copy-out (D2H of those samples),
ordered with CUDA events, so the PCIe/C2C transfers hide under the kernels.  Every transform step
runs in libsst.so; this module only orders launches.  Frames are independent (Eq. 7-9); the
inverse's overlap-add (Eq. 26) is linear, so accumulating chunk by chunk and normalising each
sample once all its frames are in gives the single-call result up to fp32 re-association.
"""

from __future__ import annotations

import gc

import torch


class RoundTrip:
    """Reusable device buffers + streams for repeated round trips of one plan."""

    def __init__(self, plan, chunks: int = 8):
        from ._lib import SST_GAMMA_RELATIVE
        if (plan.flags & SST_GAMMA_RELATIVE) and plan._absmax_ref is None:
            # each chunk's forward would otherwise take max|S| over its own frames only, so the
            # chunks would use different thresholds (Eq. 13): require the record's max up front
            raise ValueError("RoundTrip with SST_GAMMA_RELATIVE needs the record's max|S|: call "
                             "plan.set_absmax(plan.absmax(x_device)) (or an all-reduced max) first")
        self.plan = plan
        lay = plan.layout
        self.N, self.H, self.c, self.L, self.F = lay["n"], lay["hop"], lay["center"], lay["win_len"], lay["frames"]
        self.chunks = max(1, min(chunks, self.F))
        dev = plan.device
        self.x = torch.empty(self.N, dtype=torch.float32, device=dev)
        self.y = torch.empty(self.N, dtype=torch.float32, device=dev)
        self.s_in = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        F = self.F
        self.cuts = [F * i // self.chunks for i in range(self.chunks + 1)]

    def _span_hi(self, fe):
        return min(self.N, (fe - 1) * self.H - self.c + self.L)

    def run(self, x_host: torch.Tensor, y_host: torch.Tensor, T: torch.Tensor):
        plan, H, c, N = self.plan, self.H, self.c, self.N
        comp = torch.cuda.current_stream(plan.device)
        # y is accumulated: clear it on the compute stream (ordered before the first accumulate)
        self.y.zero_()
        start = torch.cuda.Event()
        start.record(comp)
        self.s_in.wait_event(start)
        self.s_out.wait_event(start)
        copied = 0            # x samples [0, copied) are on the device (or queued)
        finalized = 0         # y samples [0, finalized) are final
        for i in range(self.chunks):
            fb, fe = self.cuts[i], self.cuts[i + 1]
            hi = self._span_hi(fe)
            with torch.cuda.stream(self.s_in):
                if hi > copied:
                    self.x[copied:hi].copy_(x_host[copied:hi], non_blocking=True)
                    copied = hi
                ready = torch.cuda.Event()
                ready.record(self.s_in)
            comp.wait_event(ready)
            plan.forward(self.x, fb, fe, out=T[fb:fe])
            lo = max(0, fb * H - c)
            plan.inverse_accumulate(T[fb:fe], fb, fe, self.y[lo:hi], y_off=lo)
            # samples below fe*H - c receive no frame >= fe (frame m starts at m H - c)
            fin = N if i == self.chunks - 1 else min(N, max(0, fe * H - c))
            if fin > finalized:
                plan.inverse_finalize(self.y[finalized:fin], y_off=finalized)
                done = torch.cuda.Event()
                done.record(comp)
                self.s_out.wait_event(done)
                with torch.cuda.stream(self.s_out):
                    y_host[finalized:fin].copy_(self.y[finalized:fin], non_blocking=True)
                finalized = fin
        end = torch.cuda.Event()
        end.record(self.s_out)
        comp.wait_event(end)
        end_in = torch.cuda.Event()
        end_in.record(self.s_in)
        comp.wait_event(end_in)
        return y_host


    def capture(self, x_host: torch.Tensor, y_host: torch.Tensor, T: torch.Tensor) -> "torch.cuda.CUDAGraph":
        """Record one run() (copies, kernels, cross-stream events) as a CUDA graph bound to these
        buffers; ``graph.replay()`` then repeats the whole host-to-host round trip with one launch
        and no per-chunk host work, so many small chunks cost no Python overhead."""
        comp = torch.cuda.current_stream(self.plan.device)
        side = torch.cuda.Stream(self.plan.device)
        side.wait_stream(comp)
        with torch.cuda.stream(side):                 # warm-up on the capture stream (torch's advice)
            self.run(x_host, y_host, T)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        # no garbage collection inside the capture: a finaliser that frees device memory (a plan,
        # a tensor of another stream) would invalidate it; torch.cuda.graph collects right before
        gc_on = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(side):
                # thread_local: only this thread's capture-unsafe calls invalidate the capture
                with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                    self.run(x_host, y_host, T)
        finally:
            if gc_on:
                gc.enable()
        comp.wait_stream(side)
        return g


def roundtrip(plan, x_host: torch.Tensor, y_host: torch.Tensor, T: torch.Tensor, chunks: int = 8):
    """One host->host forward + inverse with overlapped transfers (see module doc)."""
    return RoundTrip(plan, chunks).run(x_host, y_host, T)
