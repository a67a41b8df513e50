"""Time sharding of one long record over ranks.

Rank r of P owns frames [F r / P, F (r+1) / P).  Frames are independent (Eq. 7-9), so the
forward needs no communication: each rank reads its own samples plus a window-length halo.
The inverse's overlap-add (Eq. 26) couples neighbours: samples in
``seam(r) = [fb_r H - c, (fb_r - 1) H - c + L)`` (L - H of them) receive frames from ranks r-1
and r.  Rank r-1 sends its partial sums there to rank r (one NCCL send/recv per boundary);
rank r owns and finalises ``[fb_r H - c, fb_{r+1} H - c)`` clipped to [0, N).

Pure host logic plus torch.distributed point-to-point calls; works with the NCCL backend on
device tensors and with gloo on CPU tensors (tests/test_dist_gloo.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    frame_begin: int
    frame_end: int
    span_lo: int      # samples [span_lo, span_hi) read by the forward / written by the accumulate
    span_hi: int
    own_lo: int       # samples this rank finalises
    own_hi: int
    seam_in: int      # length of the left seam received from rank-1 (0 for rank 0)
    seam_out: int     # length of the right seam sent to rank+1 (0 for the last rank)

    frames_total: int = 0   # F of the whole record

    @property
    def frames(self) -> int:
        return self.frame_end - self.frame_begin


def frames_of(n: int, hop: int) -> int:
    return (n - 1) // hop + 1


def shard(n: int, hop: int, win_len: int, center: int, world: int, rank: int) -> Shard:
    """Frame range, sample span and owned output range of ``rank`` (see module doc)."""
    F = frames_of(n, hop)
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    min_frames = -(-win_len // hop)
    if F // world < min_frames and world > 1:
        raise ValueError(f"each rank needs >= ceil(L/H) = {min_frames} frames; F={F}, world={world}")
    fb = F * rank // world
    fe = F * (rank + 1) // world
    span_lo = max(0, fb * hop - center)
    span_hi = min(n, (fe - 1) * hop - center + win_len)
    own_lo = 0 if rank == 0 else max(0, fb * hop - center)
    own_hi = n if rank == world - 1 else min(n, fe * hop - center)
    seam_in = 0
    if rank > 0:
        lo = max(0, fb * hop - center)
        hi = min(n, (fb - 1) * hop - center + win_len)
        seam_in = max(0, hi - lo)
    seam_out = 0
    if rank < world - 1:
        lo = max(0, fe * hop - center)
        hi = min(n, (fe - 1) * hop - center + win_len)
        seam_out = max(0, hi - lo)
    return Shard(rank, world, fb, fe, span_lo, span_hi, own_lo, own_hi, seam_in, seam_out, F)


def _staged(t: torch.Tensor, group) -> bool:
    """gloo moves host tensors only: device buffers are staged through the host."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def exchange_seams(y_span: torch.Tensor, sh: Shard, hop: int, center: int, group=None):
    """Send this rank's right-seam partial sums to rank+1 and receive rank-1's partial sums of this
    rank's left seam (ncclSend / ncclRecv via batch_isend_irecv; through the host under gloo).
    Only moves bytes: the addition (Eq. 26) happens in the library, fused into the finalize pass
    (``Plan.inverse_finalize_seam``).  ``y_span`` holds the unnormalised partial y over
    [span_lo, span_hi).  Returns the received seam (global samples [own_lo, own_lo + seam_in)) or
    None."""
    if sh.world == 1:
        return None
    stage = _staged(y_span, group)
    ops = []
    recv = None
    if sh.seam_out > 0:
        lo = max(0, sh.frame_end * hop - center) - sh.span_lo
        out = y_span[lo:lo + sh.seam_out].contiguous()
        ops.append(dist.P2POp(dist.isend, out.cpu() if stage else out, sh.rank + 1, group))
    if sh.seam_in > 0:
        recv = torch.empty(sh.seam_in, dtype=y_span.dtype, device="cpu" if stage else y_span.device)
        ops.append(dist.P2POp(dist.irecv, recv, sh.rank - 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if recv is not None and stage:
        recv = recv.to(y_span.device, non_blocking=False)
    return recv


def finalize_owned(plan, y_span: torch.Tensor, sh: Shard, recv) -> torch.Tensor:
    """Normalise the samples this rank owns, adding the received left seam in the same pass
    (sst_inverse_finalize_seam).  Returns the owned slice (a view of ``y_span``)."""
    own = own_slice(y_span, sh)
    plan.inverse_finalize_seam(own, sh.own_lo, recv, sh.own_lo)
    return own


class ShardedRun:
    """One rank's share of the hot path over a time-sharded record: sst_forward of
    its frames (no collective), and with ``inverse`` the accumulate of its frames' Eq. 26 partial
    sums over its sample span, the seam exchange with its neighbours, and the owned-range finalise.
    ``chunk_frames`` bounds the T buffer (records whose band plane does not fit, e.g. C5's 256 GiB
    on one GPU): the frames are then processed chunk by chunk, forward then accumulate, reusing it.
    This is the multi-rank step ``bench.py --gpus N`` times."""

    def __init__(self, plan, sh: Shard, x_span: torch.Tensor, inverse: bool = True, chunk_frames: int = 0,
                 group=None):
        self.plan, self.sh, self.x, self.inverse, self.group = plan, sh, x_span, inverse, group
        lay = plan.layout
        self.hop, self.c = lay["hop"], lay["center"]
        n = sh.frames
        self.chunk = n if chunk_frames <= 0 else min(n, chunk_frames)
        self.T = torch.empty((self.chunk, plan.bins), dtype=torch.complex64, device=plan.device)
        self.y = torch.empty(sh.span_hi - sh.span_lo, dtype=torch.float32, device=plan.device) if inverse else None
        self.own = None

    def step(self, forward_only: bool = False):
        """One pass; ``forward_only`` runs just the chunked forward (timing of the forward share)."""
        sh, plan = self.sh, self.plan
        inv = self.inverse and not forward_only
        if inv:
            self.y.zero_()
        for fb in range(sh.frame_begin, sh.frame_end, self.chunk):
            fe = min(sh.frame_end, fb + self.chunk)
            T = self.T[:fe - fb]
            plan.forward(self.x, fb, fe, x_off=sh.span_lo, out=T)
            if inv:
                plan.inverse_accumulate(T, fb, fe, self.y, y_off=sh.span_lo)
        if inv:
            recv = exchange_seams(self.y, sh, self.hop, self.c, self.group)
            self.own = finalize_owned(plan, self.y, sh, recv)
        return self.own

    @property
    def launches_per_step(self) -> int:
        """Library kernels per step: per chunk the forward (main, R23 re-decision, R23 repair) and the
        accumulate (inverse kernel, CTA-seam kernel); one finalize."""
        chunks = -(-self.sh.frames // self.chunk)
        return chunks * 3 if not self.inverse else chunks * 5 + 1


def own_slice(y_span: torch.Tensor, sh: Shard) -> torch.Tensor:
    """View of the samples this rank finalises."""
    return y_span[sh.own_lo - sh.span_lo: sh.own_hi - sh.span_lo]


def gather_owned(y_own: torch.Tensor, sh: Shard, n: int, dst: int = 0, group=None):
    """Collect every rank's owned samples into one [N] tensor on ``dst`` (verification only;
    excluded from throughput; staged through the host under gloo).  Returns the tensor on dst,
    None elsewhere."""
    if sh.world == 1:
        return y_own
    if _staged(y_own, group):
        out = gather_owned(y_own.cpu(), sh, n, dst, group)
        return None if out is None else out.to(y_own.device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=y_own.device) for _ in range(sh.world)]
    dist.all_gather(sizes, torch.tensor([y_own.numel()], dtype=torch.int64, device=y_own.device), group=group)
    mx = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros(mx, dtype=y_own.dtype, device=y_own.device)
    pad[:y_own.numel()] = y_own
    bufs = [torch.zeros(mx, dtype=y_own.dtype, device=y_own.device) for _ in range(sh.world)]
    dist.all_gather(bufs, pad, group=group)
    if sh.rank != dst:
        return None
    return torch.cat([b[:int(s.item())] for b, s in zip(bufs, sizes)])[:n]


def gather_band(T_local: torch.Tensor, sh: Shard, dst: int = 0, group=None):
    """Collect the ranks' band rows T[frame_begin:frame_end, :B] into the whole-record plane on
    ``dst`` (row order = rank order = frame order; SURVEY §8(e) 'optional band gather', for
    verification and small records -- excluded from throughput).  Complex tensors travel as their
    real view; ranks' row counts may differ by one.  Returns [F, B] on dst, None elsewhere."""
    if sh.world == 1:
        return T_local
    if _staged(T_local, group):
        out = gather_band(T_local.cpu(), sh, dst, group)
        return None if out is None else out.to(T_local.device)
    rows_per = [frames_of_rank(sh, r) for r in range(sh.world)]
    mx = max(rows_per)
    real = torch.view_as_real(T_local.contiguous())                  # [rows, B, 2]
    pad = torch.zeros((mx,) + tuple(real.shape[1:]), dtype=real.dtype, device=real.device)
    pad[:real.shape[0]] = real
    bufs = [torch.zeros_like(pad) for _ in range(sh.world)]
    dist.all_gather(bufs, pad, group=group)
    if sh.rank != dst:
        return None
    return torch.view_as_complex(torch.cat([b[:n] for b, n in zip(bufs, rows_per)]).contiguous())


def frames_of_rank(sh: Shard, r: int) -> int:
    """Frame count of rank r under the same partition as ``shard``."""
    F = sh.frames_total
    return F * (r + 1) // sh.world - F * r // sh.world


def max_over_ranks(value: float, device, group=None) -> float:
    """all_reduce(MAX) of one float (timings, max|S|)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        if _staged(t, group):
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


__all__ = ["Shard", "shard", "exchange_seams", "finalize_owned", "ShardedRun", "own_slice", "gather_owned",
           "gather_band", "max_over_ranks", "frames_of"]
