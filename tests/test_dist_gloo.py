"""Multi-rank host logic of the time-sharded path on CPU / gloo.

The forward needs no collective (frames are independent, Eq. 7-9), so what couples ranks is the
inverse's overlap-add (Eq. 26): each rank accumulates the unnormalised sum of its own
frames over its sample span, ``dist.exchange_seams`` moves rank r-1's right spill to rank r (one
send/recv per boundary), rank r adds it to its left seam while normalising the samples it owns,
and ``gather_owned`` concatenates them.  Here the per-rank partial sums come from the fp64 oracle
(test-side only), so the check isolates the sharding arithmetic + the collectives:
sharded result == the oracle's single-process inverse, to fp64 rounding.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2003_07065_b200 import dist as D

CASES = [
    # N, L, sigma, hop, nfft, f1, f2, z
    (3001, 64, 8.0, 4, 64, 0.0, 512.0, 1),
    (4099, 96, 12.0, 7, 128, 96.0, 296.0, 3),
    (2600, 128, 16.0, 16, 128, 0.0, 480.0, 2),
]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(case):
    N, L, sigma, hop, nfft, f1, f2, z = case
    fs = 1024.0
    rng = np.random.default_rng(7)
    t = np.arange(N) / fs
    x = np.cos(2 * np.pi * 150 * t) + 0.5 * np.cos(2 * np.pi * (220 * t + 20 * t * t)) + 0.1 * rng.standard_normal(N)
    g, gd, c = O.gaussian_window(L, sigma)
    T = O.sst_forward(x, g, gd, c, hop, nfft, fs, f1, f2, z, 0.0)
    k1 = O.band_grid(fs, nfft, f1, f2, z)["k1"]
    return N, L, hop, nfft, z, g, c, T, k1


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, L, hop, nfft, z, g, c, T, k1 = _problem(case)
        sh = D.shard(N, hop, L, c, world, rank)
        # unnormalised partial OLA of this rank's frames over its span: the oracle's normalised
        # output times C d[n] (d over the whole record), i.e. sum_m g r~_m (Eq. 26 numerator)
        C = np.sqrt(2.0)
        xr = O.sst_inverse(T[sh.frame_begin:sh.frame_end], g, c, hop, nfft, z, k1, N,
                           frame_begin=sh.frame_begin, n0=sh.span_lo, n1=sh.span_hi)
        d = O.frame_diagonal(g, c, hop, N, sh.span_lo, sh.span_hi)
        y = torch.from_numpy(xr * C * d)
        recv = D.exchange_seams(y, sh, hop, c)
        own = D.own_slice(y, sh).clone()
        if recv is not None:                      # the library fuses this add into its finalize pass
            own[:recv.numel()] += recv
        d_own = O.frame_diagonal(g, c, hop, N, sh.own_lo, sh.own_hi)
        own = own / torch.from_numpy(C * d_own)
        full = D.gather_owned(own.contiguous(), sh, N)
        mx = D.max_over_ranks(float(rank), torch.device("cpu"))
        Tg = D.gather_band(torch.from_numpy(T[sh.frame_begin:sh.frame_end].astype(np.complex64)), sh)
        if rank == 0:
            out_q.put((full.numpy(), mx, Tg.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES)
def test_sharded_inverse_equals_single(world, case):
    N, L, hop, nfft, z, g, c, T, k1 = _problem(case)
    ref = O.sst_inverse(T, g, c, hop, nfft, z, k1, N)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, mx, Tg = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert mx == world - 1
    assert full.shape == (N,)
    err = np.max(np.abs(full - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err
    assert np.array_equal(Tg, T.astype(np.complex64))              # band gather restores the plane


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_shard_partition_properties(world):
    """Frame ranges tile [0, F); owned samples tile [0, N); each span covers every sample its
    frames touch; seam lengths are L - H (interior) and match between neighbours."""
    N, L, hop = 100_003, 512, 4
    c = L // 2
    F = D.frames_of(N, hop)
    shards = [D.shard(N, hop, L, c, world, r) for r in range(world)]
    assert shards[0].frame_begin == 0 and shards[-1].frame_end == F
    assert shards[0].own_lo == 0 and shards[-1].own_hi == N
    for a, b in zip(shards, shards[1:]):
        assert a.frame_end == b.frame_begin
        assert a.own_hi == b.own_lo
        assert a.seam_out == b.seam_in == L - hop
    for s in shards:
        assert s.span_lo == max(0, s.frame_begin * hop - c)
        assert s.span_hi == min(N, (s.frame_end - 1) * hop - c + L)
        assert s.span_lo <= s.own_lo < s.own_hi <= s.span_hi


def test_shard_rejects_too_many_ranks():
    with pytest.raises(ValueError):
        D.shard(1000, 10, 512, 256, 8, 0)


class _OraclePlan:
    """Stand-in for ``Plan`` with the oracle's arithmetic (test-side only), so that
    ``dist.ShardedRun`` -- the multi-rank step bench.py times -- runs on CPU / gloo: forward rows,
    unnormalised Eq. 26 partial sums, seam add + normalisation."""

    def __init__(self, case):
        self.N, self.L, self.hop, self.nfft, self.z, self.g, self.c, self.Tfull, self.k1 = _problem(case)
        self.bins = self.Tfull.shape[1]
        self.layout = {"hop": self.hop, "center": self.c}
        self.device = torch.device("cpu")
        self.calls = []

    def forward(self, x, fb, fe, x_off=0, out=None):
        self.calls.append(("forward", fb, fe))
        out[:fe - fb] = torch.from_numpy(self.Tfull[fb:fe].astype(np.complex64))
        return out

    def inverse_accumulate(self, T, fb, fe, y, y_off=0):
        self.calls.append(("accumulate", fb, fe))
        n1 = y_off + y.numel()
        xr = O.sst_inverse(T[:fe - fb].numpy().astype(np.complex128), self.g, self.c, self.hop, self.nfft, self.z,
                           self.k1, self.N, frame_begin=fb, n0=y_off, n1=n1)
        d = O.frame_diagonal(self.g, self.c, self.hop, self.N, y_off, n1)
        y += torch.from_numpy(xr * np.sqrt(2.0) * d).to(y.dtype)
        return y

    def inverse_finalize_seam(self, y, y_off, seam, seam_off):
        if seam is not None:
            y[seam_off - y_off:seam_off - y_off + seam.numel()] += seam
        d = O.frame_diagonal(self.g, self.c, self.hop, self.N, y_off, y_off + y.numel())
        y /= torch.from_numpy(np.sqrt(2.0) * d).to(y.dtype)
        return y


def _run_worker(rank, world, port, case, chunk, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = _OraclePlan(case)
        sh = D.shard(plan.N, plan.hop, plan.L, plan.c, world, rank)
        run = D.ShardedRun(plan, sh, torch.zeros(sh.span_hi - sh.span_lo), inverse=True, chunk_frames=chunk)
        run.y = run.y.double()
        own = run.step()
        full = D.gather_owned(own.contiguous(), sh, plan.N)
        chunks = sum(1 for k in plan.calls if k[0] == "forward")
        if rank == 0:
            out_q.put((full.numpy(), chunks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunk", [(1, 0), (2, 0), (2, 37), (3, 50)])
def test_sharded_run_step(world, chunk):
    """dist.ShardedRun (chunked forward + accumulate, seam exchange, fused seam-add finalise) over
    world ranks equals the single-process inverse; chunking reuses one T buffer."""
    case = CASES[1]
    N, L, hop, nfft, z, g, c, T, k1 = _problem(case)
    ref = O.sst_inverse(T.astype(np.complex64).astype(np.complex128), g, c, hop, nfft, z, k1, N)   # T travels as complex64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_worker, args=(r, world, port, case, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, chunks = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    F0 = D.shard(N, hop, L, c, world, 0).frames
    assert chunks == (1 if chunk == 0 else -(-F0 // chunk))
    err = np.max(np.abs(full - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err
