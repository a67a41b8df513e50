"""The multi-rank step bench.py times (dist.ShardedRun: forward of the rank's frames, inverse
accumulate over its span, seam exchange, fused seam-add finalise) run by 2 processes on ONE GPU
(ranks share cuda:0; gloo with the seams staged through the host -- NCCL needs distinct devices),
against the single-rank forward + inverse.  Kernels of the two ranks never wait on each other (the
seam exchange is host-mediated between launches), as B200_PROFILING.md requires for ranks sharing
a GPU.  T rows must match bitwise (frames are independent, P12 / P13), x_hat to fp32
re-association of the seam sums."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SPEC = (60000, 51200.0, 2048, 256.0, 16, 2048, 0.0, 4000.0, 4)
CHUNKED = (30011, 25600.0, 512, 64.0, 4, 512, 0.0, 12800.0, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _signal(N, fs):
    rng = np.random.default_rng(21)
    t = np.arange(N) / fs
    x = np.cos(2 * np.pi * 0.02 * fs * t) + 0.5 * np.cos(2 * np.pi * (0.05 * fs * t + 0.01 * fs * t * t / t[-1]))
    return (x + 0.1 * rng.standard_normal(N)).astype(np.float32)


def _rank(rank, world, port, spec, chunk, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2003_07065_b200 as P
        from paper_2003_07065_b200 import dist as D
        N, fs, L, sigma, hop, nfft, f1, f2, z = spec
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        x = _signal(N, fs)
        plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
        sh = D.shard(N, hop, L, L // 2, world, rank)
        xs = torch.from_numpy(x[sh.span_lo:sh.span_hi].copy()).to(dev)
        run = D.ShardedRun(plan, sh, xs, inverse=True, chunk_frames=chunk)
        own = run.step()
        full = D.gather_owned(own.contiguous(), sh, N)
        T = plan.forward(xs, sh.frame_begin, sh.frame_end, x_off=sh.span_lo)
        Tg = D.gather_band(T, sh)
        torch.cuda.synchronize()
        if rank == 0:
            q.put((full.cpu().numpy(), Tg.cpu().numpy()))
        plan.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec,chunk", [(SPEC, 0), (CHUNKED, 1000)], ids=["C3-like", "C5-like-chunked"])
def test_two_ranks_on_one_gpu_equal_single_rank(spec, chunk):
    import paper_2003_07065_b200 as P
    N, fs, L, sigma, hop, nfft, f1, f2, z = spec
    x = _signal(N, fs)
    plan = P.Plan(N, fs, L, sigma, hop, nfft, f1, f2, z, gamma=1e-4, device=0)
    xd = torch.from_numpy(x).cuda()
    T_ref = plan.forward(xd)
    y_ref = plan.inverse(T_ref).cpu().numpy()
    T_ref = T_ref.cpu().numpy()
    plan.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, spec, chunk, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, Tg = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(Tg, T_ref)
    err = np.linalg.norm(full - y_ref) / np.linalg.norm(y_ref)
    assert err <= 1e-6, err
