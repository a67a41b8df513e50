#!/usr/bin/env python
"""Benchmark of the fast downsampled SST hot path (forward + approximate inverse) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl ours|reference]

One step = the whole hot path over one record: sst_forward of every
frame (band output T in HBM) then the inverse (Eq. 25-26) back to x_hat.  The workload is
BASELINE.json configs[2] (C3, aero-engine run-up, forward + inverse; DESIGN.md §8 says why).
For N>1 (torchrun, one rank per GPU, NCCL) the same record is time-sharded over the ranks (strong
scaling): each rank forwards its frames, accumulates its inverse partial sums, exchanges the OLA
seams with its neighbours over NCCL and finalises the samples it owns (dist.ShardedRun).  Legs
(``--legs``, default C4,C5): the largest configs on their fixed records, sharded the same way --
C4 forward (T resident), C5 forward + inverse in frame chunks with one reused T buffer (its 256 GiB
plane never exists whole on one GPU) -- so t_1 / (P t_P) can be read per config.

Prints ONE JSON line on rank 0.  ``--impl reference`` times the fp64 CPU oracle instead
(the reference arm of this tier), on the box's host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from gen import generate, get_config  # noqa: E402

WORKLOAD_DESC = {
    "C1": "C1 tiny standard SST (100 Hz tone + chirp + noise), N=4096, fs=1024, L=257, H_t=1, N_f=4096, full band, z=1",
    "C2": "C2 spindle-like, N=2^20, fs=25.6k, L=1024, H_t=8, N_f=1024, band 0-2 kHz, z=2",
    "C3": "C3 aero-engine run-up, N=2^24, fs=51.2k, L=2048, H_t=16, N_f=2048, band 0-4 kHz, z=4, fwd+inverse",
    "C4": "C4 long record, N=2^28, fs=51.2k, L=4096, H_t=32, N_f=4096, band 0-6.4 kHz, z=2",
    "C5": "C5 dense grid, N=2^26, fs=25.6k, L=512, H_t=4, N_f=512, full band, z=8",
}
FP32_PEAK_NOTE = "148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz (B200_PROFILING.md unit counts, clocks.max.sm)"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), float(mp.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def _traffic_committed(workload, kernel, frames):
    """DRAM bytes per launch from the committed ncu --set full capture (profiles/traffic.json, written
    by tools/ncu_traffic.py); the fallback when ncu cannot run in this bench."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[workload][kernel]
        return e["dram_bytes"] if e["frames"] == frames else None
    except Exception:
        return None


TRAFFIC_KERNELS = {"forward": "fwd_kernel", "inverse": "inv_(nb_)?kernel"}   # residue-split / narrow-band inverse


def traffic_probe(workload):
    """Child of the bench (under ncu): one forward + one inverse of the workload, nothing timed."""
    import torch

    import paper_2003_07065_b200 as P
    cfg = get_config(workload)
    g, _ = P.gaussian_window(cfg.L, cfg.sigma)
    x_host = generate(cfg, 0, cfg.N)
    gamma = 1e-6 * float(np.sum(g)) * float(np.abs(x_host).max())
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=gamma, device=0)
    x = torch.from_numpy(x_host).cuda()
    T = plan.forward(x)
    plan.inverse(T)
    torch.cuda.synchronize()
    plan.close()


def measure_traffic(workload, kernel, frames, timeout=600):
    """DRAM bytes (read + write) per launch of the dominant kernel, measured in this bench run: ncu
    (dram__bytes_read.sum + dram__bytes_write.sum, --clock-control none) on a child process doing one
    forward + one inverse of the same workload; the first launch of the kernel is the full-size one.
    Falls back to the committed capture when ncu is unavailable or fails (reported in `source`)."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    name = TRAFFIC_KERNELS[kernel]
    if os.path.exists(ncu):
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
               "-k", f"regex:^{name}", "-c", "1", "--csv", sys.executable, os.path.abspath(__file__),
               "--traffic-probe", "--workload", workload]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
            import csv
            import io
            vals = {}
            for row in csv.reader(io.StringIO(r.stdout)):
                if len(row) > 10 and row[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    unit, v = row[-2], float(row[-1].replace(",", ""))
                    vals[row[-3]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            if len(vals) == 2:
                return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                        "read": vals["dram__bytes_read.sum"], "write": vals["dram__bytes_write.sum"],
                        "source": f"ncu in this run (first {name} launch of one forward + inverse)"}
            err = (r.stderr or r.stdout)[-300:]
        except Exception as e:  # noqa: BLE001
            err = repr(e)
    else:
        err = "ncu not found"
    b = _traffic_committed(workload, kernel, frames)
    return {"bytes": b, "source": f"committed profiles/traffic.json ({err.strip()[:200]})"}


def algorithmic_counts(cfg):
    """Per-frame algorithmic work."""
    K = cfg.nfft // 2 + 1
    B = cfg.bins
    zN = cfg.zoom * cfg.nfft
    fwd_flops = 5.0 * cfg.nfft * math.log2(cfg.nfft) + 2.0 * cfg.L + 20.0 * K
    inv_flops = 2.5 * zN * math.log2(zN) + 2.0 * cfg.L + 8.0 * B
    fwd_bytes = 4.0 * cfg.hop + 8.0 * B
    inv_bytes = 8.0 * B + 4.0 * cfg.hop
    return fwd_flops, inv_flops, fwd_bytes, inv_bytes


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------- reference arm
def host_info():
    """Cores this process may use (sched_getaffinity) and the CPU model (/proc/cpuinfo)."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return cores, model


def _oracle_window_record(cfg, nfr, f0=None):
    """A local record for timing the oracle on ``nfr`` consecutive frames of the workload starting at
    global frame f0 (default: a third into the record): local sample j = global sample f0*H + j, so
    local frame m = global frame f0 + m."""
    f0 = cfg.frames // 3 if f0 is None else f0
    lo = f0 * cfg.hop
    hi = min(cfg.N, lo + nfr * cfg.hop + cfg.L)
    return generate(cfg, lo, hi).astype(np.float64)


def _oracle_step(O, cfg, xl, g, gd, c, gamma, nfr):
    """Forward of nfr frames + inverse of the interior half (output window fully covered)."""
    T = O.sst_forward(xl, g, gd, c, cfg.hop, cfg.nfft, cfg.fs, cfg.f1, cfg.f2, cfg.zoom, gamma,
                      frames=np.arange(nfr))
    n0, n1 = (nfr // 4) * cfg.hop, (3 * nfr // 4) * cfg.hop
    O.sst_inverse(T, g, c, cfg.hop, cfg.nfft, cfg.zoom, cfg.k1, xl.size, frame_begin=0, n0=n0, n1=n1)
    return nfr * cfg.hop


def _oracle_setup(name, nfr, f0=None):
    import oracle as O
    cfg = get_config(name)
    g, gd, c = O.gaussian_window(cfg.L, cfg.sigma)
    xl = _oracle_window_record(cfg, nfr, f0)
    gamma = 1e-6 * float(np.sum(g)) * float(np.abs(xl).max())     # reading R6 (bound from x)
    return O, cfg, xl, g, gd, c, gamma


def _oracle_worker(name, nfr, seconds, wid, barrier, out):
    """One process of the all-core oracle timing (BLAS / FFT threads = 1): its own chunk of frames,
    one untimed step, then steps for ``seconds`` after all workers have reached the barrier."""
    O, cfg, xl, g, gd, c, gamma = _oracle_setup(name, nfr, cfg_f0(name, wid))
    _oracle_step(O, cfg, xl, g, gd, c, gamma, nfr)
    barrier.wait()
    t0 = time.perf_counter()
    done = 0
    while time.perf_counter() - t0 < seconds:
        done += _oracle_step(O, cfg, xl, g, gd, c, gamma, nfr)
    out.put((wid, done, time.perf_counter() - t0))


def cfg_f0(name, wid):
    cfg = get_config(name)
    return (cfg.frames // 3 + wid * 4096) % max(1, cfg.frames - 8192)


def _single_thread_env():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
        os.environ[v] = "1"


def oracle_all_core(name, nfr, seconds, procs):
    """The oracle as it stands on every host core: one spawned process per core over its own
    frame chunk (SURVEY §8(c) 'Parallelism for timing'; the arithmetic is unchanged).  Returns
    (input Msamples/s aggregated over the processes, processes)."""
    import multiprocessing as mp
    _single_thread_env()
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(procs)
    out = ctx.Queue()
    ps = [ctx.Process(target=_oracle_worker, args=(name, nfr, seconds, w, barrier, out)) for w in range(procs)]
    for p in ps:
        p.start()
    res = [out.get() for _ in ps]
    for p in ps:
        p.join()
    samples = sum(r[1] for r in res)
    dt = max(r[2] for r in res)
    return samples / dt / 1e6, procs


def oracle_gamma_prepass(name, nfr, seconds):
    """The relative-gamma pre-pass of the oracle (max |S| over the frames, Eq. 13 / R6):
    one STFT per frame, timed on its own, single process; input Msamples/s."""
    O, cfg, xl, g, gd, c, gamma = _oracle_setup(name, nfr)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        float(np.abs(O.stft(xl, g, c, cfg.hop, cfg.nfft, frames=np.arange(nfr))).max())
        done += nfr * cfg.hop
    return done / (time.perf_counter() - t0) / 1e6


def run_reference(args, cfg):
    """The fp64 numpy oracle, as it stands, on the box's host cores: each step is one bounded sample
    of the workload per core (``--ref-frames`` consecutive frames, forward + inverse of the interior),
    all cores in parallel (one spawned process each); the step time is the wall time of the slowest."""
    import multiprocessing as mp
    cores, model = host_info()
    procs = max(1, min(cores, args.ref_procs or cores))
    _single_thread_env()
    ctx = mp.get_context("spawn")
    nfr = args.ref_frames
    with ctx.Pool(procs) as pool:
        def step():
            return sum(pool.starmap(_ref_step_worker, [(cfg.name, nfr, w) for w in range(procs)]))
        pool.starmap(_ref_step_worker, [(cfg.name, 8, w) for w in range(procs)])   # import + cache warm-up
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        samples = 0
        for _ in range(args.steps):
            samples += step()
        dt = time.perf_counter() - t0
    value = samples / dt / 1e6
    sample_desc = (f"per step {procs} processes x {nfr} consecutive frames of {cfg.name} (forward of all frames + "
                   f"inverse of the interior half), numpy fp64, one process per core, BLAS/FFT threads 1")
    line = {
        "impl": "reference", "metric": "SST fwd+inverse input Msamples/s", "value": value, "unit": "Msamples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[cfg.name], "sample_frames_per_process": nfr},
        "cpu_baseline": {"value": value, "unit": "Msamples/s", "cores": procs, "cpu_model": model,
                         "kind": "oracle", "sample": sample_desc},
        "e2e": {"value": value, "unit": "Msamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_REF_CACHE = {}


def _ref_step_worker(name, nfr, wid):
    key = (name, nfr, wid)
    if key not in _REF_CACHE:
        _REF_CACHE[key] = _oracle_setup(name, nfr, cfg_f0(name, wid))
    O, cfg, xl, g, gd, c, gamma = _REF_CACHE[key]
    return _oracle_step(O, cfg, xl, g, gd, c, gamma, nfr)


def cpu_baseline(cfg, seconds_target=12.0):
    """Oracle timed on bounded samples of the workload (rank 0, N=1 only): single process and all
    cores (one process per core), each for about ``seconds_target`` s of 128-frame chunks, plus the
    relative-gamma pre-pass on its own; Msamples/s = frames * H_t / time."""
    O, cfg_, xl, g, gd, c, gamma = _oracle_setup(cfg.name, 128)
    nfr = 128
    done = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds_target:
        done += _oracle_step(O, cfg, xl, g, gd, c, gamma, nfr)
    dt = time.perf_counter() - t0
    single = done / dt / 1e6
    cores, model = host_info()
    allc, procs = oracle_all_core(cfg.name, nfr, seconds_target, cores)
    pre = oracle_gamma_prepass(cfg.name, nfr, min(5.0, seconds_target))
    return {"value": allc, "unit": "Msamples/s", "cores": procs, "cpu_model": model, "kind": "oracle",
            "single_core_value": single, "gamma_prepass_single_core": pre,
            "sample": f"{cfg.name}: chunks of {nfr} consecutive frames (forward + inverse of each chunk's interior "
                      f"half), numpy fp64; value = {procs} processes (one per core, BLAS/FFT threads 1) for "
                      f"{seconds_target:.0f} s; single_core_value = one process for {dt:.1f} s ({done // cfg.hop} "
                      f"frames); gamma_prepass_single_core = the relative-gamma max|S| pre-pass alone, one process"}


# ------------------------------------------------------------------------------------- our arm
def measure_extras(P, plan, cfg, x, T, y, stream, ev, reps=5):
    """SURVEY §8(f) rows built beyond the hot path, timed outside the step (CUDA events, after one
    warm-up): f2 plain STFT synthesis (sst_stft + sst_istft, Eq. 10-11) and f4 Renyi entropy
    (Eq. 32) on this workload; f1 ridge DP + Eq. 15 retrieval on configs[0] (C1, H_t = 1: the
    ridge DP is sequential over frames, one CTA)."""
    import torch

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    out = {}
    S, Sd = plan.stft(x)
    t_stft = timed(lambda: plan.stft(x))
    del Sd
    t_istft = timed(lambda: plan.istft(S, out=y))
    K = cfg.nfft // 2 + 1
    out["f2_stft_ms"] = t_stft
    out["f2_istft_ms"] = t_istft
    out["f2_istft_gbs"] = (cfg.frames * K * 8 + cfg.N * 4) / (t_istft * 1e-3) / 1e9
    del S
    t_ren = timed(lambda: plan.renyi(T))
    out["f4_renyi_ms"] = t_ren
    out["f4_renyi_gbs"] = cfg.frames * cfg.bins * 8 / (t_ren * 1e-3) / 1e9
    # f1 on C1 (H_t = 1)
    from gen import generate, get_config
    c1 = get_config("C1")
    x1 = torch.from_numpy(generate(c1)).to(x.device)
    g1, _ = P.gaussian_window(c1.L, c1.sigma)
    p1 = P.Plan(c1.N, c1.fs, c1.L, c1.sigma, c1.hop, c1.nfft, c1.f1, c1.f2, c1.zoom,
                gamma=1e-6 * float(np.sum(g1)) * float(x1.abs().max()), device=x.device.index)
    T1 = p1.forward(x1)

    def ridge_and_mode():
        paths = p1.ridges(T1, 0.01, 2)
        p1.mode_full(T1, paths[0].contiguous(), 40)
    out["f1_ridge2_mode_c1_ms"] = timed(ridge_and_mode)
    out["f1_config"] = f"C1: F={c1.frames}, B={c1.bins}, 2 ridges (lambda 0.01) + Eq. 15 retrieval"
    p1.close()
    # f3: the paper's §5.2 Fig. 16(c) shape (N_f = 2^15, H_t = 667, 1200-1400 Hz) on the synthetic
    # stand-in, through the multi-pass large-N_f path
    from gen.signals import s52_milling
    x5 = torch.from_numpy(s52_milling()).to(x.device)
    p5 = P.Plan(573440, 10240.0, 8193, 1024.0, 667, 32768, 1200.0, 1400.0, 1, gamma=1e-6, device=x.device.index)
    T5 = torch.empty((p5.frames, p5.bins), dtype=torch.complex64, device=x.device)
    y5 = torch.empty(573440, dtype=torch.float32, device=x.device)
    out["f3_s52_forward_ms"] = timed(lambda: p5.forward(x5, out=T5))
    out["f3_s52_inverse_ms"] = timed(lambda: p5.inverse(T5, out=y5))
    out["f3_config"] = f"§5.2 Fig. 16(c) shape: N=573440, N_f=32768, H_t=667, F={p5.frames}, B={p5.bins} (paper: 0.8 s MATLAB)"
    p5.close()
    return out


def store_peak_gbs(dev, gib=4, reps=5):
    """Write-only HBM bandwidth on this GPU (C5's forward traffic is ~all writes): a
    `fill_` of a buffer larger than L2, CUDA events, best of `reps`."""
    import torch
    buf = torch.empty(gib << 28, dtype=torch.float32, device=dev)
    buf.fill_(1.0)
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        buf.fill_(2.0)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    del buf
    torch.cuda.empty_cache()
    return (gib << 30) / (best * 1e-3) / 1e9


def measure_leg(P, D, name, world, rank, local, dev, steps, warmup, chunk_frames, hbm_gbs, store_gbs):
    """A SURVEY §8(d) leg on a fixed record, time-sharded over the ranks (strong scaling): C4 (forward,
    T resident) or C5 (forward + inverse; frames processed in chunks of ``chunk_frames`` with one
    reused T buffer -- its 256 GiB plane never exists whole).  Device time, max over ranks; the
    forward share is timed by forward-only passes."""
    import torch
    cfg = get_config(name)
    c = cfg.L // 2
    sh = D.shard(cfg.N, cfg.hop, cfg.L, c, world, rank)
    x_host = generate(cfg, sh.span_lo, sh.span_hi)
    g, gd = P.gaussian_window(cfg.L, cfg.sigma)
    gamma = 1e-6 * float(np.sum(g)) * D.max_over_ranks(float(np.abs(x_host).max()), dev)   # reading R6
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom, gamma=gamma,
                  device=local)
    x = torch.from_numpy(x_host).to(dev)
    del x_host
    run = D.ShardedRun(plan, sh, x, inverse=cfg.inverse, chunk_frames=chunk_frames if cfg.inverse else 0)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, k):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return D.max_over_ranks(a.elapsed_time(b) / k, dev)

    step_ms = timed(run.step, steps)
    fwd_ms = timed(lambda: run.step(forward_only=True), steps) if cfg.inverse else step_ms
    fwd_fl, inv_fl, fwd_b, inv_b = algorithmic_counts(cfg)
    F = cfg.frames
    out = {"workload": WORKLOAD_DESC[name], "ms_per_step": step_ms, "fwd_ms": fwd_ms,
           "msamples_per_s": cfg.N / (step_ms * 1e-3) / 1e6, "tf_coeffs_per_s": F * cfg.bins / (step_ms * 1e-3),
           "fwd_hbm_gbs": F * fwd_b / (fwd_ms * 1e-3) / 1e9 / world,
           "fwd_hbm_frac": F * fwd_b / (fwd_ms * 1e-3) / 1e9 / world / hbm_gbs,
           "fwd_fp32_frac": F * fwd_fl / (fwd_ms * 1e-3) / 1e12 / world / (148 * 128 * 2 * 1.965e9 / 1e12),
           "chunk_frames": run.chunk, "T_chunk_gib": run.chunk * cfg.bins * 8 / 2 ** 30,
           "launches_per_step": run.launches_per_step, "r23": plan.counters()}
    if cfg.inverse:
        inv_ms = step_ms - fwd_ms
        out.update({"inv_ms": inv_ms, "inv_hbm_gbs": F * inv_b / (inv_ms * 1e-3) / 1e9 / world,
                    "inv_hbm_frac": F * inv_b / (inv_ms * 1e-3) / 1e9 / world / hbm_gbs,
                    "inv_fp32_frac": F * inv_fl / (inv_ms * 1e-3) / 1e12 / world / (148 * 128 * 2 * 1.965e9 / 1e12)})
    if store_gbs:
        out["fwd_frac_of_store_peak"] = out["fwd_hbm_gbs"] / store_gbs
    del run, x
    plan.close()
    torch.cuda.empty_cache()
    return out


def run_ours(args, cfg_base):
    import torch
    import torch.distributed as dist

    import paper_2003_07065_b200 as P
    from paper_2003_07065_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = cfg_base                                  # strong scaling: one fixed record over the ranks
    g, gd = P.gaussian_window(cfg.L, cfg.sigma)
    c = cfg.L // 2
    sh = D.shard(cfg.N, cfg.hop, cfg.L, c, world, rank)

    x_host = generate(cfg, sh.span_lo, sh.span_hi)
    gamma = 1e-6 * float(np.sum(g)) * D.max_over_ranks(float(np.abs(x_host).max()), dev)   # reading R6
    plan = P.Plan(cfg.N, cfg.fs, cfg.L, cfg.sigma, cfg.hop, cfg.nfft, cfg.f1, cfg.f2, cfg.zoom,
                  gamma=gamma, device=local)
    x = torch.from_numpy(x_host).to(dev)
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    if world == 1:
        T = torch.empty((sh.frames, plan.bins), dtype=torch.complex64, device=dev)
        y = torch.empty(cfg.N, dtype=torch.float32, device=dev)
        run = None
    else:
        run = D.ShardedRun(plan, sh, x, inverse=True)    # forward, accumulate, NCCL seams, finalize

    def step(record=None):
        e0, e1, e2 = (ev(), ev(), ev()) if record is not None else (None, None, None)
        if e0: e0.record(stream)
        if run is None:
            plan.forward(x, out=T)
            if e1: e1.record(stream)
            plan.inverse(T, out=y)
        else:
            run.step()
            if e1: e1.record(stream)
        if e2: e2.record(stream)
        if record is not None:
            record.append((e0, e1, e2))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    recs = []
    with ClockSampler(local) as clk:
        t_start, t_end = ev(), ev()
        t_start.record(stream)
        for _ in range(args.steps):
            step(recs)
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms_local = t_start.elapsed_time(t_end)
    per_step = sorted(a.elapsed_time(cc) for a, _, cc in recs)      # median and min too
    step_stats = {"median_ms": per_step[len(per_step) // 2], "min_ms": per_step[0], "max_ms": per_step[-1]}
    ms_total = D.max_over_ranks(ms_local, dev)
    ms_step = ms_total / args.steps
    if run is None:
        fwd_ms = sum(a.elapsed_time(b) for a, b, _ in recs) / len(recs)
        inv_ms = sum(b.elapsed_time(cc) for _, b, cc in recs) / len(recs)
    else:
        # forward share of a rank's step from forward-only passes (after the timed region)
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(3):
            run.step(forward_only=True)
        b.record(stream)
        torch.cuda.synchronize()
        fwd_ms = a.elapsed_time(b) / 3
        inv_ms = max(0.0, ms_local / args.steps - fwd_ms)
    fwd_ms = D.max_over_ranks(fwd_ms, dev)
    inv_ms = D.max_over_ranks(inv_ms, dev)
    value = cfg.N / (ms_step * 1e-3) / 1e6
    coeffs_per_s = cfg.frames * cfg.bins / (ms_step * 1e-3)

    # ---- end to end through the public API with host buffers (pinned), per step
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x_host).pin_memory()
        own = sh.own_hi - sh.own_lo
        yh = torch.empty(own, dtype=torch.float32).pin_memory()
        rt = graph = None
        if world == 1:
            # host -> host through the public pipeline helper: chunked H2D / forward / inverse /
            # finalize / D2H on three streams, transfers overlapped with the kernels
            from paper_2003_07065_b200.pipeline import RoundTrip
            rt = RoundTrip(plan, chunks=args.e2e_chunks)
            rt.run(xh, yh, T)
            torch.cuda.synchronize()
            # one CUDA graph per round trip: no per-chunk host work inside the timed region
            graph = rt.capture(xh, yh, T) if not args.e2e_no_graph else None
        for it in range(args.warmup + args.steps):
            if it == args.warmup:
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                a0 = ev()
                a0.record(stream)
            if rt is not None:
                if graph is not None:
                    graph.replay()
                else:
                    rt.run(xh, yh, T)
                continue
            x.copy_(xh, non_blocking=True)
            own_y = run.step()
            yh.copy_(own_y, non_blocking=True)
        a1 = ev()
        a1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = D.max_over_ranks(a0.elapsed_time(a1), dev) / args.steps
        e2e = {"value": cfg.N / (e2e_ms * 1e-3) / 1e6, "unit": "Msamples/s",
               "h2d_bytes_per_step": int(D.max_over_ranks(xh.numel() * 4, dev) * world),
               "d2h_bytes_per_step": int(cfg.N * 4), "ms_per_step": e2e_ms}

    hbm_gbs, sm_max_mhz, peak_src = _peaks()
    fwd_fl, inv_fl, fwd_b, inv_b = algorithmic_counts(cfg)
    nfr_rank = sh.frames
    fp32_peak = 148 * 128 * 2 * sm_max_mhz * 1e6 / 1e12   # TFLOP/s
    fwd_tf = fwd_fl * nfr_rank / (fwd_ms * 1e-3) / 1e12
    inv_tf = inv_fl * nfr_rank / (inv_ms * 1e-3) / 1e12 if inv_ms > 0 else 0.0
    fwd_gbs = fwd_b * nfr_rank / (fwd_ms * 1e-3) / 1e9
    inv_gbs = inv_b * nfr_rank / (inv_ms * 1e-3) / 1e9 if inv_ms > 0 else 0.0
    # the two calls tie within ~0.5 % on C3 (8.85 vs 8.83 ms): a tie (< 2 %) reports the forward, the
    # one further from its roofline, so that the headline fraction does not flip from run to run
    dom = "forward" if fwd_ms >= 0.98 * inv_ms else "inverse"
    ach = fwd_tf if dom == "forward" else inv_tf
    traffic = {"bytes": None, "source": "not measured (N > 1 or --no-traffic)"}
    roofline = {"bound": "alu", "kernel": f"sst_{dom}", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": ach / fp32_peak, "traffic": None,
                "peak_source": f"derived: {FP32_PEAK_NOTE}",
                "hbm": {"forward_gbs": fwd_gbs, "inverse_gbs": inv_gbs, "peak_gbs": hbm_gbs,
                        "forward_frac": fwd_gbs / hbm_gbs, "inverse_frac": inv_gbs / hbm_gbs,
                        "peak_source": f"{peak_src} copy bandwidth (MEASURED_PEAKS.json)"},
                "alu": {"forward_tflops": fwd_tf, "inverse_tflops": inv_tf,
                        "forward_frac": fwd_tf / fp32_peak, "inverse_frac": inv_tf / fp32_peak},
                "per_frame": {"fwd_flops": fwd_fl, "inv_flops": inv_fl, "fwd_bytes": fwd_b, "inv_bytes": inv_b}}
    r23 = plan.counters()
    launches_per_step = (3 + 2) if run is None else run.launches_per_step
    extras = None
    if world == 1 and not args.no_extras:
        extras = measure_extras(P, plan, cfg, x, T, y, stream, ev)
    del x
    if run is None:
        del T, y
    else:
        del run
    plan.close()
    torch.cuda.empty_cache()
    if world == 1 and not args.no_traffic:
        traffic = measure_traffic(cfg_base.name, dom, nfr_rank)
    roofline["traffic"] = traffic["bytes"]
    roofline["traffic_source"] = traffic["source"]
    if traffic["bytes"]:
        roofline["traffic_vs_algorithmic"] = traffic["bytes"] / ((fwd_b if dom == "forward" else inv_b) * nfr_rank)
    legs = {}
    store = store_peak_gbs(dev) if args.legs not in ("", "none", "''") else None
    for name in [s for s in args.legs.split(",") if s and s not in ("none", "''")]:
        legs[name] = measure_leg(P, D, name, world, rank, local, dev, args.leg_steps, 3, args.c5_chunk, hbm_gbs, store)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg_base, args.cpu_seconds)
    if rank == 0:
        line = {
            "metric": "SST fwd+inverse input Msamples/s", "value": value, "unit": "Msamples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC[cfg_base.name], "N": cfg.N, "N_per_gpu": sh.frames * cfg.hop,
                       "frames": cfg.frames, "bins": cfg.bins, "T_bytes": cfg.frames * cfg.bins * 8,
                       "parallelism": f"time-shard x{world}",
                       "l2": "inputs larger than L2 (T = %.1f GiB written and read per step)" % (
                           cfg.frames * cfg.bins * 8 / 2 ** 30)},
            "tf_coeffs_per_s": coeffs_per_s,
            "fwd_ms": fwd_ms, "inv_ms": inv_ms, "step_ms_stats": step_stats,
            "roofline": roofline,
            "r23": r23,
            "legs": legs or None,
            "hbm_store_gbs": store,
            "cpu_baseline": cpu,
            "extras": extras,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4)
    ap.add_argument("--e2e-no-graph", action="store_true", help="launch the e2e round trip chunk by chunk")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--legs", default="C4,C5", help="extra fixed-record legs (strong scaling), 'none' for none")
    ap.add_argument("--leg-steps", type=int, default=3)
    ap.add_argument("--c5-chunk", type=int, default=1 << 20, help="C5 frames per chunk (T buffer 16 GiB)")
    ap.add_argument("--ref-frames", type=int, default=512)
    ap.add_argument("--ref-procs", type=int, default=0, help="reference arm processes (default: every core)")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic child run")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.traffic_probe:
        traffic_probe(args.workload)
        return
    if args.warmup < 3:
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    cfg = get_config(args.workload)
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, cfg)
        return
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
