"""CUDA-event timings of the paper's §5.2 chatter analysis shapes through the library's
multi-pass large-N_f path, on the synthetic stand-in gen.signals.s52_milling (not the dataset).
Context, not targets: the paper's 0.8 s / 3 s are MATLAB on an i5-8250 "after 20 averages".

    python tools/s52_timing.py [out.json]
    python tools/s52_timing.py --once     # one forward + one inverse of the Fig. 16(c) shape (for ncu)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen.signals import s52_milling  # noqa: E402

N, FS, SIGMA, L = 573440, 10240.0, 1024.0, 8193
SHAPES = {
    "fig16c_chatter_Ht667_1200_1400": dict(hop=667, f1=1200.0, f2=1400.0, zoom=1, paper_s=0.8),
    "fig16e_spindle_Ht200_630_640_z20": dict(hop=200, f1=630.0, f2=640.0, zoom=20, paper_s=3.0),
    "fig17_recon_Ht667_1300_1400": dict(hop=667, f1=1300.0, f2=1400.0, zoom=1, paper_s=None),
}


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def once():
    x = torch.from_numpy(s52_milling(52, N, FS)).cuda()
    s = SHAPES["fig16c_chatter_Ht667_1200_1400"]
    pl = P.Plan(N, FS, L, SIGMA, s["hop"], 32768, s["f1"], s["f2"], s["zoom"], gamma=1e-6, device=0)
    pl.inverse(pl.forward(x))
    torch.cuda.synchronize()


def main():
    if "--once" in sys.argv:
        return once()
    x = torch.from_numpy(s52_milling(52, N, FS)).cuda()
    res = {"signal": "gen.signals.s52_milling (synthetic stand-in), N = 573440, fs = 10240 Hz, sigma = 0.1 s, "
                     "L = 8193, N_f = 2^15", "note": "20-call averages, CUDA events"}
    for name, s in SHAPES.items():
        pl = P.Plan(N, FS, L, SIGMA, s["hop"], 32768, s["f1"], s["f2"], s["zoom"], gamma=1e-6, device=0)
        T = torch.empty((pl.frames, pl.bins), dtype=torch.complex64, device="cuda")
        y = torch.empty(N, dtype=torch.float32, device="cuda")
        c0 = pl.counters()
        pl.forward(x, out=T)
        c1 = pl.counters()
        fwd = timed(lambda: pl.forward(x, out=T))
        inv = timed(lambda: pl.inverse(T, out=y))
        res[name] = {"frames": pl.frames, "bins": pl.bins, "forward_ms": fwd, "inverse_ms": inv,
                     "r23_redecided_per_frame": (c1["redecided"] - c0["redecided"]) / pl.frames,
                     "r23_changed_per_frame": (c1["changed"] - c0["changed"]) / pl.frames,
                     "paper_sst_s": s["paper_s"]}
        pl.close()
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "s52_timing.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
