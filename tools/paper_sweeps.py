"""The paper's §3 experiment grid on the Eq. 30 signal, run through this library on the GPU
("Table 1-2 and Fig. 3/6/7 sweep presets at desk scale").  Context, not
targets: the paper's numbers are MATLAB on an i5-8250, and its f_w / noise realisation
for the SNR figures are unstated.

  Table 1: SST time, H_t in {1, 20, 40} x H_f in {1, 2}, full band.
  Table 2: full band vs selective [0, 80] Hz at H_t = 20, H_f in {1, 2}.
  Fig. 3: Renyi entropy (alpha = 3, Eq. 32) over an H_t x H_f grid.
  Fig. 6: output SNR (Eq. 33) of the three modes vs H_t = H_f, 5 dB noise, retrieved
                        with ridge (R22) + zone (f_w = 10 Hz) + the downsampled inverse (Eq. 25-26);
                        the full-rate reference through Eq. 15 (paper: 14.98 / 14.57 / 12.36 dB).
  Fig. 7: output SNR vs half bandwidth f_w at H_t = H_f = 4, 0 and 5 dB.

    python tools/paper_sweeps.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen.signals import eq30_noisy  # noqa: E402

FS, N = 1024.0, 8192
SIGMA = 0.03 * FS                    # sigma = 0.03 s in samples
L = 2 * int(np.ceil(3 * SIGMA)) + 1  # truncated at +-3 sigma (length unstated)
DEV = torch.device("cuda", 0)


def noisy(snr_db, seed=0):
    return eq30_noisy(snr_db, seed, N, FS)


def plan_for(hop, hf, f2=FS / 2, zoom=1):
    nfft = N // hf
    return P.Plan(N, FS, L, SIGMA, hop, nfft, 0.0, f2, zoom, gamma=1e-6, device=0)


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def snr_db(ref, est):
    return float(10 * np.log10(np.sum(ref ** 2) / np.sum((ref - est) ** 2)))


LAM = 0.1   # ridge smoothness per squared fine bin (R22); 0.01 lets the x2 / x3 ridges swap at 5 dB


def true_paths(plan):
    """zone centres from the true IFs of Eq. 31, for the 'ideal zone' variant."""
    from gen.signals import eq30_true_ifs
    dfz = FS / plan.layout["nfft"] / plan.layout["zoom"]
    fr = np.arange(plan.frames) * plan.layout["hop"]
    return [torch.from_numpy(np.round(f[fr] / dfz).astype(np.int32)).to(DEV) for f in eq30_true_ifs(N, FS)]


def modes(plan, T, fw_hz, count=3):
    """ridges (R22) -> zones of half width f_w -> zone-masked inverse; modes ordered by mean IF."""
    dfz = FS / plan.layout["nfft"] / plan.layout["zoom"]
    half = int(round(fw_hz / dfz))
    paths = plan.ridges(T, LAM, count)
    out = []
    for q in range(count):
        p = paths[q].contiguous()
        out.append((float(p.float().mean()) * dfz, plan.retrieve_mode(T, p, half).cpu().numpy()))
    return [m for _, m in sorted(out, key=lambda t: t[0])]       # x1 (50 Hz) < x2 < x3 in mean IF


def main():
    res = {"signal": "Eq. 30 (P:L228-236), N = 8192, fs = 1024 Hz, sigma = 30.72 samples, L = %d" % L,
           "note": "B200 timings of this library; the paper's are MATLAB R2017b on an i5-8250 (P:L226)"}
    x, comps = noisy(200.0)                                    # effectively noiseless for timing
    xd = torch.from_numpy(x).to(DEV)
    # Table 1 + Fig. 3 grid
    t1 = {}
    for hf in (1, 2):
        for hop in (1, 20, 40):
            pl = plan_for(hop, hf)
            T = torch.empty((pl.frames, pl.bins), dtype=torch.complex64, device=DEV)
            ms = timed(lambda: pl.forward(xd, out=T))
            t1[f"Ht{hop}_Hf{hf}"] = {"sst_ms": ms, "paper_s": {(1, 1): 10.29, (20, 1): 0.50, (40, 1): 0.24,
                                                                (1, 2): 5.37, (20, 2): 0.27, (40, 2): 0.13}[(hop, hf)],
                                     "renyi": float(pl.renyi(T)[2])}
            pl.close()
    res["table1"] = t1
    # Table 2: full band vs selective [0, 80] Hz, H_t = 20
    t2 = {}
    for hf in (1, 2):
        for name, f2 in (("full", FS / 2), ("sel_0_80", 80.0)):
            pl = plan_for(20, hf, f2=f2)
            T = torch.empty((pl.frames, pl.bins), dtype=torch.complex64, device=DEV)
            t2[f"{name}_Hf{hf}"] = {"sst_ms": timed(lambda: pl.forward(xd, out=T)), "bins": pl.bins}
            pl.close()
    res["table2"] = t2
    # Fig. 3: Renyi entropy grid
    f3 = {}
    for hop in (1, 10, 20, 40, 60):
        for hf in (1, 2, 4, 8, 16, 32):
            pl = plan_for(hop, hf)
            f3[f"Ht{hop}_Hf{hf}"] = float(pl.renyi(pl.forward(xd))[2])
            pl.close()
    res["fig3_renyi"] = f3
    # Fig. 6: output SNR vs H_t = H_f, 5 dB
    x5, comps = noisy(5.0, seed=1)
    x5d = torch.from_numpy(x5).to(DEV)
    f6 = {}
    for h in (2, 4, 8, 16, 32):
        pl = plan_for(h, h)
        T = pl.forward(x5d)
        ms = modes(pl, T, 10.0)
        f6[f"Ht{h}_Hf{h}"] = [snr_db(c, m) for c, m in zip(comps, ms)]
        half = int(round(10.0 / (FS / pl.layout["nfft"])))
        f6[f"Ht{h}_Hf{h}_true_if_zone"] = [snr_db(c, pl.retrieve_mode(T, p, half).cpu().numpy())
                                           for c, p in zip(comps, true_paths(pl))]
        pl.close()
    # full-rate reference through Eq. 15 (H_t = H_f = 1)
    pl = plan_for(1, 1)
    T = pl.forward(x5d)
    paths = pl.ridges(T, LAM, 3)
    dfz = FS / N
    hw = int(round(10.0 / dfz))
    full = sorted(((float(paths[q].float().mean()) * dfz, pl.mode_full(T, paths[q].contiguous(), hw).cpu().numpy())
                   for q in range(3)), key=lambda t: t[0])
    f6["full_sst_eq15"] = [snr_db(c, m) for c, (_, m) in zip(comps, full)]
    f6["full_sst_eq15_true_if_zone"] = [snr_db(c, pl.mode_full(T, p, hw).cpu().numpy())
                                        for c, p in zip(comps, true_paths(pl))]
    f6["paper_full_sst_eq15"] = [14.98, 14.57, 12.36]
    pl.close()
    res["fig6_snr_db"] = f6
    # Fig. 7: SNR vs f_w at H_t = H_f = 4
    f7 = {}
    for snr in (0.0, 5.0):
        xs, comps = noisy(snr, seed=2)
        xsd = torch.from_numpy(xs).to(DEV)
        pl = plan_for(4, 4)
        T = pl.forward(xsd)
        for fw in (2.0, 5.0, 10.0, 20.0, 30.0):
            f7[f"in{int(snr)}dB_fw{int(fw)}"] = [snr_db(c, m) for c, m in zip(comps, modes(pl, T, fw))]
        pl.close()
    res["fig7_snr_db"] = f7
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "paper_sweeps.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
