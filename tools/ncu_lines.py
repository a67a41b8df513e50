"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
fname = ""
hdr = None
tot_inst = tot_samp = 0
stall_tot = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        inst = float(d["Instructions Executed"])
        samp = float(d["Warp Stall Sampling (All Samples)"])
    except Exception:
        continue
    tot_inst += inst
    tot_samp += samp
    stalls = {k: float(v) for k, v in d.items() if k.startswith("stall_") and v not in ("", "-")}
    for k, v in stalls.items():
        stall_tot[k] = stall_tot.get(k, 0) + v
    top3 = sorted(stalls.items(), key=lambda t: -t[1])[:3]
    out.append((samp, inst, fname, r[0], r[1][:90], top3))
print(f"total inst {tot_inst:,.0f}  samples {tot_samp:,.0f}")
print("stalls:", ", ".join(f"{k[6:]}={v/tot_samp*100:.1f}%" for k, v in sorted(stall_tot.items(), key=lambda t: -t[1])[:12]))
for samp, inst, f, ln, src, t3 in sorted(out, key=lambda t: -t[0])[:top]:
    print(f"{samp/tot_samp*100:5.1f}% smp {inst/tot_inst*100:5.1f}% inst {f}:{ln:>4} {src:90s} {' '.join(k[6:]+'='+str(int(v)) for k,v in t3)}")
