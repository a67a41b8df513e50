"""Summarise an `ncu --page source --csv --print-source sass` dump: instruction mix by opcode,
stall reasons overall, and the hottest instruction windows.
    python tools/ncu_sass.py dump.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
recs = []
for r in rows:
    if len(r) > 2 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 1 or not r[0].startswith("0x"):
        continue
    recs.append(dict(zip(hdr, r)))


def f(d, k):
    try:
        return float(d.get(k, "0") or 0)
    except ValueError:
        return 0.0


tot_i = sum(f(d, "Instructions Executed") for d in recs)
tot_s = sum(f(d, "Warp Stall Sampling (All Samples)") for d in recs)
print(f"warp instructions {tot_i:,.0f}  stall samples {tot_s:,.0f}")
op_i = collections.Counter()
op_s = collections.Counter()
for d in recs:
    src = d["Source"].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0].split(".")[0] if src else "?"
    op_i[op] += f(d, "Instructions Executed")
    op_s[op] += f(d, "Warp Stall Sampling (All Samples)")
print("opcode mix (share of warp instructions / of stall samples):")
for op, v in op_i.most_common(22):
    print(f"  {op:10s} {v / tot_i * 100:5.1f}%  {op_s[op] / max(tot_s, 1) * 100:5.1f}%")
st = collections.Counter()
for d in recs:
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            st[k[6:]] += f(d, k)
print("stalls:", ", ".join(f"{k}={v / max(tot_s, 1) * 100:.1f}%" for k, v in st.most_common(10)))
# shared-memory conflicts
wf = sum(f(d, "L1 Wavefronts Shared") for d in recs)
wfi = sum(f(d, "L1 Wavefronts Shared Ideal") for d in recs)
print(f"shared wavefronts {wf:,.0f} ideal {wfi:,.0f} (excess {100 * (wf - wfi) / max(wfi, 1):.1f}%)")
# hottest windows of 16 instructions
win = 16
scores = []
for i in range(0, len(recs), win):
    s = sum(f(d, "Warp Stall Sampling (All Samples)") for d in recs[i:i + win])
    scores.append((s, i))
for s, i in sorted(scores, reverse=True)[:top]:
    ops = " ".join(recs[j]["Source"].strip().split()[0] for j in range(i, min(i + win, len(recs))))
    print(f"{s / max(tot_s, 1) * 100:5.1f}% @{i:5d} {ops[:150]}")
