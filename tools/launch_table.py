"""Summarise an ncu launch list (gpu__time_duration.sum CSV of `bench.py`) into the profiles/ table:
the device-timed step (first 3 (W) + K whole-record launches per kernel) and the e2e leg (the rest).

    python tools/launch_table.py gpurun_out/launches_TAG.csv bench_TAG.json > profiles/rN_launches_c3.txt
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    seq.append((r[ki], v * scale))
bench = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
# the step ends at the last whole-record inverse (plus its seam launch)
inv_max = max(ms for k, ms in seq if ("inv_kernel" in k or "inv_nb_kernel" in k))
last_whole = max(i for i, (k, ms) in enumerate(seq) if ("inv_kernel" in k or "inv_nb_kernel" in k) and ms > 0.5 * inv_max)
step, e2e = seq[:last_whole + 2], seq[last_whole + 2:]


def table(part):
    acc = collections.OrderedDict()
    for k, ms in part:
        n, t = acc.get(k, (0, 0.0))
        acc[k] = (n + 1, t + ms)
    tot = sum(t for _, t in acc.values())
    return [f"{k} | {n} | {t / n:.3f} | {100 * t / tot:.1f}%" for k, (n, t) in acc.items()]


print("# ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras` (C3 workload, --legs none)")
print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
print("## device-timed step (whole-record forward + inverse): kernel | launches | mean ms | share")
print("\n".join(table(step)))
if bench:
    f, i = bench["fwd_ms"], bench["inv_ms"]
    print(f"# bench run of the same build (no ncu): fwd {f:.3f} ms, inv {i:.3f} ms per step (CUDA events) -> "
          f"fwd share {100 * f / (f + i):.1f}%")
print("## e2e leg (pipeline.RoundTrip: --e2e-chunks frame chunks per step (CUDA graph replay), forward / inverse_accumulate / finalize per chunk)")
print("\n".join(table(e2e)))
