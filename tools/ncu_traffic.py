"""Write profiles/traffic.json (or OUT) from an ncu --set full capture of bench.py's kernels:
    python tools/ncu_traffic.py rep.ncu-rep WORKLOAD FRAMES [OUT]"""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, workload, frames = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
path = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
seen = set()
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"]
    kern = "forward" if "fwd_kernel" in name else "inverse" if ("inv_kernel" in name or "inv_nb_kernel" in name) else None
    if kern is None or kern in seen:   # first launch per kernel: later ones are list-mode R23 repair launches
        continue
    seen.add(kern)
    def mb(k):
        v = float(d[k]); u = units[h.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    t.setdefault(workload, {})[kern] = {"frames": frames, "dram_bytes": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                                        "dram_read": mb("dram__bytes_read.sum"), "dram_write": mb("dram__bytes_write.sum"),
                                        "kernel": name, "report": os.path.basename(rep)}
json.dump(t, open(path, "w"), indent=1)
print(json.dumps(t, indent=1))
