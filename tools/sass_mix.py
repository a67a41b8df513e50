"""Opcode mix of one kernel in a .so: python tools/sass_mix.py lib.so name_substring"""
import collections, re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
cur = None; funcs = collections.defaultdict(list)
for ln in out.split("\n"):
    m = re.search(r"Function : (\S+)", ln)
    if m: cur = m.group(1); continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", ln)
    if m and cur: funcs[cur].append(m.group(1))
for f, ins in funcs.items():
    if all(s in f for s in sys.argv[2:]):
        c = collections.Counter()
        for i in ins:
            t = i.split(); op = t[1] if t[0].startswith("@") else t[0]
            c[op.split(".")[0]] += 1
        print(f, len(ins)); print("  ", " ".join(f"{k}:{v}" for k, v in c.most_common(30)))
