"""Ridge DP on configs[0] (C1: F = 4096 frames, B = 2048 bins), for profiling: python tools/ridge_prof.py [lam]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2003_07065_b200 as P  # noqa: E402
from gen import generate, get_config  # noqa: E402

lam = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
c1 = get_config("C1")
x1 = torch.from_numpy(generate(c1)).cuda()
g1, _ = P.gaussian_window(c1.L, c1.sigma)
p1 = P.Plan(c1.N, c1.fs, c1.L, c1.sigma, c1.hop, c1.nfft, c1.f1, c1.f2, c1.zoom,
            gamma=1e-6 * float(np.sum(g1)) * float(x1.abs().max()))
T1 = p1.forward(x1)
E, fl = p1.ridge_emission(T1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
p1.ridge(E, fl, lam, 1, 3)                      # warm-up (module load, attributes)
for _ in range(2):
    a.record()
    p1.ridge(E, fl, lam, 1, 3)
    b.record()
    torch.cuda.synchronize()
    print(f"C1 one ridge DP lambda {lam}: {a.elapsed_time(b):.2f} ms")
