timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_dist.py -q -rf > gpurun_out/pytest_next.log 2>&1; echo "exit $?" >> gpurun_out/pytest_next.log
timeout 600 python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import torch, numpy as np, time
import paper_2003_07065_b200 as P
from gen import generate, get_config
c1 = get_config('C1')
x1 = torch.from_numpy(generate(c1)).cuda()
g1, _ = P.gaussian_window(c1.L, c1.sigma)
p1 = P.Plan(c1.N, c1.fs, c1.L, c1.sigma, c1.hop, c1.nfft, c1.f1, c1.f2, c1.zoom, gamma=1e-6 * float(np.sum(g1)) * float(x1.abs().max()))
T1 = p1.forward(x1)
for lam in (0.01, 0.001, 0.0):
    p1.ridges(T1, lam, 2); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); p1.ridges(T1, lam, 2); b.record(); torch.cuda.synchronize()
    print('C1 2 ridges lambda', lam, a.elapsed_time(b), 'ms')
" > gpurun_out/ridge_time.log 2>&1
