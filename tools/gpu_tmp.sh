NLIM=16777216 timeout 300 python tools/time_cfg.py C5 1 > gpurun_out/plain_k.log 2>&1 && \
NLIM=16777216 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv python tools/time_cfg.py C5 1 > gpurun_out/ncu_k.log 2>&1
python -c "
import torch
for dt in (torch.uint8, torch.float32, torch.float4_e2m1fn_x2 if hasattr(torch,'float4_e2m1fn_x2') else torch.int64):
    b = torch.empty(4<<30, dtype=torch.uint8, device='cuda').view(dt)
    b.zero_(); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); b.zero_(); e1.record(); torch.cuda.synchronize()
    print(dt, 'zero_', (4<<30)/e0.elapsed_time(e1)/1e6, 'GB/s')
    del b
" > gpurun_out/store_peak.log 2>&1
