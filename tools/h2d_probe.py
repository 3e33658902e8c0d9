import torch, time
n=256; WH=640*480
hd=torch.empty((n,WH),dtype=torch.float32,pin_memory=True); hc=torch.empty((n,WH*3),dtype=torch.uint8,pin_memory=True)
dd=torch.empty((n,WH),dtype=torch.float32,device='cuda'); dc=torch.empty((n,WH*3),dtype=torch.uint8,device='cuda')
s=torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for i in range(n):
            dd[i].copy_(hd[i], non_blocking=True); dc[i].copy_(hc[i], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    ms=e0.elapsed_time(e1); print('per-frame copies', ms, 'ms', n*WH*7/ms/1e6, 'GB/s')
    e0.record(s); dd.copy_(hd, non_blocking=True); dc.copy_(hc, non_blocking=True); e1.record(s)
    torch.cuda.synchronize(); ms=e0.elapsed_time(e1); print('one copy', ms, 'ms', n*WH*7/ms/1e6, 'GB/s')
