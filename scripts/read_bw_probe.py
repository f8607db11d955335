import torch, time
x = torch.randn(2**30, dtype=torch.bfloat16, device='cuda')  # 2 GiB
y = torch.empty(64, dtype=torch.float32, device='cuda')
for f,name in ((lambda: x.sum(dtype=torch.float32), 'sum'), (lambda: torch.amax(x.view(2**20, 1024), dim=1), 'amax_rows'), (lambda: x.view(torch.int32).view(-1, 4096).sum(dim=1), 'isum')):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(name, round(best*1e3,1), 'us', round(2**31/best/1e9, 1), 'TB/s')
