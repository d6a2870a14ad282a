import torch, time
d = torch.empty(800*800*3, device="cuda"); h = torch.empty(800*800*3, pin_memory=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f in [("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))]:
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(name, f"{ms*1e3:.1f} us per 7.68 MB = {7.68e6/ms/1e6:.1f} GB/s")
