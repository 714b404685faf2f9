import torch
n = 1024**3
xs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2)]
ss = [torch.cuda.Stream() for _ in range(3)]
def run(k, d2h=False):
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            ds[i].copy_(xs[i], non_blocking=True)
    if d2h:
        with torch.cuda.stream(ss[2]):
            xs[1].copy_(ds[1], non_blocking=True)
for k, d2h in ((1, False), (2, False), (1, True)):
    run(k, d2h); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(k, d2h); torch.cuda.synchronize(); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print("h2d streams", k, "with d2h" if d2h else "", round(k * n / (ms * 1e-3) / 1e9, 1), "GB/s h2d", round(ms, 2), "ms")
