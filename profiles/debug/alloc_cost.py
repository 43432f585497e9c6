import time, torch
torch.cuda.init()
x = []
for shape, kw in (((3, 1080, 1440, 512), dict(device="cuda")), ((16,), dict(dtype=torch.int64, pin_memory=True)),
                  ((1080, 1440), dict(dtype=torch.uint8, pin_memory=True)), ((3, 1080, 1440), dict(dtype=torch.float64, device="cuda"))):
    ts = []
    for i in range(6):
        t = time.perf_counter(); a = torch.empty(shape, **kw); ts.append(time.perf_counter() - t)
        x.append(a)
        if len(x) > 2: x.pop(0)
    print(shape, kw.get("pin_memory", False), [f"{1e6*v:.0f}us" for v in ts])
