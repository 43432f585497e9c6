"""Throughput of config-C frames run serially vs alternating over two streams (two engines,
double-buffered workspaces/outputs); development experiment."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
from paper_2507_07136_b200 import synthetic, _native as N
from paper_2507_07136_b200.device import QuerySpec, device_scene, FrameEngine

n, W, H = 2_000_000, 1440, 1080
scene = synthetic.make_scene(n)
cam = synthetic.make_camera(W, H)
qv, canon = synthetic.make_query()
ds = device_scene(scene)
engs = [ds.engine, FrameEngine(ds)]
lv = (0, 1, 2)
outs = [e.allocate(W, H, lv, coeff_map=False, features=True, query=True) for e in engs]
spec = QuerySpec(qv, canon, 11, -1, 0.5)
qdev = (torch.from_numpy(qv).cuda(), torch.from_numpy(canon).cuda())
for e, o in zip(engs, outs):
    e.run(cam, lv, o, query=spec, qdev=qdev)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
for prio in ((0, 0), (0, -1)):
    streams = [torch.cuda.Stream(priority=prio[0]), torch.cuda.Stream(priority=prio[1])]
    for mode in ("serial", "two-stream"):
        K = 20
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for s in streams:
            s.wait_event(ev0)
        for k in range(K):
            i = k % 2 if mode == "two-stream" else 0
            with torch.cuda.stream(streams[i]):
                engs[i].enqueue(cam, lv, outs[i], query=spec, qdev=qdev)
        for s in streams:
            e = torch.cuda.Event(); e.record(s); torch.cuda.current_stream().wait_event(e)
        ev1.record()
        torch.cuda.synchronize()
        print(prio, mode, f"{K / (ev0.elapsed_time(ev1) / 1e3):.1f} FPS")
