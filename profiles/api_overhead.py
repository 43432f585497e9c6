"""Host-side cost breakdown of one query_pipeline(features='eager') call (config C)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import synthetic, sparse_splat, device

scene = synthetic.make_scene(2_000_000); cam = synthetic.make_camera(1440, 1080)
qv, canon = synthetic.make_query(); qe = sf.QueryEmbedding('q', qv)
for _ in range(3):
    r = sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
torch.cuda.synchronize()
T = {}
orig_run = device.FrameEngine.run
orig_alloc = device.FrameEngine.allocate
def timed(name, f):
    def w(*a, **k):
        t = time.perf_counter(); out = f(*a, **k); torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t; return out
    return w
device.FrameEngine.run = timed('run(enqueue+sync)', orig_run)
device.FrameEngine.allocate = timed('allocate', orig_alloc)
n = 10
t0 = time.perf_counter()
for _ in range(n):
    r = sf.query_pipeline(scene, cam, qe, canon, features='eager', instrument=False, max_elements=1 << 40)
    m = r.mask
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f'per call {1e3*tot/n:.2f} ms')
for k, v in T.items(): print(f'  {k}: {1e3*v/n:.2f} ms')
# device-only frame for comparison
eng = device.device_scene(scene).engine
out = eng.allocate(1440, 1080, (0,1,2), coeff_map=False, features=True, query=True)
spec = device.QuerySpec(qv, canon, 11, -1, 0.5)
qdev = (torch.from_numpy(qv).cuda(), torch.from_numpy(canon).cuda())
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(n): eng.enqueue(cam, (0,1,2), out, query=spec, qdev=qdev)
torch.cuda.synchronize(); print(f'enqueue-only loop {1e3*(time.perf_counter()-t0)/n:.2f} ms/frame')
t0 = time.perf_counter()
for _ in range(n): eng.enqueue(cam, (0,1,2), out, query=spec, qdev=qdev)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f'host launch cost {1e3*(t1-t0)/n:.3f} ms/frame')
