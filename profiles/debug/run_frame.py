"""Run a few config-C frames (features decoded, one query) -- for timeline / profiler captures."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
from paper_2507_07136_b200 import synthetic, _native as N
from paper_2507_07136_b200.device import QuerySpec, device_scene

n, W, H = 2_000_000, 1440, 1080
scene = synthetic.make_scene(n)
cam = synthetic.make_camera(W, H)
qv, canon = synthetic.make_query()
eng = device_scene(scene).engine
fused = bool(N.load().sf_decode_fused(3, 64, 4, 512))
out = eng.allocate(W, H, (0, 1, 2), coeff_map=not fused, features=True, query=True)
spec = QuerySpec(qv, canon, 11, -1, 0.5)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    eng.run(cam, (0, 1, 2), out, query=spec, timing=True)
    torch.cuda.synchronize()
    print("stage ms", out.stage_ms(), "blend", out.blend_ms())
