"""Median blend-kernel time (k_blend<DEC> incl. the fused decode) of feature-splat
frames at a BASELINE config, from the frame's CUDA events.  Dev aid.

    python profiles/debug/blend_time.py [C] [--query]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np

import bench
from paper_2507_07136_b200 import synthetic
from paper_2507_07136_b200.device import QuerySpec, device_scene

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C"
query = "--query" in sys.argv
n_g, W, H = bench.CONFIGS[cfg]
scene = synthetic.make_scene(n_g)
cam = synthetic.make_camera(W, H)
qv, canon = synthetic.make_query()
eng = device_scene(scene).engine
levels = (0, 1, 2)
out = eng.allocate(W, H, levels, coeff_map=False, features=True, query=query)
spec = QuerySpec(qv, canon) if query else None
for _ in range(3):
    eng.run(cam, levels, out, timing=True, query=spec)
b, f = [], []
for _ in range(15):
    eng.run(cam, levels, out, timing=True, query=spec)
    b.append(out.blend_ms())
    f.append(sum(out.stage_ms()))
print(f"config {cfg} query={query}: blend kernel median {np.median(b):.3f} ms, frame (events) median {np.median(f):.3f} ms")
