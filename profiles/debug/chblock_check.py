"""Blend-kernel time (coefficient map only, config C) vs channels per CTA (SF_CH_BLOCK)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
from paper_2507_07136_b200 import synthetic
from paper_2507_07136_b200.device import device_scene
scene = synthetic.make_scene(2_000_000)
cam = synthetic.make_camera(1440, 1080)
eng = device_scene(scene).engine
out = eng.allocate(1440, 1080, (0, 1, 2), coeff_map=True, features=False, query=False)
for _ in range(2):
    eng.run(cam, (0, 1, 2), out, timing=True)
ts = []
for _ in range(5):
    eng.run(cam, (0, 1, 2), out, timing=True)
    ts.append(out.blend_ms())
print(os.environ.get("SF_CH_BLOCK"), "blend ms", sorted(ts)[2])
