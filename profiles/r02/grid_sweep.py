"""Development aid: k_splat_tc time at config C for the grid size in SF_TC_GRID
(default: one CTA per SM).  Text-query frames (NC=4, fused decode) and feature
frames (no query), median of 7 event-timed frames each.

usage: SF_TC_GRID=74 python profiles/r02/grid_sweep.py
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2507_07136_b200 import synthetic  # noqa: E402
from paper_2507_07136_b200.device import QuerySpec, device_scene  # noqa: E402

scene = synthetic.make_scene(2000000)
cam = synthetic.make_camera(1440, 1080)
qv, canon = synthetic.make_query()
ds = device_scene(scene)
eng = ds.engine
levels = (0, 1, 2)
spec = QuerySpec(qv, canon, 11, -1, 0.5)
res = {}
for name, q in (("query", spec), ("features", None)):
    out = eng.allocate(1440, 1080, levels, coeff_map=False, features=True, query=q is not None)
    eng.run(cam, levels, out, query=q)
    ts = []
    for _ in range(7):
        eng.enqueue(cam, levels, out, query=q, timing=True)
        torch.cuda.synchronize()
        ts.append(out.blend_ms())
    res[name] = round(statistics.median(ts), 3)
    del out
    torch.cuda.empty_cache()
print("grid", os.environ.get("SF_TC_GRID", "sms"), res, flush=True)
