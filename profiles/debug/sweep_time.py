"""Time query_sweep (one render + n prompt posts, sf_query_sweep) against n
separate lazy query frames, at a BASELINE config.  Dev aid.

    python profiles/debug/sweep_time.py [E|C] [n_prompts] [once]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import torch

import bench
from paper_2507_07136_b200 import synthetic
from paper_2507_07136_b200.device import QuerySpec, device_scene

cfg = sys.argv[1] if len(sys.argv) > 1 else "E"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
n_g, W, H = bench.CONFIGS[cfg]
scene = synthetic.make_scene(n_g)
cam = synthetic.make_camera(W, H)
qv, canon = synthetic.make_query()
rng = np.random.default_rng(5)
prompts = np.concatenate([qv[None], rng.standard_normal((n - 1, qv.shape[0]))])
ds = device_scene(scene)
eng = ds.engine
levels = (0, 1, 2)
out = eng.allocate(W, H, levels, coeff_map=True, mask=False)
if len(sys.argv) > 3 and sys.argv[3] == "once":  # one sweep, for an ncu launch list
    eng.sweep(cam, levels, out, prompts, canon)
    sys.exit(0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(2):
    eng.sweep(cam, levels, out, prompts, canon)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    ev[0].record()
    eng.sweep(cam, levels, out, prompts, canon)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
sweep_ms = float(np.median(ts))
# n separate lazy query frames (query_pipeline's frame, no host round trips)
o = eng.allocate(W, H, levels, coeff_map=False, query=True)
qd = [(torch.from_numpy(p).cuda(), torch.from_numpy(canon).cuda()) for p in prompts]
for i in range(3):
    eng.enqueue(cam, levels, o, query=QuerySpec(prompts[i], canon), qdev=qd[i])
torch.cuda.synchronize()
ev[0].record()
for i in range(n):
    eng.enqueue(cam, levels, o, query=QuerySpec(prompts[i], canon), qdev=qd[i])
ev[1].record()
torch.cuda.synchronize()
sep_ms = ev[0].elapsed_time(ev[1])
print({"config": cfg, "prompts": n, "sweep_ms": sweep_ms, "sweep_prompt_frames_per_s": n / sweep_ms * 1e3,
       "separate_ms": sep_ms, "separate_prompt_frames_per_s": n / sep_ms * 1e3})
