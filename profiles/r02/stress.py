"""Development aid: run eager-feature query frames of growing size with a
watchdog; on a hang, dump k_splat_tc's per-CTA role progress (SF_TC_PROGRESS,
mapped pinned memory) and exit.  Also compares each frame with the legacy
kernel's (SF_BLEND_IMPL=legacy in a child process) when --compare is given.

usage: python profiles/r02/stress.py [G W H] ...
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
prog = torch.zeros(148 * 16, dtype=torch.int64).pin_memory()
os.environ["SF_TC_PROGRESS"] = str(prog.data_ptr())

import paper_2507_07136_b200 as sf  # noqa: E402
from paper_2507_07136_b200 import synthetic  # noqa: E402
from paper_2507_07136_b200.device import QuerySpec, device_scene  # noqa: E402

ROLES = ["prod", "bl0", "bl1", "bl2", "bl3", "dr0", "dr1", "dr2", "dr3", "mma"]


def dump(n_cta):
    p = prog.numpy().reshape(148, 16)
    for c in range(n_cta):
        row = []
        for r in range(10):
            v = int(p[c, r]) & ((1 << 63) - 1)
            a, b = v >> 32, v & 0xFFFFFFFF
            if r == 9:
                row.append(f"mma te={a >> 16} td={a & 0xFFFF} be={b >> 16} Gd={b & 0xFFFF}")
            else:
                row.append(f"{ROLES[r]} it={a} st={b >> 16} n={b & 0xFFFF}")
        print(c, " | ".join(row))


def run(G, W, H, timeout=60.0):
    scene = synthetic.make_scene(G)
    cam = synthetic.make_camera(W, H)
    qv, canon = synthetic.make_query()
    ds = device_scene(scene)
    eng = ds.engine
    eng.pair_capacity = max(eng.pair_capacity, 48 * G)
    levels = (0, 1, 2)
    out = eng.allocate(W, H, levels, coeff_map=False, features=True, query=True)
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    torch.cuda.synchronize()
    prog.zero_()
    t0 = time.time()
    keep = eng.enqueue(cam, levels, out, query=spec)
    ev = torch.cuda.Event()
    ev.record()
    while not ev.query():
        if time.time() - t0 > timeout:
            print(f"HANG at G={G} {W}x{H} after {timeout}s", flush=True)
            n_half = 2 * ((W + 15) // 16) * ((H + 15) // 16)
            dump(min(148, n_half))
            sys.stdout.flush()
            os._exit(3)
        time.sleep(0.05)
    del keep
    st = out.stats_i64.cpu().numpy()
    print(f"ok G={G} {W}x{H} in {time.time() - t0:.2f}s pairs={st[1]} fixups={st[7]} level={st[3]}", flush=True)
    f = out.features
    print("  features finite:", bool(torch.isfinite(f).all().item()), "max", f.abs().max().item(), flush=True)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [20000, 512, 384, 200000, 1024, 768, 2000000, 1440, 1080]
    for i in range(0, len(args), 3):
        run(*args[i:i + 3])
