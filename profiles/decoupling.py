"""Cost decoupling of sparse-coefficient splatting from L (the reference's
sparse-vs-dense harness, splatfield/bench.py:109-131) on the GPU.

For L in {16, 64, 256}: the multilevel coefficient map rendered sparsely
(splat_multilevel: K channels per Gaussian and level scattered into the tile's
accumulator) and densely (render_dense of the densified (G, levels*L) rows,
16 channels per pass).  Device time from the frames' CUDA events; both maps
(through the public API) must agree to 2e-6.

    python profiles/decoupling.py [num_gaussians] [width] [height]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 512
H = int(sys.argv[3]) if len(sys.argv) > 3 else 512
cam = synthetic.make_camera(W, H)


from paper_2507_07136_b200.device import device_scene
from paper_2507_07136_b200.rasterizer import DENSE_CHANNELS_PER_PASS


def device_ms(run, reps=3):
    """Median of the frames' event-timed render stage (projection .. blend)."""
    run()
    ts = []
    for _ in range(reps):
        ts.append(run())
    return float(np.median(ts))


print(f"# {n} Gaussians, {W}x{H}, 3 levels, K=min(4, L), D=512")
print("# device ms from the frames' CUDA events (render = projection + sort + binning + blend);")
print("# dense = render_dense's passes of 16 channels; max abs(sparse - dense) via the public API")
print("| L | sparse render | dense render (passes) | dense / sparse | max abs(sparse - dense) |")
print("|---|---|---|---|---|")
for L in (16, 64, 256):
    scene = synthetic.make_scene(n, L=L, K=min(4, L))
    cfg = scene.config
    levels = tuple(range(cfg.num_levels))
    rows = np.concatenate([scene.densified_coefficients(lv) for lv in range(cfg.num_levels)], axis=1)
    ds = device_scene(scene)
    eng = ds.engine
    out = eng.allocate(W, H, levels, coeff_map=True)

    def sparse_run():
        eng.run(cam, levels, out, timing=True)
        return out.stage_ms()[0]
    t_sp = device_ms(sparse_run)
    vals = torch.from_numpy(np.ascontiguousarray(rows[ds.orig_rows.cpu().numpy()] if ds.orig_rows is not None
                                                 else rows, dtype=np.float32)).cuda()
    g = ds.num_gaussians
    plans = []
    for c0 in range(0, rows.shape[1], DENSE_CHANNELS_PER_PASS):
        cc = min(DENSE_CHANNELS_PER_PASS, rows.shape[1] - c0)
        half = (4 * cc + 15) // 16 * 4
        plan = torch.zeros((g, 2 * half), dtype=torch.int32, device="cuda")
        plan[:, :cc] = torch.arange(cc, dtype=torch.int32, device="cuda") * 516
        plan[:, half:half + cc] = vals[:, c0:c0 + cc].contiguous().view(torch.int32)
        plans.append((plan, cc))
    fo = eng.allocate(W, H, (0,), coeff_map=False)

    def dense_run():
        tot = 0.0
        for plan, cc in plans:
            fo.coeff_map = torch.empty((H, W, cc), dtype=torch.float32, device="cuda")
            eng.run(cam, (0,), fo, dense=(plan, cc), timing=True)
            tot += fo.stage_ms()[0]
        return tot
    t_dn = device_ms(dense_run)
    diff = float(np.abs(sf.splat_multilevel(scene, cam, max_elements=1 << 40).data
                        - sf.render_dense(scene, cam, rows, tag="coefficient", max_elements=1 << 40).data).max())
    print(f"| {L} | {t_sp:.3f} | {t_dn:.3f} ({len(plans)}) | {t_dn / t_sp:.1f}x | {diff:.1e} |")
