"""Debug: error pattern of the fused blend+decode against W @ atoms (fp64) of the same frame."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np, torch
from conftest import random_scene, make_camera
from paper_2507_07136_b200.device import device_scene

for D, op in ((64, (0.2, 0.5)), (512, (0.2, 0.5)), (64, (0.5, 0.98))):
    rng = np.random.default_rng(3)
    scene = random_scene(rng, 3000, num_levels=3, L=64, K=4, D=D, opacity_range=op)
    cam = make_camera(64, 48)
    eng = device_scene(scene).engine
    out = eng.allocate(cam.width, cam.height, (0, 1, 2), coeff_map=True, final_t=True, features=True)
    eng.run(cam, (0, 1, 2), out)
    torch.cuda.synchronize()
    st = out.host_stats()[0]
    print(f"D={D} opacity={op} fixups={st[7]}")
    w = out.coeff_map.double()
    for b in range(3):
        atoms = torch.from_numpy(scene.codebooks[b].atoms).cuda().double()
        ref = (w[:, :, 64 * b:64 * (b + 1)] @ atoms).cpu().numpy()
        f = out.features[b].double().cpu().numpy()
        err = np.abs(f - ref)
        bad = err > 1e-4 * np.abs(ref).max()
        print(f"  level {b}: max err {err.max():.3e} bad frac {bad.mean():.4f}")
        if bad.any():
            H, W = bad.shape[:2]
            ys, xs, ns = np.nonzero(bad)
            print("   bad by col%32:", np.bincount(ns % 32, minlength=32))
            print("   bad by chunk:", np.bincount(ns // 32))
            lx, ly = xs % 16, ys % 16
            slot_warp = (ly // 4) * 2 + (lx // 8)
            lane = (ly % 4) * 8 + (lx % 8)
            print("   bad by warp8:", np.bincount(slot_warp, minlength=8))
            print("   bad by lane:", np.bincount(lane, minlength=32))
            pix_bad = bad.any(axis=2)
            print("   bad pixels:", pix_bad.sum(), "of", H * W, " rows:", np.nonzero(pix_bad.any(axis=1))[0][:20])
            y, x, n = ys[0], xs[0], ns[0]
            print("   first bad", (y, x, n), f[y, x, :8], ref[y, x, :8])
            # is the wrong value the product with a different A row?
            fr = f[y, x]
            dist = np.abs(ref.reshape(-1, D) - fr[None]).max(axis=1)
            print("   closest ref pixel to the bad row:", np.argmin(dist), dist.min(), "own:", y * W + x)
