"""Per-SM timeline of the fused blend kernel from SF_BLEND_TIMELINE dumps (development aid).

usage: SF_BLEND_TIMELINE=/tmp/tl.bin python bench.py --steps 1 --warmup 1 ...; python profiles/debug/timeline.py /tmp/tl.bin
"""
import sys
import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 4).astype(np.int64)
ok = (t > 0).all(axis=1)
t = t[ok]
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
blend = t[:, 1] - t[:, 0]
conv = t[:, 2] - t[:, 1]
dec = t[:, 3] - t[:, 2]
print(f"CTAs {len(t)}  kernel span {t[:, 3].max():.1f} us")
for name, v in (("blend", blend), ("epilogue+convert", conv), ("decode", dec)):
    print(f"  {name:18s} mean {v.mean():7.2f} us  p10 {np.percentile(v, 10):7.2f}  p90 {np.percentile(v, 90):7.2f}  sum/296 {v.sum() / 296:8.1f}")
# concurrency: how many CTAs in decode vs blend over time
grid = np.linspace(0, t[:, 3].max(), 200)
nb = [(np.sum((t[:, 0] <= g) & (t[:, 1] > g))) for g in grid]
nd = [(np.sum((t[:, 2] <= g) & (t[:, 3] > g))) for g in grid]
print("  mean CTAs blending", np.mean(nb), " decoding", np.mean(nd))
