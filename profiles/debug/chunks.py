"""Per-chunk clock64 stamps of CTA 2001's fused decode (SF_BLEND_TIMELINE dump, development aid)."""
import sys
import numpy as np
raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
d = raw[-8 * 512:].reshape(8, 64, 8)
iss = d[0]
t0 = iss[0, 0]
print("issuer: g | bfull accempty fence mmas commits bfree bulk (deltas)  | chunk period")
for g in range(0, 24, 2):
    r = iss[g]
    nxt = iss[g + 1, 0] - r[0] if g + 1 < 24 else 0
    print("  ", g, "|", *np.diff(r), "|", nxt)
for w in range(1, 5):
    c = d[w][:, :4]
    print(f"consumer warp {w-1}: g  start  accfull  ldtm  stored  (rel)")
    for g in range(0, 24, 4):
        print("  ", g, *(c[g] - t0))
e = raw[-8 * 512:].reshape(8, 64, 8)[6, 0, :4]
print("epilogue stamps (cycles): pre-rel->Pd staged", e[1] - e[0], " rel", e[2] - e[1], " convert", e[3] - e[2])
b = raw[-8 * 512:].reshape(8, 64, 8)[7, :4, :7]
for w in range(4):
    t_wait, t_a, t_b, nc, ns, nbat, nlist = b[w]
    print(f"warp {w}: list {nlist} batches {nbat} cand {nc} scatters {ns} | cycles wait {t_wait} phaseA {t_a} phaseB {t_b} -> {t_b / max(nc, 1):.0f}/cand")
