"""Time sf_decode (tcgen05 3xTF32) alone on the config C shape: 1440x1080 pixels,
a 192-channel coefficient map (3 levels x L=64), D=512, one launch per level.
Prints ms per frame (3 levels) and the algorithmic GB/s.  Tuning knobs are read by
the library from the environment (SF_DECODE_*), once per process."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_07136_b200 import _native as N  # noqa: E402

lib = N.load()
H, W, L, D, nl = 1080, 1440, 64, 512, 3
P = H * W
g = torch.Generator(device="cuda").manual_seed(0)
wmap = torch.rand(P, nl * L, device="cuda", generator=g)
cbs = torch.randn(nl, L, D, device="cuda", generator=g)
out = torch.empty(nl, P, D, device="cuda")
ws = torch.empty(int(lib.sf_decode_workspace_bytes(L, D)), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def frame():
    for b in range(nl):
        N.check(lib.sf_decode(P, L, D, N.ptr(wmap[:, b * L:]), nl * L, N.ptr(cbs[b]), N.ptr(out[b]),
                              N.ptr(ws), ws.numel(), ctypes.c_void_p(st)))


for _ in range(3):
    frame()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record()
    frame()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
nbytes = nl * (P * D * 4 + P * L * 4 + L * D * 4)
ref = torch.einsum("pl,ld->pd", wmap[:1000, :L].double(), cbs[0].double())
err = ((out[0, :1000].double() - ref).abs().max() / ref.abs().max()).item()
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("SF_DECODE"))
print(f"[{tag or 'default'}] decode {ms:.3f} ms/frame  {nbytes / ms / 1e6:.0f} GB/s  max rel err {err:.2e}")
