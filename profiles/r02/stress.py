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
prog = torch.zeros(148 * 128 + 16 * 256 + 8 * 2048, dtype=torch.int64).pin_memory()
if not os.environ.get("STRESS_NOPROG"):
    os.environ["SF_TC_PROGRESS"] = str(prog.data_ptr())

import paper_2507_07136_b200 as sf  # noqa: E402
from paper_2507_07136_b200 import synthetic  # noqa: E402
from paper_2507_07136_b200.device import QuerySpec, device_scene  # noqa: E402

ROLES = ["prod", "bl0", "bl1", "bl2", "bl3", "dr0", "dr1", "dr2", "dr3", "ev", "dec", "done"]


def dump(n_cta):
    p = prog.numpy()[:148 * 128].reshape(148, 128)
    for c in range(n_cta):
        row = []
        for r in range(12):
            v = int(p[c, r]) & ((1 << 63) - 1)
            a, b = v >> 32, v & 0xFFFFFFFF
            if r >= 9:
                row.append(f"{ROLES[r]} t={a} n={b}")
            else:
                row.append(f"{ROLES[r]} it={a} st={b >> 16} n={b & 0xFFFF}")
        print(c, " | ".join(row))


def run(G, W, H, timeout=float(os.environ.get("STRESS_TIMEOUT", "60"))):
    scene = synthetic.make_scene(G)
    cam = synthetic.make_camera(W, H)
    qv, canon = synthetic.make_query()
    ds = device_scene(scene)
    eng = ds.engine
    eng.pair_capacity = max(eng.pair_capacity, 48 * G)
    levels = (0, 1, 2)
    out = eng.allocate(W, H, levels, coeff_map=False, features=not os.environ.get("STRESS_NOFEAT"), query=True)
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    torch.cuda.synchronize()
    prog.zero_()
    torch.cuda.synchronize()
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
    if f is not None:
        print("  features finite:", bool(torch.isfinite(f).all().item()), "max", f.abs().max().item(), flush=True)
    if not os.environ.get("STRESS_NOPROG"):
        prof_report(min(148, 2 * ((W + 15) // 16) * ((H + 15) // 16)))
        timeline_report()
        chunk_report()


def timeline_report():
    """CTA 0's per-tile events (cycles relative to the first), us at 1.965 GHz."""
    t = prog.numpy()[148 * 128:148 * 128 + 16 * 256].reshape(256, 16).astype(np.int64)
    names = ["blend_start", "blend_end", "epi_done", "ev_wfull", "dec_start", "dec_end", "drain_start",
             "drain_last", "drain_first", "prod_start", "prod_end"]
    n = int((t[:, 0] > 0).sum())
    t0 = t[0, 0]
    print("  tile " + " ".join(f"{x[:11]:>11s}" for x in names))
    for i in list(range(min(n, 6))) + list(range(max(6, n - 3), n)):
        print(f"  {i:4d} " + " ".join(f"{(t[i, e] - t0) / 1965.0:11.2f}" if t[i, e] else f"{'-':>11s}" for e in range(11)))
    if n > 10:
        blend = (t[:n, 1] - t[:n, 0]) / 1965.0
        epi = (t[:n, 2] - t[:n, 1]) / 1965.0
        dec = [(t[i, 5] - t[i, 4]) / 1965.0 for i in range(n) if t[i, 5] and t[i, 4]]
        print(f"  per tile (us): blend mean {blend.mean():.2f} median {np.median(blend):.2f} max {blend.max():.2f}; "
              f"blend_end->epi_done mean {epi.mean():.2f}; decode issue span mean {np.mean(dec) if dec else 0:.2f} "
              f"over {len(dec)} non-empty tiles of {n}")
        d = np.diff(t[:n, :11], axis=0) / 1965.0
        print("  mean per-tile period (us): " + " ".join(f"{x[:6]}={v:.2f}" for x, v in zip(names, d.mean(axis=0))))
        dr = (t[:n, 11] > 0) & (t[:n, 2] > 0) & (t[:n, 12] == 0)
        if dr.any():  # fused decode: the drains run the W epilogue (stamps 11 = w_full, 2 = done)
            tt = t[:n][dr]
            print("  drain epilogue (us, drain 0, mean over %d tiles): blend_end->w_full %.2f, epilogue %.2f" % (
                dr.sum(), ((tt[:, 11] - tt[:, 1]) / 1965.0).mean(), ((tt[:, 2] - tt[:, 11]) / 1965.0).mean()))
        ok = (t[:n, 11] > 0) & (t[:n, 12] > 0) & (t[:n, 13] > 0) & (t[:n, 14] > 0)
        if ok.any():
            tt = t[:n][ok]
            parts = [("loop->bar13", 1, 11), ("bar13->w_full", 11, 12), ("relevancy", 12, 13), ("convert", 13, 14),
                     ("rel_final", 14, 2)]
            print("  epilogue (us, warp 0, mean over %d tiles): " % ok.sum()
                  + " ".join(f"{nm} {((tt[:, b] - tt[:, a]) / 1965.0).mean():.2f}" for nm, a, b in parts))


def chunk_report():
    """CTA 0's per-chunk decode events: issuer start/commit, drain 0 acc_full/ld/bulk/store (cycles)."""
    c = prog.numpy()[148 * 128 + 16 * 256:].reshape(2048, 8).astype(np.int64)
    n = int((c[:, 4] > 0).sum())
    if n < 4:
        return
    t0 = c[0, 4]
    names = ["acc_full", "ld_done", "bulk_ok", "stored", "iss_start", "iss_end"]
    print("  chunk " + " ".join(f"{x:>9s}" for x in names) + "   (cycles from chunk 0 issue)")
    for i in list(range(min(n, 30))) + list(range(max(30, n - 30), n)):
        print(f"  {i:5d} " + " ".join(f"{c[i, e] - t0:9d}" if c[i, e] else f"{'-':>9s}" for e in [0, 1, 2, 3, 4, 5]))
    d = c[:n]
    ok = (d[:, [0, 1, 2, 3, 4, 5]] > 0).all(axis=1)
    d = d[ok]
    print("  mean: issue->commit %.0f, issue->acc_full %.0f, acc_full->ld_done %.0f, ld_done->bulk_ok %.0f, bulk_ok->stored %.0f cycles; chunk period %.0f" % (
        (d[:, 5] - d[:, 4]).mean(), (d[:, 0] - d[:, 4]).mean(), (d[:, 1] - d[:, 0]).mean(), (d[:, 2] - d[:, 1]).mean(),
        (d[:, 3] - d[:, 2]).mean(), np.median(np.diff(d[:, 4]))))


def prof_report(n_cta):
    """Cycle accounting per role (mean over CTAs, in % of the role's total)."""
    p = prog.numpy()[:148 * 128].reshape(148, 128)[:n_cta, 16:].astype(np.float64)
    # 4 counters per warp (slot 4 * warp): blend warps 0-7, drains 8-11, producer 12, E V issuer 13, decode issuer 14
    names = {0: "blend", 32: "drain", 48: "producer", 52: "ev_issuer", 56: "dec_issuer"}
    labels = {"blend": ("waits", "alpha", "walk"), "drain": ("dq_full", "acc_full", "bulk_read(lane0)"),
              "producer": ("ev_empty", "batches", "entries"), "ev_issuer": ("ev_full", "slot_free", "candidate_entries"),
              "dec_issuer": ("a_ready/dq", "b_full", "acc_empty")}
    dur = p[:, 0]  # warp 0's elapsed cycles (persistent CTAs start together)
    print(f"  CTA duration (warp 0, kcyc): min {dur.min() / 1e3:.0f} mean {dur.mean() / 1e3:.0f} max {dur.max() / 1e3:.0f}"
          f" (max/mean {dur.max() / max(dur.mean(), 1):.3f})")
    for base, nm in names.items():
        warps = 8 if base == 0 else (4 if base == 32 else 1)
        tot = p[:, base:base + 4 * warps:4].sum(axis=1)
        print(f"  {nm:9s} total {tot.mean() / 1e3:9.1f} kcyc/CTA", end="")
        for k in range(3):
            v = p[:, base + 1 + k:base + 4 * warps:4].sum(axis=1)
            lab = labels[nm][k]
            if lab == "-":
                continue
            if lab in ("entries", "candidate_entries"):
                print(f"  {lab} {v.mean():.0f}/CTA", end="")
            elif lab == "batches":
                print(f"  batches {v.mean():.0f}/CTA", end="")
            elif lab == "skipped_batches":
                print(f"  skipped batches {v.mean():.0f}/CTA", end="")
            elif lab == "progress_iters":
                print(f"  {lab} {v.mean():.0f}", end="")
            elif lab == "cand":
                raw = prog.numpy()[:148 * 128].reshape(148, 128)[:n_cta, 16:80][:, base + 1 + k:base + 4 * warps:4].astype(np.int64)
                cand, ent = (raw >> 32).sum(), (raw & 0xFFFFFFFF).sum()
                print(f"  candidates {cand / max(ent, 1):.2f} of {ent / n_cta / warps:.0f} entries/warp", end="")
            else:
                print(f"  {lab} {100 * v.mean() / max(tot.mean(), 1):5.1f}%", end="")
        print()


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [20000, 512, 384, 200000, 1024, 768, 2000000, 1440, 1080]
    for i in range(0, len(args), 3):
        run(*args[i:i + 3])
