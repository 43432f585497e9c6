"""Benchmark: text-query FPS (and feature-splat FPS) at 1440x1080 with 2M Gaussians.

One step = one full query frame of config C (BASELINE.json
configs[2]): preprocess -> depth-rank sort -> binning -> blend (+ fused
projected-codebook relevancy, + the 3 x 512-d feature decode on tcgen05
inside the same CTA, written to HBM) -> mean filter -> select_level /
localize / segment.  That
is the reference's query_pipeline (sparse_splat.py:243-297) plus segment,
with every feature map materialised, so the same step also bounds
feature-splat FPS (render + decode).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun): one rank per GPU renders its own frames of the scene
(view sharding, config D; weak scaling); the only collective is an NCCL
all-gather of each frame's final mask to every rank (the "gather the final
maps" step).  Timing: CUDA events on the launching stream between a barrier
+ synchronize on both sides; max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "feature-splat FPS and text-query FPS at 1440×1080, ~2M Gaussians, 1/2/4/8 B200"
CONFIGS = {
    "A": (10_000, 256, 256),
    "B": (1_000_000, 988, 731),
    "C": (2_000_000, 1440, 1080),
    "E": (5_000_000, 1920, 1080),
}
# Kernels launched per query frame (sf_render_frame), from the ncu launch list in
# profiles/r01_launches_latest.csv: preprocess, CUB onesweep depth sort (10),
# rank_of_row, count, tile scan, emit, 3 tile-sort kernels, project codebook,
# blend, blend fixup, 3 x (codebook split + tcgen05 decode), 2 x box filter,
# reduce, finalize, mask.
KERNELS_PER_FRAME = 32
# With the decode fused into the blend (profiles/r01_launches_fused.csv): preprocess,
# CUB onesweep depth sort (10), rank_of_row, count, tile scan, emit, 3 tile-sort
# kernels, project codebook, blend (+ decode), fixup, fused box filter + statistics,
# finalize, mask (the codebook image is cached per level selection).
KERNELS_PER_FRAME_FUSED = 24


def ncu_traffic(kernel: str = "decode", summary: str = "r01_ncu_summary.txt"):
    """dram read+write bytes per launch of `kernel` from a committed ncu summary."""
    try:
        cur, rd, wr = None, None, None
        for ln in open(os.path.join(ROOT, "profiles", summary)):
            ln = ln.strip()
            if ln.startswith("kernel:"):
                cur = ln.split(":", 1)[1].strip()
            elif cur == kernel and ln.startswith("dram__bytes_read.sum"):
                v, u = ln.split("=")[1].split()
                rd = float(v) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[u]
            elif cur == kernel and ln.startswith("dram__bytes_write.sum"):
                v, u = ln.split("=")[1].split()
                wr = float(v) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[u]
        return None if rd is None or wr is None else rd + wr
    except OSError:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # nvidia-smi needs a moment to start: wait for its first sample so
            # the timed region is covered, then keep only samples taken in it
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.t_start = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        self.t_stop = time.time()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if self.t_start <= t <= self.t_stop + 0.02]
        for ln in inside or [ln for _, ln in self.lines[-1:]]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        return world, rank, local, dist
    return 1, 0, 0, None


def cpu_baseline_run(scene, cam, qv, canon, band_rows: int = 2):
    """Oracle (C port, OpenMP) on a bounded sample: full projection + binning,
    blend + decode + relevancy of `band_rows` tile rows.  Returns (fps, info)."""
    import numpy as np

    from oracle import oracle as O
    t0 = time.perf_counter()
    proj = O.project_scene(scene, cam)
    binning = O.bin_projected(proj, cam)
    t1 = time.perf_counter()
    tiles_x = binning.tiles_x
    rows = min(band_rows, binning.tiles_y)
    cm = O.splat_levels(scene, cam, range(scene.config.num_levels), binning=binning,
                        tile_range=(0, rows * tiles_x))
    hb = min(rows * 16, cam.height)
    for lv in range(scene.config.num_levels):
        f = O.decode_level(cm.level_view(lv)[:hb], scene.codebooks[lv].atoms)
        O.relevancy_map(f, qv, canon)
        del f
    t2 = time.perf_counter()
    frac = hb / cam.height
    frame_s = (t1 - t0) + (t2 - t1) / frac
    info = {"projection_binning_s": round(t1 - t0, 3), "band_s": round(t2 - t1, 3),
            "band_fraction": round(frac, 5)}
    return 1.0 / frame_s, info, frame_s


def run_reference(args, scene, cam, qv, canon):
    """--impl reference: the CPU oracle port, rank 0 only."""
    from oracle import oracle as O
    ncores = O.num_threads()
    samples = []
    for i in range(args.warmup + args.steps):
        fps, info, _ = cpu_baseline_run(scene, cam, qv, canon, band_rows=args.band_rows)
        if i >= args.warmup:
            samples.append(fps)
    fps = statistics.median(samples)
    n, w, h = CONFIGS[args.config]
    sample = (f"config {args.config}: full projection+binning of {n} Gaussians + blend/decode/"
              f"relevancy of {args.band_rows} tile rows ({info['band_fraction']*100:.2f}% of the "
              f"frame), extrapolated to the frame; median of {args.steps}")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / fps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY 8(d) generator, seed 1)",
        "config": {"workload": f"config {args.config}: {n} Gaussians, {w}x{h}, L=64, K=4, 3 levels, "
                               f"D=512, 1 text query + 4 canonicals", "parallelism": "cpu"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": ncores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": info,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C", choices=sorted(CONFIGS))
    ap.add_argument("--band-rows", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local, dist = dist_setup(args.gpus)
    from paper_2507_07136_b200 import synthetic
    n_g, W, H = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        scene = synthetic.make_scene(n_g)
        cam = synthetic.make_camera(W, H)
        qv, canon = synthetic.make_query()
        run_reference(args, scene, cam, qv, canon)
        return

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    if dist is not None:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2507_07136_b200 as sf
    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200.device import QuerySpec, device_scene

    scene = synthetic.make_scene(n_g)
    cam = synthetic.make_camera(W, H)
    qv, canon = synthetic.make_query()
    ds = device_scene(scene)
    eng = ds.engine
    levels = (0, 1, 2)
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    # decode fused into the blend kernel: the coefficient map never reaches HBM
    fused = bool(N.load().sf_decode_fused(3, 64, 4, 512))
    out = eng.allocate(W, H, levels, coeff_map=not fused, features=True, query=True)
    qdev = (torch.from_numpy(qv).cuda(), torch.from_numpy(canon).cuda())
    eng.run(cam, levels, out, query=spec, qdev=qdev)  # sizes the pair buffer
    stream = torch.cuda.current_stream()
    gathered = None
    if dist is not None:
        gathered = torch.empty((world, H, W), dtype=torch.uint8, device="cuda")

    def step(timing=False):
        eng.enqueue(cam, levels, out, query=spec, qdev=qdev, timing=timing)
        if dist is not None:
            dist.all_gather_into_tensor(gathered, out.mask)

    # the timed loop pipelines frames (device.FramePipeline): every frame does
    # the complete work into its own buffers, but frame i+1's projection /
    # sort / binning and blend overlap frame i's blend tail, fixup and post
    from paper_2507_07136_b200.device import FramePipeline
    pipe = FramePipeline(ds, W, H, levels, coeff_map=not fused, features=True, query=True)

    def pstep():
        o = pipe.enqueue(cam, levels, query=spec, qdev=qdev)
        if dist is not None:
            with torch.cuda.stream(pipe.render[(pipe.k - 1) % 2]):
                dist.all_gather_into_tensor(gathered, o.mask)

    for _ in range(args.warmup):
        step()
    pipe.begin()
    for _ in range(args.warmup):
        pstep()
    pipe.end()
    # per-stage kernel times (render / decode / post) over a few frames
    stage = []
    for _ in range(3):
        step(timing=True)
        stage.append(out.stage_ms() + (out.blend_ms(),))
    torch.cuda.synchronize()
    st = out.stats_i64.cpu().numpy()
    assert st[N.STAT_OVERFLOW] == 0

    # ---- timed region: K frames ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        pipe.begin()
        for _ in range(args.steps):
            pstep()
        pipe.end()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    for o in pipe.outs:
        assert int(o.stats_i64[N.STAT_OVERFLOW].item()) == 0
    # the same K frames one after the other on one stream (no overlap)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    fps_serial = args.steps / (ev0.elapsed_time(ev1) / 1e3)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    fps_total = world * args.steps / (ms / 1e3)

    # decode-stage (dominant kernel) roofline, measured live with CUDA events
    r_ms = statistics.median(s[0] for s in stage)
    d_ms = statistics.median(s[1] for s in stage)
    p_ms = statistics.median(s[2] for s in stage)
    b_ms = statistics.median(s[3] for s in stage)
    P = W * H
    pairs = int(st[N.STAT_PAIRS])
    if fused:
        # fused blend + decode: compulsory HBM bytes = features written + the
        # per-Gaussian records read once (80 B GeomRec + 96 B scatter plan;
        # a record's re-reads by the other tiles it touches hit L2) + one u32
        # tile-list entry per pair + the codebook image
        dom_kernel = "k_blend<DEC> (blend + fused relevancy + fused 3-term fp16 tcgen05 decode, one frame)"
        dec_bytes = 3 * P * 512 * 4 + int(st[N.STAT_VISIBLE]) * (80 + 96) + pairs * 4 + 3 * 8 * 16384
        dom_ms = b_ms
        traffic = ncu_traffic("blend_dec", "r01_ncu_fused.txt")
        traffic_src = "profiles/r01_ncu_fused.txt (ncu --set full, one launch)"
    else:
        dom_kernel = "k_decode_tc (3 levels, one frame)"
        dec_bytes = 3 * P * 512 * 4 + P * 192 * 4 + 3 * 64 * 512 * 4  # F written + W read + codebooks
        dom_ms = d_ms
        t1 = ncu_traffic("decode")
        traffic = 3 * t1 if t1 else None
        traffic_src = "profiles/r01_ncu_summary.txt (ncu --set full, per launch x 3 levels)"
    hbm_peak, peak_kind = peaks()
    achieved = dec_bytes / (dom_ms / 1e3) / 1e9

    # ---- e2e through the public API: query_pipeline with host query inputs ----
    e2e = None
    if not args.no_e2e:
        del out  # release the device-loop buffers; the API allocates its own results
        torch.cuda.empty_cache()
        qe = sf.QueryEmbedding("bench", qv)
        canon_pinned = torch.from_numpy(canon).pin_memory().numpy()
        for _ in range(3):
            sf.query_pipeline(scene, cam, qe, canon_pinned, features="eager", instrument=False,
                              max_elements=1 << 40)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        n_e2e = max(3, args.steps // 2)
        for _ in range(n_e2e):
            res = sf.query_pipeline(scene, cam, qe, canon_pinned, features="eager", instrument=False,
                                    max_elements=1 << 40)
            _ = res.mask  # already on the host: the step's result
            del res  # one frame's results alive at a time (the allocator reuses the block)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": world * n_e2e / dt, "unit": "frames/s",
               "h2d_bytes_per_step": int(qv.nbytes + canon.nbytes),
               "d2h_bytes_per_step": int(H * W + 16 * 8 + (8 + 2 * 8) * 8), "steps": n_e2e,
               "api": "paper_2507_07136_b200.query_pipeline(..., features='eager')"}
        # the same frames through the pipelined serving API: per frame the query
        # vector goes up from pinned memory and the mask + statistics come back;
        # results are read one frame behind the submits
        qstream = sf.QueryStream(scene, W, H, canon, features="eager")
        for _ in range(3):
            qstream.result(qstream.submit(cam, qe))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        n_st = max(3, args.steps)
        pending = None
        for _ in range(n_st):
            h = qstream.submit(cam, qe)
            if pending is not None:
                _ = qstream.result(pending).mask
            pending = h
        _ = qstream.result(pending).mask
        qstream.close()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e["pipelined"] = {"value": world * n_st / dt, "unit": "frames/s", "steps": n_st,
                            "h2d_bytes_per_step": int(qv.nbytes), "d2h_bytes_per_step": int(H * W + 16 * 8),
                            "api": "paper_2507_07136_b200.QueryStream(..., features='eager').submit / .result"}
        del qstream
        torch.cuda.empty_cache()

    # feature-splat FPS (render + decode, no query post) and lazy-feature query FPS
    del pipe
    torch.cuda.empty_cache()
    extra = {}
    for name, alloc, q in (("feature_splat", dict(coeff_map=not fused, features=True, query=False), None),
                           ("text_query_lazy_features", dict(coeff_map=False, features=False, query=True), spec)):
        o = eng.allocate(W, H, levels, **alloc)
        p2 = FramePipeline(ds, W, H, levels, **alloc)
        p2.begin()
        for _ in range(3):
            eng.enqueue(cam, levels, o, query=q, qdev=qdev)
            p2.enqueue(cam, levels, query=q, qdev=qdev)
        p2.end()
        for mode in ("serial", "pipelined"):
            torch.cuda.synchronize()
            ev0.record(stream)
            if mode == "pipelined":
                p2.begin()
            for _ in range(args.steps):
                if mode == "serial":
                    eng.enqueue(cam, levels, o, query=q, qdev=qdev)
                else:
                    p2.enqueue(cam, levels, query=q, qdev=qdev)
            if mode == "pipelined":
                p2.end()
            ev1.record(stream)
            torch.cuda.synchronize()
            fps = args.steps / (ev0.elapsed_time(ev1) / 1e3)
            extra[name if mode == "pipelined" else name + "_serial"] = fps
        del o, p2
        torch.cuda.empty_cache()

    # config E's prompt sweep: 32 prompts over one view -- one
    # render of the coefficient map, then every prompt's relevancy / filter /
    # select / mask from it (sf_query_sweep); reported beside the main line
    sweep = None
    if not args.no_sweep:
        n_prompts = 32
        prng = np.random.default_rng(7)
        prompts = np.concatenate([qv[None], prng.standard_normal((n_prompts - 1, qv.shape[0]))])
        so = eng.allocate(W, H, levels, coeff_map=True, mask=False)
        for _ in range(2):
            eng.sweep(cam, levels, so, prompts, canon)
        n_sw = max(3, args.steps // 4)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(n_sw):
            eng.sweep(cam, levels, so, prompts, canon)
        ev1.record(stream)
        torch.cuda.synchronize()
        sw_ms = ev0.elapsed_time(ev1) / n_sw
        sweep = {"prompts": n_prompts, "ms_per_sweep": sw_ms, "prompt_frames_per_s": n_prompts / sw_ms * 1e3,
                 "sweeps": n_sw,
                 "note": ("paper_2507_07136_b200.query_sweep's device part (FrameEngine.sweep): each sweep "
                          "renders the view and answers 32 prompts; one host sync per sweep (its statistics)")}
        del so
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        fps_cpu, info, _ = cpu_baseline_run(scene, cam, qv, canon, band_rows=args.band_rows)
        cpu = {"value": fps_cpu, "unit": "frames/s", "cores": O.num_threads(), "kind": "port",
               "sample": (f"oracle C port (OpenMP): full projection+binning of {n_g} Gaussians + "
                          f"blend/decode/relevancy of {args.band_rows} tile rows "
                          f"({info['band_fraction']*100:.2f}% of the frame), extrapolated"),
               "detail": info}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": fps_total, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SURVEY 8(d) generator, seed 1; random codebooks/query)",
            "config": {
                "workload": (f"config {args.config}: {n_g} Gaussians, {W}x{H}, 3 levels, L=64, K=4, "
                             "D=512 features decoded (3-term fp16 tcgen05, fused into the blend) + 1 text query vs 4 canonicals, "
                             "window 11, level select + localize + segment"),
                "parallelism": f"views x{world}" if world > 1 else "single",
                "l2": "inputs/outputs larger than L2 (9.56 GB of features per frame)",
                "visible": int(st[N.STAT_VISIBLE]), "pairs": int(st[N.STAT_PAIRS]),
                "exact_fp64_fixup_pixels": int(st[7]),
            },
            "fps": {"text_query_full": fps_total / world,
                    "text_query_full_serial": fps_serial,
                    "feature_splat": extra["feature_splat"],
                    "feature_splat_serial": extra["feature_splat_serial"],
                    "text_query_lazy_features": extra["text_query_lazy_features"],
                    "text_query_lazy_features_serial": extra["text_query_lazy_features_serial"],
                    "note": ("pipelined (value): every frame does the complete work into its own buffers; "
                             "frame i's projection/sort/binning run on a shared prepare stream and its "
                             "blend/decode/post on render stream i%2 (sf_render_frame_split, two "
                             "workspaces), so consecutive frames overlap; serial: one frame after another "
                             "on one stream")},
            "stage_ms": {"render": r_ms, "decode": d_ms, "post": p_ms, "blend_kernel": b_ms,
                         "decode_fused_into_blend": fused},
            "roofline": {"bound": "hbm", "kernel": dom_kernel,
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "algorithmic_bytes": dec_bytes, "time_ms": dom_ms,
                         "traffic": traffic, "traffic_source": traffic_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "query_sweep": sweep,
            "gpu_launches": (KERNELS_PER_FRAME_FUSED if fused else KERNELS_PER_FRAME) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
