"""Benchmark: text-query FPS (and feature-splat FPS) at 1440x1080 with 2M Gaussians.

One step = one full query frame of config C (BASELINE.json
configs[2]): preprocess -> depth sort -> binning -> blend (+ fused
projected-codebook relevancy, + the 3 x 512-d feature decode on tcgen05
inside the same CTA, written to HBM) -> mean filter -> select_level /
localize / segment.  That is the reference's query_pipeline
(sparse_splat.py:243-297) plus segment, with every feature map
materialised, so the same step also bounds feature-splat FPS (render +
decode).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N = 1: config C, plus (after the timed region) a full-frame parity check of
the benchmarked frame path against the CPU oracle (``parity``), whose oracle
time is the ``cpu_baseline``.  N > 1 (re-executed under torch.distributed.run
when WORLD_SIZE is unset): config D -- 64 orbit views sharded by view, K
frames per rank, masks NCCL all-gathered each step (weak scaling) -- and
config E's tile-band sharded 32-prompt sweep.  Timing: CUDA events on the
launching stream between a barrier + synchronize on both sides; max over
ranks.  ``--impl reference``: the CPU oracle, one full frame per step, rank 0.
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
# Kernels launched per query frame (sf_render_frame) with the decode fused into
# the splat (round 2 launch list, profiles/r02/evidence/): preprocess, count,
# tile scan, emit, 3 per-tile depth sorts, project codebook, splat (+ decode),
# fixup, fused box filter + statistics, finalize, mask.  The single-GPU path
# counts them live (count_kernels_per_frame); this constant serves the N > 1 line.
KERNELS_PER_FRAME_FUSED = 13


NCU_SUMMARY = "r02_ncu_splat.txt"


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


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args) -> None:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this script
    under torch.distributed.run with N ranks (one process per GPU) and exit
    with its status, so a plain invocation measures N GPUs, not one."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))


def host_info() -> dict:
    """CPU model, cores and numpy / BLAS of the host (the reference arm's machine)."""
    import numpy as np
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "numpy": np.__version__, "blas": blas,
            "omp_threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or None}


PY_REFERENCE_SCRIPT = r"""
import json, os, sys, time
sys.path.insert(0, os.path.join(sys.argv[1], "baseline", "_ref"))
sys.path.insert(0, sys.argv[1])
import numpy as np
import splatfield as R
from paper_2507_07136_b200 import synthetic
n, w, h = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ours = synthetic.make_scene(n)
cfg = R.SceneConfig(num_levels=3, L=64, K=4, D=512)
scene = R.Scene(positions=ours.positions, rotations=ours.rotations, scales=ours.scales,
                opacities=ours.opacities, colors=ours.colors, coeff_indices=ours.coeff_indices,
                coeff_values=ours.coeff_values,
                codebooks=tuple(R.Codebook(cb.atoms, level=cb.level) for cb in ours.codebooks), config=cfg)
cam = R.Camera.look_at((0.0, 0.0, -3.0), (0.0, 0.0, 0.0), fov_y_deg=45.0, width=w, height=h)
qv, canon = synthetic.make_query()
q = R.QueryEmbedding("bench", qv)
t = {}
t0 = time.perf_counter()
cmap = R.splat_multilevel(scene, cam, workers=os.cpu_count(), max_elements=1 << 34)
t["render"] = time.perf_counter() - t0
t0 = time.perf_counter()
fms = R.decode(cmap, scene.codebooks)
t["decode"] = time.perf_counter() - t0
t0 = time.perf_counter()
maps = [R.mean_filter(R.relevancy_map(fms.maps[b], q, canon, level=b), 11) for b in range(3)]
lv, chosen = R.select_level(maps)
pt = R.localize(chosen)
seg = R.segment(chosen)
t["post"] = time.perf_counter() - t0
t["total"] = sum(t.values())
print(json.dumps({"seconds": t, "fps": 1.0 / t["total"], "level": int(lv), "point": [int(pt[0]), int(pt[1])],
                  "workers": os.cpu_count()}))
"""


def python_reference_once(config: str, timeout_s: float = 900.0) -> dict:
    """the reference package as shipped (splatfield,
    installed into baseline/_ref), one frame of `config` stage by stage with
    the thread pool over all host cores, in a subprocess with a time limit."""
    ref = os.path.join(ROOT, "baseline", "_ref", "splatfield")
    if not os.path.isdir(ref):
        return {"unavailable": "baseline/_ref/splatfield is not installed"}
    n, w, h = CONFIGS[config]
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(os.cpu_count()))
    try:
        r = subprocess.run([sys.executable, "-c", PY_REFERENCE_SCRIPT, ROOT, str(n), str(w), str(h)],
                           capture_output=True, text=True, timeout=timeout_s, env=env)
    except subprocess.TimeoutExpired:
        return {"unavailable": f"did not finish within {timeout_s:.0f} s"}
    if r.returncode != 0:
        return {"unavailable": "rc=%d: %s" % (r.returncode, r.stderr.strip().splitlines()[-1:] or "")}
    out = json.loads(r.stdout.strip().splitlines()[-1])
    out["what"] = (f"splatfield (the reference package, baseline/_ref) config {config}: splat_multilevel("
                   "workers=nproc, max_elements=2**34) -> decode -> 3 x mean_filter(relevancy_map) -> "
                   "select_level / localize / segment, one frame, perf_counter per stage")
    return out


def run_reference(args):
    """--impl reference: the CPU oracle (a C restatement of the reference,
    OpenMP over tiles) timing one FULL frame of the config per step -- project,
    bin, splat, decode, relevancy, mean filter, select, localize, segment
    (oracle/parity.oracle_frame) -- on the host cores; rank 0 only.  At N=1
    the reference package itself (Python) is also timed once (detail)."""
    from oracle import oracle as O
    from oracle.parity import oracle_frame
    from paper_2507_07136_b200 import synthetic

    n, w, h = CONFIGS[args.config]
    scene = synthetic.make_scene(n)
    cam = synthetic.make_camera(w, h)
    qv, canon = synthetic.make_query()
    warm = min(args.warmup, 1)  # the CPU port has no warm-up effects worth a 10 s frame
    secs, stages = [], None
    t_all = time.perf_counter()
    for i in range(warm + args.steps):
        t0 = time.perf_counter()
        o = oracle_frame(scene, cam, qv, canon)
        dt = time.perf_counter() - t0
        del o
        if i >= warm:
            secs.append(dt)
            stages = stages or {}
    wall = time.perf_counter() - t_all
    fps = len(secs) / sum(secs)
    o = oracle_frame(scene, cam, qv, canon)
    stage_s = {k: round(v, 3) for k, v in o["seconds"].items()}
    del o
    ncores = O.num_threads()
    sample = (f"config {args.config}: one full frame per step ({n} Gaussians, {w}x{h}, 3 levels x 512-d "
              f"features, 1 query + 4 canonicals): project + bin + splat + decode + relevancy + mean filter + "
              f"select/localize/segment; {args.steps} timed frames after {warm} warm-up")
    detail = {"host": host_info(), "stage_s_one_frame": stage_s, "frame_s": [round(x, 3) for x in secs],
              "wall_s": round(wall, 1)}
    if args.world == 1 and not args.no_python_reference:
        detail["python_reference"] = python_reference_once(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": warm, "ms_per_step": 1e3 / fps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY 8(d) generator, seed 1)",
        "config": {"workload": workload_name(args.config), "parallelism": f"cpu x{ncores} threads"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": ncores, "kind": "port", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": detail,
    }
    print(json.dumps(line), flush=True)


def workload_name(config: str) -> str:
    n, w, h = CONFIGS[config]
    return (f"config {config}: {n} Gaussians, {w}x{h}, 3 levels, L=64, K=4, D=512 features decoded + "
            "1 text query vs 4 canonicals, window 11, level select + localize + segment")


def run_parity(scene, cam, qv, canon) -> tuple:
    """The benchmarked frame path (fused blend + decode, every output
    materialised) against the CPU oracle over the full frame
    (oracle/parity.py); also yields the oracle's full-frame time (cpu_baseline)."""
    import gc

    from oracle import oracle as O
    from oracle import parity as OP
    gpu = OP.gpu_frame(scene, cam, qv, canon)
    rep = OP.compare_frame(scene, cam, qv, canon, gpu)
    rep.update(fixups=gpu["fixups"], pairs=gpu["pairs"], visible=gpu["visible"])
    del gpu
    gc.collect()
    frame_s = rep["oracle_stage_s"]["total"]
    cpu = {"value": 1.0 / frame_s, "unit": "frames/s", "cores": O.num_threads(), "kind": "port",
           "sample": ("oracle C port (OpenMP over tiles): one full frame of the benchmarked config -- "
                      "project, bin, splat, decode, relevancy, mean filter, select/localize/segment -- the "
                      "same frame the parity check compares"),
           "detail": {"stage_s": rep["oracle_stage_s"], "host": host_info()}}
    return rep, cpu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the parity / oracle leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-python-reference", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_spawn(args)

    world, rank, local, dist = dist_setup(args.gpus)
    args.world = world
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return
    if world > 1:
        return run_multi(args, world, rank, local, dist)
    return run_single(args)


def tf32_peak() -> dict:
    """Dense TF32 tensor throughput on this GPU (cuBLAS 8192^3, median of 5):
    the denominator for the decode GEMM's tensor roofline (the
    frame's decode is 2 H W 3 64 512 = 305.8 GFLOP at config C, issued 3x by
    the 3-term split)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(2):
            a @ b
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[2]
        return {"tf32_dense_tflops": 2 * n ** 3 / (ms / 1e3) / 1e12, "probe": "torch.matmul fp32 8192^3, allow_tf32",
                "decode_gflop_per_frame": 2 * 1440 * 1080 * 3 * 64 * 512 / 1e9}
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def count_kernels_per_frame(enqueue, pipe) -> int:
    """Kernels one pipelined frame launches, counted by the CUDA profiler on an
    untimed frame (every one is this repo's: the frame path calls no library
    kernels; memsets and copies are not counted)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pipe.begin()
        enqueue()
        pipe.end()
        torch.cuda.synchronize()
    kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
            and "memset" not in e.name.lower() and "memcpy" not in e.name.lower()]
    return len(kern)


def run_single(args):
    import numpy as np
    import torch

    import paper_2507_07136_b200 as sf
    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200 import synthetic
    from paper_2507_07136_b200.device import FramePipeline, QuerySpec, device_scene

    torch.cuda.set_device(0)
    n_g, W, H = CONFIGS[args.config]
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

    def step(timing=False):
        eng.enqueue(cam, levels, out, query=spec, qdev=qdev, timing=timing)

    # the timed loop pipelines frames (device.FramePipeline): every frame does
    # the complete work into its own buffers, but frame i+1's projection /
    # sort / binning and blend overlap frame i's blend tail, fixup and post
    pipe = FramePipeline(ds, W, H, levels, coeff_map=not fused, features=True, query=True)
    for _ in range(args.warmup):
        step()
    pipe.begin()
    for _ in range(args.warmup):
        pipe.enqueue(cam, levels, query=spec, qdev=qdev)
    pipe.end()
    launches_per_frame = count_kernels_per_frame(lambda: pipe.enqueue(cam, levels, query=spec, qdev=qdev), pipe)
    stage = []
    for _ in range(3):
        step(timing=True)
        stage.append(out.stage_ms() + (out.blend_ms(),))
    torch.cuda.synchronize()
    st = out.stats_i64.cpu().numpy()
    assert st[N.STAT_OVERFLOW] == 0

    # ---- timed region: K frames ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        ev0.record(stream)
        pipe.begin()
        for _ in range(args.steps):
            pipe.enqueue(cam, levels, query=spec, qdev=qdev)
        pipe.end()
        ev1.record(stream)
        torch.cuda.synchronize()
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
    ms_per_step = ms / args.steps
    fps_total = args.steps / (ms / 1e3)

    # dominant-kernel roofline, measured live with CUDA events on the launch stream
    b_ms = statistics.median(s[3] for s in stage)
    r_ms = statistics.median(s[0] for s in stage)
    d_ms = statistics.median(s[1] for s in stage)
    p_ms = statistics.median(s[2] for s in stage)
    P = W * H
    vis = int(st[N.STAT_VISIBLE])
    # SURVEY 8(d) algorithmic bytes of the fused blend + decode: the scene read
    # once (116 B per visible Gaussian), the codebooks, the fp32 features written
    alg_bytes = 3 * P * 512 * 4 + vis * 116 + 3 * 64 * 512 * 4
    dom_kernel = ("tcs::k_splat_tc<4,DEC> (persistent splat: E V blend products + fused relevancy + "
                  "3-term fp16 decode on tcgen05, one frame)")
    traffic = ncu_traffic("splat_tc", NCU_SUMMARY)
    hbm_peak, peak_kind = peaks()
    achieved = alg_bytes / (b_ms / 1e3) / 1e9

    e2e = None if args.no_e2e else measure_e2e(args, scene, cam, qv, canon, W, H, 1, None)
    del out
    torch.cuda.empty_cache()
    extra = measure_variants(args, ds, eng, cam, levels, spec, qdev, W, H, fused)
    sweep = None if args.no_sweep else measure_sweep(args, eng, cam, levels, qv, canon, W, H)
    # config D's orbit views on this one GPU (the per-GPU term of the N-GPU runs)
    orbit = measure_orbit(args, ds, levels, spec, qdev, W, H, fused, 0, 1, None)
    del pipe
    torch.cuda.empty_cache()
    # config E's own load on one GPU: 5M Gaussians at 1920x1080, 32 prompts
    config_e = None
    if not args.no_sweep and args.config == "C":
        config_e = measure_band_sweep(args, 1, 0, None)
        torch.cuda.empty_cache()
    tf32 = tf32_peak()

    parity, cpu = None, None
    if not args.no_cpu_baseline:
        parity, cpu = run_parity(scene, cam, qv, canon)

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": fps_total, "unit": "frames/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SURVEY 8(d) generator, seed 1; random codebooks/query)",
        "config": {
            "workload": workload_name(args.config) + " (3-term fp16 tcgen05 decode fused into the blend)",
            "parallelism": "single",
            "l2": "inputs/outputs larger than L2 (9.56 GB of features per frame)",
            "visible": vis, "pairs": int(st[N.STAT_PAIRS]), "exact_fp64_fixup_pixels": int(st[N.STAT_FIXUPS]),
        },
        "fps": {"text_query_full": fps_total, "text_query_full_serial": fps_serial, **extra,
                "orbit_views": orbit,
                "note": ("pipelined (value): every frame does the complete work into its own buffers; "
                         "frame i's projection/sort/binning run on a shared prepare stream and its "
                         "blend/decode/post on render stream i%2 (sf_render_frame_split, two "
                         "workspaces), so consecutive frames overlap; serial: one frame after another "
                         "on one stream")},
        "stage_ms": {"render": r_ms, "decode": d_ms, "post": p_ms, "blend_kernel": b_ms,
                     "decode_fused_into_blend": fused},
        "roofline": {"bound": "hbm", "kernel": dom_kernel, "achieved": achieved, "peak": hbm_peak,
                     "unit": "GB/s", "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                     "algorithmic_bytes": alg_bytes,
                     "algorithmic_bytes_rule": "SURVEY 8(d): 116 B x visible Gaussians + 3x64x512x4 B codebooks "
                                               "+ H x W x 3 x 512 x 4 B features",
                     "time_ms": b_ms, "traffic": traffic, "traffic_source": f"profiles/{NCU_SUMMARY}"},
        "cpu_baseline": cpu,
        "parity": parity,
        "e2e": e2e,
        "query_sweep": sweep,
        "config_e_sweep": config_e,
        "tensor_peak": tf32,
        "gpu_launches": launches_per_frame * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def measure_e2e(args, scene, cam, qv, canon, W, H, world, dist):
    """query_pipeline through the public API with host inputs (pinned) and the
    mask + statistics read back each frame; then the pipelined QueryStream."""
    import torch

    import paper_2507_07136_b200 as sf
    torch.cuda.empty_cache()
    qe = sf.QueryEmbedding("bench", qv)
    canon_pinned = torch.from_numpy(canon).pin_memory().numpy()
    for _ in range(3):
        sf.query_pipeline(scene, cam, qe, canon_pinned, features="eager", instrument=False, max_elements=1 << 40)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    n_e2e = max(3, args.steps // 2)
    for _ in range(n_e2e):
        res = sf.query_pipeline(scene, cam, qe, canon_pinned, features="eager", instrument=False,
                                max_elements=1 << 40)
        _ = res.mask  # already on the host: the step's result
        del res
    torch.cuda.synchronize()
    dt = _max_over_ranks(time.perf_counter() - t0, dist)
    e2e = {"value": world * n_e2e / dt, "unit": "frames/s", "h2d_bytes_per_step": int(qv.nbytes + canon.nbytes),
           "d2h_bytes_per_step": int(H * W + 16 * 8 + (8 + 2 * 8) * 8), "steps": n_e2e,
           "api": "paper_2507_07136_b200.query_pipeline(..., features='eager')"}
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
    dt = _max_over_ranks(time.perf_counter() - t0, dist)
    e2e["pipelined"] = {"value": world * n_st / dt, "unit": "frames/s", "steps": n_st,
                        "h2d_bytes_per_step": int(qv.nbytes), "d2h_bytes_per_step": int(H * W + 16 * 8),
                        "api": "paper_2507_07136_b200.QueryStream(..., features='eager').submit / .result"}
    del qstream
    torch.cuda.empty_cache()
    return e2e


def _max_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measure_variants(args, ds, eng, cam, levels, spec, qdev, W, H, fused):
    """feature-splat FPS (render + decode, no query post) and lazy-feature query FPS."""
    import torch

    from paper_2507_07136_b200.device import FramePipeline
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
    return extra


def measure_sweep(args, eng, cam, levels, qv, canon, W, H):
    """config E's prompt load: 32 prompts over one view -- one
    render of the coefficient map, then every prompt's relevancy / filter /
    select / mask from it (sf_query_sweep)."""
    import numpy as np
    import torch
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
    del so
    torch.cuda.empty_cache()
    return {"prompts": n_prompts, "ms_per_sweep": sw_ms, "prompt_frames_per_s": n_prompts / sw_ms * 1e3,
            "sweeps": n_sw,
            "note": ("paper_2507_07136_b200.query_sweep's device part (FrameEngine.sweep): each sweep "
                     "renders the view and answers 32 prompts; one host sync per sweep (its statistics)")}


def measure_orbit(args, ds, levels, spec, qdev, W, H, fused, rank, world, dist, timed_steps=None, clk_index=None):
    """Config D: the 64 orbit cameras (synthetic.orbit_cameras), views sharded
    round-robin over ranks (distributed.shard_views); each step renders one of
    this rank's views (full query frame, features materialised) and NCCL
    all-gathers every rank's mask (the "gather the final maps" step).
    Returns frames/s over all ranks (max-over-ranks device time)."""
    import torch

    from paper_2507_07136_b200 import synthetic
    from paper_2507_07136_b200.device import FramePipeline
    from paper_2507_07136_b200.distributed import shard_views
    cams = synthetic.orbit_cameras(64, W, H)
    mine = [cams[j] for j in shard_views(64, world, rank)]
    steps = timed_steps or min(len(mine), 16)
    pipe = FramePipeline(ds, W, H, levels, coeff_map=not fused, features=True, query=True)
    gathered = torch.empty((world, H, W), dtype=torch.uint8, device="cuda") if dist is not None else None
    for c in mine[:2]:
        ds.engine.run(c, levels, ds.engine.allocate(W, H, levels, coeff_map=not fused, features=False, query=True),
                      query=spec, qdev=qdev)  # sizes the pair buffers of these views
    for e in pipe.engines:
        e.pair_capacity = max(e.pair_capacity, ds.engine.pair_capacity)

    def pstep(i):
        o = pipe.enqueue(mine[i % len(mine)], levels, query=spec, qdev=qdev)
        if dist is not None:
            with torch.cuda.stream(pipe.render[(pipe.k - 1) % 2]):
                dist.all_gather_into_tensor(gathered, o.mask)

    pipe.begin()
    for i in range(args.warmup):
        pstep(i)
    pipe.end()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    import contextlib
    cm = ClockSampler(clk_index) if clk_index is not None else contextlib.nullcontext()
    with cm as clk:
        ev0.record(stream)
        pipe.begin()
        for i in range(steps):
            pstep(i)
        pipe.end()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = _max_over_ranks(ev0.elapsed_time(ev1), dist)
    from paper_2507_07136_b200 import _native as N
    for o in pipe.outs:
        assert int(o.stats_i64[N.STAT_OVERFLOW].item()) == 0
    del pipe
    torch.cuda.empty_cache()
    res = {"value": world * steps / (ms / 1e3), "unit": "frames/s", "ms": ms, "frames_per_rank": steps,
           "views_per_rank": len(mine)}
    if clk_index is not None:
        res["clocks"] = clk.summary()
    return res


def run_multi(args, world, rank, local, dist):
    """N > 1 (torchrun, one rank per GPU, NCCL): config D -- 64 orbit views of
    the 2M-Gaussian scene sharded by view, K frames per rank per run (weak
    scaling), masks all-gathered each step -- plus config E's tile-band
    sharded 32-prompt sweep (distributed.band_query_sweep: one band per
    rank, selection by two NCCL max-all-reduces, masks written per band)."""
    import numpy as np
    import torch

    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200 import synthetic
    from paper_2507_07136_b200.device import QuerySpec, device_scene

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_g, W, H = CONFIGS[args.config]
    scene = synthetic.make_scene(n_g)
    qv, canon = synthetic.make_query()
    ds = device_scene(scene)
    levels = (0, 1, 2)
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    fused = bool(N.load().sf_decode_fused(3, 64, 4, 512))
    qdev = (torch.from_numpy(qv).cuda(), torch.from_numpy(canon).cuda())
    orbit = measure_orbit(args, ds, levels, spec, qdev, W, H, fused, rank, world, dist,
                          timed_steps=args.steps, clk_index=local)
    cam0 = synthetic.orbit_cameras(64, W, H)[rank]
    e2e = None if args.no_e2e else measure_e2e(args, scene, cam0, qv, canon, W, H, world, dist)
    del ds
    torch.cuda.empty_cache()
    band = None if args.no_sweep else measure_band_sweep(args, world, rank, dist)
    if rank == 0:
        line = {
            "metric": METRIC, "value": orbit["value"], "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": orbit["ms"] / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SURVEY 8(d) generator, seed 1; random codebooks/query)",
            "config": {"workload": (f"config D: 64 orbit views (synthetic.orbit_cameras) of the {n_g}-Gaussian "
                                    f"scene at {W}x{H}, sharded by view (views j = rank mod {world}); each rank "
                                    "renders K full query frames (3 x 512 features decoded) and the masks are "
                                    "NCCL all-gathered every step"),
                       "parallelism": f"views x{world}", "frames_per_rank": args.steps,
                       "l2": "outputs larger than L2 (9.56 GB of features per frame)"},
            "e2e": e2e,
            "band_sweep": band,
            "gpu_launches": KERNELS_PER_FRAME_FUSED * args.steps,
            "clocks": orbit.get("clocks"),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def measure_band_sweep(args, world, rank, dist=None):
    """Config E: 5M Gaussians at 1920x1080, 32 prompts, one tile band per rank
    (distributed.band_query_sweep); sweeps per second over all ranks.  With
    dist=None (one GPU) the single band is the whole view."""
    import numpy as np
    import torch

    from paper_2507_07136_b200 import synthetic
    from paper_2507_07136_b200.device import device_scene
    from paper_2507_07136_b200.distributed import band_query_sweep
    n_g, W, H = CONFIGS["E"]
    scene = synthetic.make_scene(n_g)
    cam = synthetic.make_camera(W, H)
    prompts = np.stack([np.random.default_rng(100 + k).standard_normal(512) for k in range(32)])
    _, canon = synthetic.make_query()
    eng = device_scene(scene).engine
    for _ in range(2):
        band_query_sweep(eng, cam, (0, 1, 2), prompts, canon, world, rank)
    n = max(3, args.steps // 4)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        bs = band_query_sweep(eng, cam, (0, 1, 2), prompts, canon, world, rank)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if dist is not None:
        dt = _max_over_ranks(dt, dist)
    del bs, eng
    torch.cuda.empty_cache()
    return {"sweeps_per_s": n / dt, "prompt_frames_per_s": 32 * n / dt, "ms_per_sweep": 1e3 * dt / n,
            "prompts": 32, "ranks": world,
            "workload": "config E: 5M Gaussians, 1920x1080, 32 prompts, tile bands x ranks",
            "timing": "wall clock per sweep incl. the host sync of each sweep's statistics, max over ranks"}


if __name__ == "__main__":
    main()
