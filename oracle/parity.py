"""Full-frame parity of a GPU frame against the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Used by ``tests/test_gpu_parity_configs.py`` (the BASELINE configs A, B, C and
sampled bands of E) and by ``bench.py``'s ``parity`` leg, after the timed
region, on the benchmarked frame itself.  The product package never imports
this module.

``oracle_frame`` is the reference's query path stage by stage
(sparse_splat.py:243-297 with query.py:65-145: splat_multilevel -> decode ->
per level relevancy_map + mean_filter -> select_level -> localize ->
segment), run by the C oracle (``oracle/splat_oracle.c``); features are
produced one level at a time and handed to a callback, so a 1440x1080x3x512
frame needs one fp64 level (6.4 GB) in host memory at a time.  It is also the
``--impl reference`` step of bench.py (each call = one full frame).

``compare_frame`` checks a GPU frame against it with the DESIGN.md section 4
tolerances and returns a JSON-able report (max errors, mask flips and the
reference margins of any flip).
"""

from __future__ import annotations

import time

import numpy as np

from . import oracle as O

W_TOL = 2e-6      # coefficient map, absolute
T_TOL = 1e-6      # final transmittance
F_REL = 2e-5      # features, relative to max |F_ref| per level
R_TOL = 1e-5      # raw and filtered relevancy, absolute
TIE_MARGIN = 1e-12
MASK_DECIDED = 1e-9


def oracle_frame(scene, cam, qv, canon, *, window=11, levels=(0, 1, 2), tile_rows=None, on_features=None,
                 query=True):
    """The reference frame on the CPU oracle.  Returns a dict with the binning,
    coefficient map, final T, raw / filtered maps, level, point, mask and
    per-stage seconds; ``on_features(b, F_b)`` receives each level's fp64
    features (rows of ``tile_rows`` only when given)."""
    t = {}
    t0 = time.perf_counter()
    proj = O.project_scene(scene, cam)
    t["project"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    binning = O.bin_projected(proj, cam)
    t["bin"] = time.perf_counter() - t0
    tiles_x, tiles_y = binning.tiles_x, binning.tiles_y
    tr = None
    y0, y1 = 0, int(cam.height)
    if tile_rows is not None:
        r0, r1 = tile_rows
        tr = (r0 * tiles_x, min(r1, tiles_y) * tiles_x)
        y0, y1 = r0 * 16, min(r1 * 16, int(cam.height))
    t0 = time.perf_counter()
    cmap, st = O.splat_levels(scene, cam, levels, binning=binning, tile_range=tr, with_stats=True)
    t["splat"] = time.perf_counter() - t0
    raws, maps = [], []
    t["decode"] = t["relevancy"] = t["filter"] = 0.0
    for b, lv in enumerate(levels):
        t0 = time.perf_counter()
        f = O.decode_level(cmap.data[y0:y1, :, b * cmap.L:(b + 1) * cmap.L], scene.codebooks[lv].atoms)
        t["decode"] += time.perf_counter() - t0
        if on_features is not None:
            on_features(b, f)
        if query:
            t0 = time.perf_counter()
            raw = O.relevancy_map(f, qv, canon)
            t["relevancy"] += time.perf_counter() - t0
            raws.append(raw)
            if tile_rows is None:
                t0 = time.perf_counter()
                maps.append(O.mean_filter(raw, window))
                t["filter"] += time.perf_counter() - t0
        del f
    out = {"binning": binning, "cmap": cmap, "final_t": st.final_transmittance, "rows": (y0, y1),
           "raw": raws, "filtered": maps, "seconds": t}
    if query and tile_rows is None:
        t0 = time.perf_counter()
        level = O.select_level(maps)
        point = O.localize(maps[level])
        mask, degenerate = O.segment(maps[level])
        t["select"] = time.perf_counter() - t0
        out.update(level=level, point=point, mask=mask, degenerate=degenerate)
    t["total"] = sum(v for v in t.values())
    return out


def _max_abs(a, b, chunk=1 << 22):
    """max |a - b| over flattened arrays, in chunks (bounded temporaries)."""
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    m = 0.0
    for i in range(0, a.size, chunk):
        d = np.abs(a[i:i + chunk].astype(np.float64) - b[i:i + chunk])
        if d.size:
            m = max(m, float(np.nanmax(d)) if not np.isnan(d).all() else float("nan"))
    return m


def selection_report(ref_maps, level, point, mask, ref_level, ref_point, threshold=0.5):
    """level / point / mask identity, tie-aware (tests/conftest.py
    assert_selection_matches): a differing choice is accepted only where the
    reference's own values tie within TIE_MARGIN; mask pixels are compared
    where the reference's normalised value is farther than 1e-9 from the
    threshold, and every flip is counted with its margin."""
    maxima = np.array([float(m.max()) for m in ref_maps])
    rep = {"level": int(level), "ref_level": int(ref_level), "point": [int(point[0]), int(point[1])],
           "ref_point": [int(ref_point[0]), int(ref_point[1])]}
    ok = True
    if level != ref_level:
        rep["level_margin"] = float(maxima[ref_level] - maxima[level])
        ok &= rep["level_margin"] <= TIE_MARGIN
    m = ref_maps[level]
    if tuple(point) != tuple(ref_point):
        rep["point_margin"] = float(m.max() - m[tuple(point)])
        ok &= rep["point_margin"] <= TIE_MARGIN
    lo, hi = float(m.min()), float(m.max())
    mask = np.asarray(mask, dtype=bool)
    if hi <= lo:
        rep["mask_flips"] = int(mask.sum())
        ok &= rep["mask_flips"] == 0
    else:
        norm = (m - lo) / (hi - lo)
        want = norm > threshold
        flips = mask != want
        decided = np.abs(norm - threshold) > MASK_DECIDED
        rep["mask_pixels"] = int(want.sum())
        rep["mask_flips"] = int(flips.sum())
        rep["mask_flips_decided"] = int((flips & decided).sum())
        if flips.any():
            rep["mask_flip_max_margin"] = float(np.abs(norm[flips] - threshold).max())
        ok &= rep["mask_flips_decided"] == 0
    rep["ok"] = bool(ok)
    return rep


def compare_frame(scene, cam, qv, canon, gpu, *, window=11, levels=(0, 1, 2), tile_rows=None):
    """Compare a GPU frame with the oracle frame of the same inputs.

    ``gpu`` maps: ``tile_offsets``/``tile_ids`` (the frame's own per-tile
    lists as source ids, optional), ``cmap`` (H,W,nl*L), ``final_t`` (H,W),
    ``features`` (callable b -> (H,W,D) fp32), ``raw`` / ``filtered``
    (nl,H,W) fp64, ``level``, ``point``, ``mask`` (H,W) -- the last four only
    for full frames.  Returns the report; ``report["ok"]`` is the verdict."""
    errs = {"features_rel": []}
    ref_f = {}

    def keep(b, f):
        gf = gpu["features"](b)
        y0, y1 = ref["rows"] if "rows" in ref else (0, f.shape[0])
        gf = gf[y0:y1] if gf.shape[0] != f.shape[0] else gf
        scale = max(float(np.abs(f).max(initial=0.0)), 1e-30)
        errs["features_rel"].append(_max_abs(gf, f) / scale)
        ref_f[b] = None

    ref = {}
    t0 = time.perf_counter()
    # rows are known before the callback runs
    if tile_rows is not None:
        ref["rows"] = (tile_rows[0] * 16, min(tile_rows[1] * 16, int(cam.height)))
    o = oracle_frame(scene, cam, qv, canon, window=window, levels=levels, tile_rows=tile_rows, on_features=keep)
    rep = {"oracle_s": round(time.perf_counter() - t0, 2), "oracle_stage_s": {k: round(v, 3) for k, v in
                                                                          o["seconds"].items()}}
    y0, y1 = o["rows"]
    rep["rows"] = [y0, y1]
    ok = True
    b = o["binning"]
    rep["pairs_ref"] = int(b.tile_offsets[-1])
    if gpu.get("tile_offsets") is not None:
        same_off = np.array_equal(np.asarray(gpu["tile_offsets"], dtype=np.int64), b.tile_offsets)
        ref_ids = b.projected.source_ids[b.tile_entries]
        same_ids = same_off and np.array_equal(np.asarray(gpu["tile_ids"], dtype=np.int64), ref_ids)
        rep["binning_identical"] = bool(same_off and same_ids)
        ok &= rep["binning_identical"]
    cm = np.asarray(gpu["cmap"])[y0:y1] if gpu.get("cmap") is not None else None
    if cm is not None:
        rep["cmap_max_abs"] = _max_abs(cm, o["cmap"].data[y0:y1])
        ok &= rep["cmap_max_abs"] <= W_TOL
    if gpu.get("final_t") is not None:
        rep["final_t_max_abs"] = _max_abs(np.asarray(gpu["final_t"])[y0:y1], o["final_t"][y0:y1])
        ok &= rep["final_t_max_abs"] <= T_TOL
    rep["features_rel"] = errs["features_rel"]
    ok &= all(e <= F_REL for e in errs["features_rel"])
    if gpu.get("raw") is not None and o["raw"]:
        rep["raw_max_abs"] = max(_max_abs(np.asarray(gpu["raw"][i])[y0:y1], o["raw"][i]) for i in range(len(levels)))
        ok &= rep["raw_max_abs"] <= R_TOL
    if tile_rows is None and gpu.get("filtered") is not None:
        rep["filtered_max_abs"] = max(_max_abs(gpu["filtered"][i], o["filtered"][i]) for i in range(len(levels)))
        ok &= rep["filtered_max_abs"] <= R_TOL
        sel = selection_report(o["filtered"], gpu["level"], gpu["point"], gpu["mask"], o["level"], o["point"])
        rep["selection"] = sel
        ok &= sel["ok"]
    rep["ok"] = bool(ok)
    rep["tolerances"] = {"cmap_abs": W_TOL, "final_t_abs": T_TOL, "features_rel": F_REL, "relevancy_abs": R_TOL,
                         "binning": "byte-identical", "level/point/mask": "identical (tie-aware)"}
    return rep


def gpu_frame(scene, cam, qv, canon, *, window=11, levels=(0, 1, 2)):
    """One GPU frame of the product path with every output materialised --
    the fused blend + decode kernel with the coefficient map also written --
    as the ``gpu`` mapping of ``compare_frame`` (features fetched per level)."""
    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200.device import QuerySpec, device_scene

    W, H = int(cam.width), int(cam.height)
    ds = device_scene(scene)
    eng = ds.engine
    out = eng.allocate(W, H, levels, coeff_map=True, final_t=True, features=True, query=True)
    eng.run(cam, levels, out, query=QuerySpec(np.asarray(qv, np.float64), np.asarray(canon, np.float64), window,
                                              -1, 0.5))
    si, sf = out.host_stats()
    offs, rows = eng.tile_lists(W, H, len(levels), int(si[N.STAT_PAIRS]))
    ids = ds.ids.cpu().numpy()
    return {
        "tile_offsets": offs, "tile_ids": ids[rows],
        "cmap": out.coeff_map.cpu().numpy(), "final_t": out.final_t.cpu().numpy(),
        "features": lambda b: out.features[b].cpu().numpy(),
        "raw": out.relevancy_raw.cpu().numpy(), "filtered": out.relevancy_filtered.cpu().numpy(),
        "level": int(si[N.STAT_LEVEL]), "point": (int(si[N.STAT_ROW]), int(si[N.STAT_COL])),
        "mask": out.mask.cpu().numpy().astype(bool), "fixups": int(si[N.STAT_FIXUPS]),
        "pairs": int(si[N.STAT_PAIRS]), "visible": int(si[N.STAT_VISIBLE]), "_out": out,
    }
