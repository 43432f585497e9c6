"""Parity of the sm_100a path against the reference (golden fixtures) and the oracle.

Tolerances:
  * projection (means2d, inv_covs, depths, opacities, ids, rows): bitwise
  * binning (per-tile source-id lists, offsets, canonical_bytes): bitwise
  * coefficient map: max |dW| <= 2e-6 absolute (fp32 accumulation of fp64
    weights; the reference values are in [0, 1]); final T <= 1e-6
  * features: max |dF| <= 2e-5 * max |F_ref| per level (3xTF32 tensor cores)
  * relevancy (raw and filtered): max abs <= 1e-5
  * level, point, mask: identical
"""

import numpy as np
import pytest

import paper_2507_07136_b200 as sf
from conftest import (assert_selection_matches, golden_names, load_golden, make_camera,
                      random_scene)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

W_TOL = 2e-6
T_TOL = 1e-6
F_REL = 2e-5
R_TOL = 1e-5


@pytest.mark.parametrize("name", golden_names())
def test_projection_bitwise_vs_reference(name):
    scene, cam, z = load_golden(name)
    p = sf.project_scene(scene, cam)
    assert p.count == z["p_means2d"].shape[0]
    for f in ("means2d", "inv_covs", "depths", "opacities", "source_ids", "rows"):
        assert getattr(p, f).tobytes() == z["p_" + f].tobytes(), f


@pytest.mark.parametrize("name", golden_names())
def test_binning_bytes_vs_reference(name):
    scene, cam, z = load_golden(name)
    b = sf.bin_projected(sf.project_scene(scene, cam), cam)
    np.testing.assert_array_equal(b.tile_offsets, z["b_offsets"])
    assert b.canonical_bytes() == z["b_canonical_bytes"].tobytes()


@pytest.mark.parametrize("name", golden_names())
def test_splat_vs_reference(name):
    scene, cam, z = load_golden(name)
    cmap, st = sf.splat_multilevel(scene, cam, with_stats=True)
    assert cmap.data.shape == z["cmap"].shape
    assert np.abs(cmap.data - z["cmap"]).max(initial=0) <= W_TOL
    assert np.abs(st.final_transmittance - z["final_t"]).max(initial=0) <= T_TOL
    assert st.pairs_blended == int(z["pairs"])
    assert st.channels_per_gaussian == int(z["channels"])


@pytest.mark.parametrize("name", golden_names())
def test_decode_vs_reference(name):
    scene, cam, z = load_golden(name)
    fms = sf.decode(sf.splat_multilevel(scene, cam), scene.codebooks)
    for b in range(len(fms.maps)):
        ref = z["features"][b]
        scale = max(np.abs(ref).max(initial=0), 1e-30)
        assert np.abs(fms.maps[b] - ref).max(initial=0) <= F_REL * scale + 1e-7


@pytest.mark.parametrize("name", golden_names(require_query=True))
def test_query_pipeline_vs_reference(name):
    scene, cam, z = load_golden(name)
    q = sf.QueryEmbedding("q", z["q_vector"])
    res = sf.query_pipeline(scene, cam, q, z["q_canon"], window=int(z["q_window"]))
    for b, m in enumerate(res.level_maps):
        assert np.abs(m.data - z["q_filtered"][b]).max(initial=0) <= R_TOL
    assert_selection_matches(list(z["q_filtered"]), res.level, res.point, res.mask,
                             int(z["q_level"]), tuple(z["q_point"]), z["q_mask"])
    seg = sf.segment(res.chosen)
    np.testing.assert_array_equal(seg.mask, res.mask)
    # the lazily decoded features are the same as an explicit decode
    assert np.abs(res.feature_maps.maps[0] - z["features"][0]).max(initial=0) <= \
        F_REL * max(np.abs(z["features"][0]).max(initial=0), 1e-30) + 1e-7


@pytest.mark.parametrize("name", golden_names(require_query=True))
def test_eager_features_vs_reference(name):
    """query_pipeline(..., features="eager"): the features are decoded inside
    the frame -- by the blend kernel itself when sf_decode_fused (fused_s5:
    L=64, 3 x K=4, D=64), else by the tcgen05 GEMM over the coefficient map."""
    scene, cam, z = load_golden(name)
    q = sf.QueryEmbedding("q", z["q_vector"])
    res = sf.query_pipeline(scene, cam, q, z["q_canon"], window=int(z["q_window"]), features="eager")
    for b in range(z["features"].shape[0]):
        ref = z["features"][b]
        scale = max(np.abs(ref).max(initial=0), 1e-30)
        assert np.abs(res.feature_maps.maps[b] - ref).max(initial=0) <= F_REL * scale + 1e-7, b
    for b, m in enumerate(res.level_maps):
        assert np.abs(m.data - z["q_filtered"][b]).max(initial=0) <= R_TOL
    assert_selection_matches(list(z["q_filtered"]), res.level, res.point, res.mask,
                             int(z["q_level"]), tuple(z["q_point"]), z["q_mask"])
    assert np.abs(res.coefficient_map.data - z["cmap"]).max(initial=0) <= W_TOL


@pytest.mark.parametrize("opacity", [(0.2, 0.95), (0.8, 0.99)])
def test_fused_decode_matches_fp64_decode_of_the_map(opacity):
    """Fused blend+decode (D = 512, ragged 16x8 half tiles) against the fp64
    product of the coefficient map the same frame wrote; the opaque case
    routes pixels through the exact fp64 fixup, whose features are redone."""
    import torch
    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200.device import device_scene
    rng = np.random.default_rng(3)
    scene = random_scene(rng, 6000, num_levels=3, L=64, K=4, D=512, opacity_range=opacity)
    cam = make_camera(150, 101)
    assert N.load().sf_decode_fused(3, 64, 4, 512) == 1
    eng = device_scene(scene).engine
    out = eng.allocate(cam.width, cam.height, (0, 1, 2), coeff_map=True, final_t=True, features=True)
    eng.run(cam, (0, 1, 2), out)
    torch.cuda.synchronize()
    w = out.coeff_map.double()
    for b in range(3):
        atoms = torch.from_numpy(scene.codebooks[b].atoms).to(w.device).double()
        ref = w[:, :, 64 * b:64 * (b + 1)] @ atoms
        err = (out.features[b].double() - ref).abs().max().item()
        assert err <= F_REL * ref.abs().max().item(), (b, err)
    fix = int(out.host_stats()[0][N.STAT_FIXUPS]) if hasattr(N, "STAT_FIXUPS") else None
    ocm = O.splat_multilevel(scene, cam)
    assert np.abs(out.coeff_map.cpu().numpy() - ocm.data).max() <= W_TOL, fix


@pytest.mark.parametrize("W,H,G,extent", [(800, 600, 30000, 1.0), (1280, 720, 12000, 0.35)])
def test_persistent_splat_many_tiles_per_cta(W, H, G, extent):
    """k_splat_tc's persistent pipeline with many half tiles per CTA (3.7k and
    7.2k half tiles on 148 SMs): W/A slots alternate, the decode of one tile
    overlaps the blend of the next, and (extent 0.35) most tiles at the
    border are empty -- their features are stored as zeros without MMAs.
    Coefficient map, final T, features and relevancy against the oracle."""
    import torch
    from paper_2507_07136_b200.device import QuerySpec, device_scene
    rng = np.random.default_rng(17)
    scene = random_scene(rng, G, num_levels=3, L=64, K=4, D=64, image_extent=extent)
    cam = make_camera(W, H)
    qv = rng.standard_normal(64)
    canon = rng.standard_normal((4, 64))
    eng = device_scene(scene).engine
    out = eng.allocate(W, H, (0, 1, 2), coeff_map=True, final_t=True, features=True, query=True)
    eng.run(cam, (0, 1, 2), out, query=QuerySpec(qv, canon, 11, -1, 0.5))
    torch.cuda.synchronize()
    ref = O.query_pipeline(scene, cam, qv, canon, window=11, keep_features=True)
    assert np.abs(out.coeff_map.cpu().numpy() - ref.cmap.data).max() <= W_TOL
    feats = out.features.cpu().numpy()
    for b in range(3):
        f_ref = ref.features[b]
        assert np.abs(feats[b] - f_ref).max() <= F_REL * np.abs(f_ref).max(), b
        # pixels no Gaussian reaches decode to exact zeros
        zero = np.all(ref.cmap.data[:, :, 64 * b:64 * (b + 1)] == 0, axis=2)
        assert not np.any(feats[b][zero]), b
    raw = out.relevancy_raw.cpu().numpy()
    for b in range(3):
        assert np.abs(raw[b] - ref.raw_maps[b]).max() <= R_TOL


@pytest.mark.parametrize("name", golden_names(require_query=True))
def test_relevancy_ops_vs_reference(name):
    scene, cam, z = load_golden(name)
    q = sf.QueryEmbedding("q", z["q_vector"])
    maps = []
    for b in range(z["features"].shape[0]):
        raw = sf.relevancy_map(z["features"][b], q, z["q_canon"], level=b)
        assert np.abs(raw.data - z["q_raw"][b]).max(initial=0) <= 1e-12
        filt = sf.mean_filter(raw, int(z["q_window"]))
        assert np.abs(filt.data - z["q_filtered"][b]).max(initial=0) <= 1e-12
        maps.append(filt)
    if scene.num_gaussians:
        lv, chosen = sf.select_level(maps)
        assert_selection_matches(list(z["q_filtered"]), lv, sf.localize(chosen),
                                 sf.segment(chosen).mask, int(z["q_level"]), tuple(z["q_point"]))


def test_config_a_full_path():
    """SURVEY 8(d) config A (10k G, 256x256, 3 levels, L=64, K=4, D=512)."""
    import os
    from conftest import GOLDEN
    from paper_2507_07136_b200 import synthetic
    z = np.load(os.path.join(GOLDEN, "configA_binning.npz"))
    scene = synthetic.make_scene(10_000)
    cam = synthetic.make_camera(256, 256)
    p = sf.project_scene(scene, cam)
    assert p.means2d.tobytes() == z["p_means2d"].tobytes()
    assert p.inv_covs.tobytes() == z["p_inv_covs"].tobytes()
    assert p.depths.tobytes() == z["p_depths"].tobytes()
    b = sf.bin_projected(p, cam)
    np.testing.assert_array_equal(b.tile_offsets, z["b_offsets"])
    np.testing.assert_array_equal(b.projected.source_ids[b.tile_entries], z["b_source_ids"])
    cmap, st = sf.splat_multilevel(scene, cam, with_stats=True)
    assert st.pairs_blended == 175_770
    assert np.abs(cmap.data[[5, 130]] - z["cmap_rows"]).max() <= W_TOL
    assert np.abs(st.final_transmittance[::8] - z["final_t"]).max() <= 1e-6
    # decode + query against the oracle (fp64) on the same inputs
    ocm = O.splat_multilevel(scene, cam)
    qv, canon = synthetic.make_query()
    fms = sf.decode(cmap, scene.codebooks)
    for lv in range(3):
        ref = O.decode_level(ocm.level_view(lv), scene.codebooks[lv].atoms)
        assert np.abs(fms.maps[lv] - ref).max() <= F_REL * np.abs(ref).max()
    res = sf.query_pipeline(scene, cam, sf.QueryEmbedding("q", qv), canon)
    ores = O.query_pipeline(scene, cam, qv, canon, window=11, keep_features=False)
    for lv in range(3):
        assert np.abs(res.level_maps[lv].data - ores.level_maps[lv]).max() <= R_TOL
    assert res.level == ores.level
    assert res.point == ores.point
    assert_selection_matches(list(ores.level_maps), res.level, res.point, res.mask, ores.level,
                             ores.point, O.segment(ores.level_maps[ores.level])[0])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_scenes_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    scene = random_scene(rng, num_gaussians=4000, num_levels=3, L=32, K=4, D=64)
    cam = make_camera(width=123, height=77)
    b = sf.bin_projected(sf.project_scene(scene, cam), cam)
    ob = O.bin_projected(O.project_scene(scene, cam), cam)
    assert b.canonical_bytes() == ob.canonical_bytes()
    cm, st = sf.splat_multilevel(scene, cam, with_stats=True)
    ocm, ost = O.splat_multilevel(scene, cam, binning=ob, with_stats=True)
    assert np.abs(cm.data - ocm.data).max() <= W_TOL
    assert st.pairs_blended == ost.pairs_blended


def test_permutation_invariance_byte_exact(rng):
    scene = random_scene(rng, num_gaussians=500, num_levels=2)
    cam = make_camera(48, 40)
    base = sf.splat_multilevel(scene, cam).data
    for _ in range(2):
        again = sf.splat_multilevel(scene.permuted(rng.permutation(500)), cam).data
        assert base.tobytes() == again.tobytes()


def test_fused_equals_per_level_byte_exact(rng):
    scene = random_scene(rng, num_gaussians=300, num_levels=3, L=16, K=4)
    cam = make_camera()
    fused = sf.splat_multilevel(scene, cam)
    for lv in range(3):
        single = sf.splat_sparse(scene, cam, lv)
        assert fused.level_view(lv).tobytes() == single.level_view(lv).tobytes()


def test_k_equals_l_and_one_hot(rng):
    scene = random_scene(rng, num_gaussians=200, num_levels=1, L=8, K=8)
    cam = make_camera()
    ocm = O.splat_multilevel(scene, cam)
    assert np.abs(sf.splat_multilevel(scene, cam).data - ocm.data).max() <= W_TOL


def test_wide_channel_blocks_match(rng):
    """L=256, 1 level -> the accumulator is split over two channel blocks."""
    scene = random_scene(rng, num_gaussians=300, num_levels=1, L=256, K=4, D=16)
    cam = make_camera(40, 36)
    ocm = O.splat_multilevel(scene, cam)
    cm = sf.splat_multilevel(scene, cam)
    assert np.abs(cm.data - ocm.data).max() <= W_TOL


def test_per_level_mass_equals_blended_opacity(rng):
    scene = random_scene(rng, num_gaussians=600, num_levels=2, L=16, K=4)
    cmap, stats = sf.splat_multilevel(scene, make_camera(), with_stats=True)
    for lv in range(2):
        np.testing.assert_allclose(cmap.level_view(lv).sum(axis=2), 1.0 - stats.final_transmittance,
                                   atol=1e-5)


def test_errors_raised_before_work(rng):
    scene = random_scene(rng, num_gaussians=5, L=16, K=2)
    bad = scene.permuted(np.arange(5))
    bad.coeff_indices = bad.coeff_indices.copy()
    bad.coeff_indices[0, 0, -1] = 40
    with pytest.raises(sf.ValidationError):
        sf.splat_sparse(bad, make_camera(), 0)
    with pytest.raises(sf.ValidationError):
        sf.splat_sparse(scene, make_camera(), 3)
    with pytest.raises(sf.ResourceLimitError):
        sf.splat_multilevel(scene, make_camera(), max_elements=100)
    with pytest.raises(sf.ValidationError):
        sf.splat_multilevel(scene, make_camera(), tile_size=8)
    q = sf.QueryEmbedding("q", np.ones(8))
    with pytest.raises(sf.ValidationError):
        sf.query_pipeline(scene, make_camera(), q, np.zeros((0, 8)))
    with pytest.raises(sf.ValidationError):
        sf.query_pipeline(scene, make_camera(), q, np.zeros((2, 8)), window=4)
    with pytest.raises(sf.ValidationError):
        sf.query_pipeline(scene, make_camera(), q, np.zeros((2, 8)), level=2)


def test_empty_scene(rng):
    scene = random_scene(rng, num_gaussians=0)
    cmap = sf.splat_multilevel(scene, make_camera())
    assert not cmap.data.any()
    b = sf.bin_projected(sf.project_scene(scene, make_camera()), make_camera())
    assert all(lst.size == 0 for lst in b.tile_lists)


def test_tensor_core_decode_matches_simt_crosscheck(rng):
    """tcgen05 3xTF32 decode vs the plain fp32 FMA-chain kernel, on a map with ragged M."""
    import torch
    from paper_2507_07136_b200 import _native as N
    from paper_2507_07136_b200.device import stream_ptr
    dev = torch.device("cuda")
    P, L, D = 128 * 37 + 5, 64, 512
    w = torch.from_numpy(rng.random((P, 3 * L)).astype(np.float32) / 8).to(dev)
    cb = torch.from_numpy(rng.standard_normal((L, D)).astype(np.float32)).to(dev)
    a = torch.empty((P, D), dtype=torch.float32, device=dev)
    s = torch.empty_like(a)
    lib = N.load()
    ws = torch.empty(int(lib.sf_decode_workspace_bytes(L, D)), dtype=torch.uint8, device=dev)
    N.check(lib.sf_decode(P, L, D, N.ptr(w[:, L:]), 3 * L, N.ptr(cb), N.ptr(a), N.ptr(ws), ws.numel(),
                          stream_ptr()))
    N.check(lib.sf_decode_simt(P, L, D, N.ptr(w[:, L:]), 3 * L, N.ptr(cb), N.ptr(s), stream_ptr()))
    ref = w[:, L:2 * L].double() @ cb.double()
    assert (a.double() - ref).abs().max().item() <= F_REL * ref.abs().max().item()
    assert (s.double() - ref).abs().max().item() <= F_REL * ref.abs().max().item()


@pytest.mark.parametrize("world,L", [(2, 64), (3, 64), (2, 128)])
def test_tile_bands_stitch_to_the_full_frame(rng, world, L):
    """tile-band sharding of one view.  Every rendered
    tile is the full frame's tile, so stitched bands equal the full frame
    exactly: coefficient map / features / final T on owned rows, filtered
    relevancy maps, and level / point / mask after the cross-band reduction."""
    from paper_2507_07136_b200.device import QuerySpec, device_scene
    from paper_2507_07136_b200.distributed import band_query, band_rows, combine_selection, mask_rows
    import torch

    scene = random_scene(rng, 3000, num_levels=3, L=L, K=4, D=128)  # L=128: relevancy from the map in HBM
    cam = make_camera(112, 90)
    qv = rng.standard_normal(scene.codebooks[0].atoms.shape[1])
    canon = rng.standard_normal((4, qv.shape[0]))
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    eng = device_scene(scene).engine
    levels = (0, 1, 2)
    full = eng.allocate(cam.width, cam.height, levels, coeff_map=True, final_t=True, features=True, query=True)
    eng.run(cam, levels, full, query=spec)
    st_i, st_f = full.host_stats()
    stats, outs = [], []
    for r in range(world):
        b = band_rows(cam.height, world, r)
        o = eng.allocate(cam.width, cam.height, levels, coeff_map=True, final_t=True, features=True, query=True)
        eng.run(cam, levels, o, query=spec, band=(b.y0, b.y1))
        torch.cuda.synchronize()
        y0, y1 = b.y0, b.y1
        assert torch.equal(o.coeff_map[y0:y1], full.coeff_map[y0:y1])
        assert torch.equal(o.final_t[y0:y1], full.final_t[y0:y1])
        assert torch.equal(o.features[:, y0:y1], full.features[:, y0:y1])
        assert torch.equal(o.relevancy_filtered[:, y0:y1], full.relevancy_filtered[:, y0:y1])
        from paper_2507_07136_b200.distributed import band_statistics
        stats.append(band_statistics(o, len(levels)))
        outs.append((b, o))
    level, idx, lo, hi = combine_selection(*zip(*stats))
    assert level == int(st_i[N_STAT_LEVEL()])
    assert divmod(idx, cam.width) == (int(st_i[4]), int(st_i[5]))
    assert lo == float(st_f[0]) and hi == float(st_f[1])
    for b, o in outs:
        mask_rows(o, level, lo, hi, 0.5, b.y0, b.y1)
        torch.cuda.synchronize()
        assert torch.equal(o.mask[b.y0:b.y1], full.mask[b.y0:b.y1])
    # the one-call helper (no process group: a world of one band = whole image)
    bq = band_query(eng, cam, levels, spec, 1, 0)
    assert bq.level == level and bq.point == divmod(idx, cam.width)
    assert torch.equal(bq.out.mask, full.mask)


def N_STAT_LEVEL():
    from paper_2507_07136_b200 import _native as N
    return N.STAT_LEVEL


def test_frame_pipeline_matches_serial_frames(rng):
    """device.FramePipeline (sf_render_frame_split: prepare stream + two render
    streams, two workspaces) gives every frame the same results as a serial frame."""
    import torch
    from paper_2507_07136_b200.device import FramePipeline, QuerySpec, device_scene
    scene = random_scene(rng, 4000, num_levels=3, L=64, K=4, D=64)
    cams = [make_camera(96, 70), make_camera(96, 70, fov=40.0), make_camera(96, 70, fov=50.0)]
    qv = rng.standard_normal(64)
    canon = rng.standard_normal((4, 64))
    spec = QuerySpec(qv, canon, 11, -1, 0.5)
    ds = device_scene(scene)
    eng = ds.engine
    levels = (0, 1, 2)
    ref = []
    for cam in cams:
        o = eng.allocate(96, 70, levels, coeff_map=False, features=True, query=True)
        eng.run(cam, levels, o, query=spec)
        ref.append(o)
    pipe = FramePipeline(ds, 96, 70, levels, coeff_map=False, features=True, query=True)
    order = cams * 2
    got = []
    for k0 in range(0, len(order), 2):  # two frames in flight (both buffers), then read them
        pipe.begin()
        outs = [pipe.enqueue(cam, levels, query=spec) for cam in order[k0:k0 + 2]]
        pipe.end()
        for o in outs:
            got.append((o.features.clone(), o.relevancy_filtered.clone(), o.mask.clone(), o.stats_i64.clone()))
    torch.cuda.synchronize()
    # bit for bit: the blend (tensor-core sums in a fixed order) and the exact
    # replay (ordered per-channel sums, no float atomics) are deterministic
    # (reference tests/test_rasterizer.py:153-158: results independent of workers)
    for k, (f, r, m, st) in enumerate(got):
        o = ref[k % 3]
        assert torch.equal(f, o.features)
        assert torch.equal(r, o.relevancy_filtered)
        assert torch.equal(m, o.mask)
        assert torch.equal(st[:8], o.stats_i64[:8])


def test_fixup_overflow_raises():
    """A frame with more early-exit-ambiguous pixels than the exact-replay list
    holds raises instead of keeping uncertified fp32 decisions.  The list holds
    W * H by default (cannot overflow); SF_FIXUP_CAPACITY lowers it, so the
    check runs in a subprocess on an opaque scene that has several ambiguous pixels."""
    import os
    import subprocess
    import sys
    code = r"""
import numpy as np, sys
sys.path.insert(0, 'tests')
import paper_2507_07136_b200 as sf
from paper_2507_07136_b200.errors import SplatfieldError
from conftest import random_scene, make_camera
rng = np.random.default_rng(11)
scene = random_scene(rng, 6000, num_levels=3, L=64, K=4, D=64, opacity_range=(0.8, 0.99))
cam = make_camera(128, 96)
try:
    sf.splat_multilevel(scene, cam, with_stats=True)
except SplatfieldError as e:
    assert "exact-replay capacity" in str(e), e
    print("raised")
else:
    print("no-raise")
"""
    env = dict(os.environ, SF_FIXUP_CAPACITY="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("raised"), r.stdout + r.stderr[-2000:]
    # the same frame at the default capacity replays every ambiguous pixel
    env.pop("SF_FIXUP_CAPACITY")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("no-raise"), r.stdout + r.stderr[-2000:]


def test_render_dense_vs_reference():
    """render_dense (rasterizer.py:206-272) against the reference's own outputs
    (tests/golden/dense_s6.npz): colours with stats, a 20-channel feature array
    (two 16-channel passes), and a background composite.  Values are blended in
    fp32: |d| <= 2e-6 for colours in [0, 1], 1e-5 x max|value| for features."""
    scene, cam, z = load_golden("dense_s6")
    fb, st = sf.render_dense(scene, cam, "color", with_stats=True)
    assert fb.tag == "color" and fb.data.shape == z["dense_color"].shape
    assert np.abs(fb.data - z["dense_color"]).max() <= W_TOL
    assert np.abs(st.final_transmittance - z["dense_color_t"]).max() <= T_TOL
    assert st.pairs_blended == int(z["dense_color_pairs"]) and st.channels_per_gaussian == 3
    fe = sf.render_dense(scene, cam, z["dense_feats"])
    assert fe.tag == "dense-feature"
    assert np.abs(fe.data - z["dense_feat"]).max() <= 1e-5 * np.abs(z["dense_feats"]).max()
    bg = sf.render_dense(scene, cam, "color", background=[0.2, 0.4, 0.6])
    assert np.abs(bg.data - z["dense_bg"]).max() <= W_TOL


def test_render_dense_contract(rng):
    """The reference's render_dense tests (test_rasterizer.py:67-163): linearity,
    one-hot coefficients == the sparse splat, permutation invariance, errors."""
    scene = random_scene(rng, num_gaussians=300, num_levels=1, L=16, K=4)
    cam = make_camera(40, 36)
    x = rng.standard_normal((300, 5))
    y = rng.standard_normal((300, 5))
    combo = sf.render_dense(scene, cam, 0.7 * x - 1.3 * y).data
    ref = 0.7 * sf.render_dense(scene, cam, x).data - 1.3 * sf.render_dense(scene, cam, y).data
    assert np.abs(combo - ref).max() <= 1e-5
    dense = np.zeros((300, 16))
    np.put_along_axis(dense, scene.coeff_indices[0].astype(np.int64), scene.coeff_values[0], axis=1)
    fb = sf.render_dense(scene, cam, dense)
    assert np.abs(fb.data - sf.splat_sparse(scene, cam, 0).level_view(0)).max() <= W_TOL
    base = sf.render_dense(scene, cam, "color").data
    assert base.tobytes() == sf.render_dense(scene.permuted(rng.permutation(300)), cam, "color").data.tobytes()
    with pytest.raises(sf.ResourceLimitError):
        sf.render_dense(scene, cam, rng.standard_normal((300, 64)), max_elements=1000)
    with pytest.raises(sf.ValidationError):
        sf.render_dense(scene, cam, "depth")
    with pytest.raises(sf.ValidationError):
        sf.render_dense(scene, cam, "color", background=[0.1, 0.2])
    empty = random_scene(rng, num_gaussians=0)
    e = sf.render_dense(empty, make_camera(8, 8), "color", background=[0.2, 0.4, 0.6])
    np.testing.assert_allclose(e.data[0, 0], [0.2, 0.4, 0.6])


@pytest.mark.parametrize("L,window,n_prompts,n_canon", [(64, 11, 5, 4), (128, 11, 5, 4), (32, 21, 5, 4),
                                                       (64, 11, 70, 4), (64, 11, 4, 9)])
def test_query_sweep_matches_per_prompt_pipelines(rng, L, window, n_prompts, n_canon):
    """query_sweep (one render, then the prompts' relevancy -- the map read once
    per 65 - n_canon prompts -- and batched filter / select / mask:
    sf_query_sweep) gives every prompt its own query_pipeline result.  Covers
    prompt chunking (70), the per-prompt passes (window 21 > the fused
    filter's, 9 canonicals > the sweep kernel's 8) and the oracle."""
    scene = random_scene(rng, 3000, num_levels=3, L=L, K=4, D=64)
    cam = make_camera(96, 72)
    canon = rng.standard_normal((n_canon, 64))
    queries = [sf.QueryEmbedding(f"q{i}", rng.standard_normal(64)) for i in range(n_prompts)]
    sweep = sf.query_sweep(scene, cam, queries, canon, window=window)
    assert len(sweep) == n_prompts
    check = range(n_prompts) if n_prompts <= 5 else [0, 7, 60, 61, 69]
    for i in check:
        q, r = queries[i], sweep[i]
        one = sf.query_pipeline(scene, cam, q, canon, window=window)
        ref = [m.data for m in one.level_maps]
        for b in range(3):
            # logit differences vs differences of logits: fp64 rounding only
            assert np.abs(r.level_maps[b].data - ref[b]).max() <= 1e-12
        assert_selection_matches(ref, r.level, r.point, r.mask, one.level, one.point)
        if i < 2:
            ores = O.query_pipeline(scene, cam, q.vector, canon, window=window, keep_features=False)
            for b in range(3):
                assert np.abs(r.level_maps[b].data - ores.level_maps[b]).max() <= R_TOL
    # the shared coefficient map is the multilevel splat
    assert np.array_equal(sweep[0].coefficient_map.data, sf.splat_multilevel(scene, cam).data)
    assert sf.query_sweep(scene, cam, [], canon) == []


def test_fused_decode_empty_half_tiles_store_exact_zeros(rng):
    """Half tiles no Gaussian contributes to skip the MMAs and store zero boxes:
    their features are exactly 0 (buffers pre-filled with NaN), the rest of the
    frame still matches the fp64 product of its coefficient map, and the fused
    relevancy there is sigmoid(0) = 0.5."""
    import torch
    from paper_2507_07136_b200.device import QuerySpec, device_scene
    scene = random_scene(rng, 2000, num_levels=3, L=64, K=4, D=512)
    scene.positions[:, 0] = -np.abs(scene.positions[:, 0]) - 0.3  # left part of the view only
    cam = make_camera(160, 96)
    eng = device_scene(scene).engine
    levels = (0, 1, 2)
    qv = rng.standard_normal(512)
    canon = rng.standard_normal((4, 512))
    out = eng.allocate(cam.width, cam.height, levels, coeff_map=True, features=True, query=True)
    out.features.fill_(float("nan"))
    out.relevancy_raw.fill_(float("nan"))
    eng.run(cam, levels, out, query=QuerySpec(qv, canon))
    torch.cuda.synchronize()
    w = out.coeff_map.double()
    empty = (w == 0).all(dim=2)
    assert empty.any() and not empty.all()
    for b in range(3):
        f = out.features[b]
        assert torch.isfinite(f).all()
        assert (f[empty] == 0).all()
        ref = w[:, :, 64 * b:64 * (b + 1)] @ torch.from_numpy(scene.codebooks[b].atoms).to(w.device).double()
        assert (f.double() - ref).abs().max().item() <= F_REL * ref.abs().max().item()
        assert (out.relevancy_raw[b][empty] == 0.5).all()


@pytest.mark.parametrize("L", [16, 256])
def test_sparse_equals_dense_coefficient_render(rng, L):
    """SURVEY 8(f) f1's cost-decoupling comparator: the dense render of the
    densified coefficient rows (render_dense, 16 channels per pass) is the
    sparse multilevel map (splat_multilevel; L = 256 spans four channel blocks)."""
    scene = random_scene(rng, 1500, num_levels=3, L=L, K=4, D=16)
    cam = make_camera(64, 48)
    rows = np.concatenate([scene.densified_coefficients(lv) for lv in range(3)], axis=1)
    sparse = sf.splat_multilevel(scene, cam, max_elements=1 << 40).data
    dense = sf.render_dense(scene, cam, rows, tag="coefficient", max_elements=1 << 40).data
    assert np.abs(sparse - dense).max() <= W_TOL


def test_query_sweep_ragged_image(rng):
    """A pixel count that is not a multiple of the sweep kernel's 256-pixel tile
    (and odd, so the relevancy rows are not 16-byte aligned): every prompt still
    equals its own query_pipeline."""
    scene = random_scene(rng, 2000, num_levels=3, L=64, K=4, D=32)
    cam = make_camera(97, 71)
    canon = rng.standard_normal((3, 32))
    queries = [sf.QueryEmbedding(f"q{i}", rng.standard_normal(32)) for i in range(11)]
    sweep = sf.query_sweep(scene, cam, queries, canon)
    for q, r in zip(queries, sweep):
        one = sf.query_pipeline(scene, cam, q, canon)
        ref = [m.data for m in one.level_maps]
        for b in range(3):
            assert np.abs(r.level_maps[b].data - ref[b]).max() <= 1e-12
        assert_selection_matches(ref, r.level, r.point, r.mask, one.level, one.point)


@pytest.mark.parametrize("features", ["lazy", "eager"])
def test_query_stream_matches_query_pipeline(rng, features):
    """QueryStream (pipelined frames, per-frame pinned H2D / D2H) returns every
    frame's query_pipeline result: level, point and mask, bit for bit."""
    from paper_2507_07136_b200 import synthetic
    scene = random_scene(rng, 3000, num_levels=3, L=64, K=4, D=512)
    canon = rng.standard_normal((4, 512))
    cams = [make_camera(96, 72)] + [synthetic.make_camera(96, 72) for _ in range(1)]
    qs = [sf.QueryEmbedding(f"q{i}", rng.standard_normal(512)) for i in range(5)]
    stream = sf.QueryStream(scene, 96, 72, canon, features=features)
    handles = [stream.submit(cams[i % 2], q) for i, q in enumerate(qs)]
    results = [stream.result(h) for h in handles]
    stream.close()
    for i, (q, r) in enumerate(zip(qs, results)):
        one = sf.query_pipeline(scene, cams[i % 2], q, canon, features=features, max_elements=1 << 40)
        assert (r.level, r.point, r.degenerate) == (one.level, one.point, one.degenerate)
        assert np.array_equal(r.mask, one.mask)


def test_query_stream_overflow_rerun(rng):
    """A streamed frame whose pairs overflow the pipeline's pair buffer is
    re-run through query_pipeline (which grows the buffer): same answer."""
    scene = random_scene(rng, 3000, num_levels=3, L=64, K=4, D=64)
    canon = rng.standard_normal((4, 64))
    cam = make_camera(96, 72)
    q = sf.QueryEmbedding("q", rng.standard_normal(64))
    stream = sf.QueryStream(scene, 96, 72, canon)
    for e in stream.pipe.engines:
        e.pair_capacity = 64  # far below the frame's pairs
    r = stream.result(stream.submit(cam, q))
    stream.close()
    one = sf.query_pipeline(scene, cam, q, canon)
    assert (r.level, r.point) == (one.level, one.point)
    assert np.array_equal(r.mask, one.mask)
    assert all(e.pair_capacity > 64 for e in stream.pipe.engines)


@pytest.mark.parametrize("world", [2, 3])
def test_band_sweep_stitches_to_the_full_sweep(rng, world):
    """Config E end to end on one GPU: every band renders once and sweeps all
    prompts over its owned rows; combining the bands' statistics selects each
    prompt's level / point / range exactly as the full-frame sweep, and the
    stitched filtered maps and masks equal it bit for bit."""
    import torch
    from paper_2507_07136_b200.device import device_scene
    from paper_2507_07136_b200.distributed import (band_sweep_statistics, combine_selection_many,
                                                   finish_band_sweep)
    scene = random_scene(rng, 3000, num_levels=3, L=64, K=4, D=64)
    cam = make_camera(112, 90)
    canon = rng.standard_normal((4, 64))
    prompts = rng.standard_normal((6, 64))
    levels = (0, 1, 2)
    eng = device_scene(scene).engine
    full = sf.query_sweep(scene, cam, [sf.QueryEmbedding(f"q{i}", p) for i, p in enumerate(prompts)], canon)
    parts = [band_sweep_statistics(eng, cam, levels, prompts, canon, world, r) for r in range(world)]
    mx, am, mn = (np.stack([p[k] for p in parts]) for k in (3, 4, 5))
    sel = combine_selection_many(mx, am, mn)
    W = cam.width
    for r, (band, filt, masks, *_ ) in enumerate(parts):
        bs = finish_band_sweep(band, filt, masks, sel, 0.5, W, cam.height)
        y0, y1 = band.y0, band.y1
        for i, res in enumerate(full):
            level, point, lo, hi, degenerate = bs.selections[i]
            assert (level, point) == (res.level, res.point)
            for b in range(3):
                assert np.array_equal(filt[i, b, y0:y1].cpu().numpy(), res.level_maps[b].data[y0:y1])
            assert np.array_equal(masks[i, y0:y1].cpu().numpy().astype(bool), res.mask[y0:y1])
