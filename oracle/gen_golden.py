"""Generate tests/golden/*.npz from the REFERENCE implementation (test infrastructure).

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Each fixture stores the inputs (scene arrays, camera, query) and the
reference's own outputs for the hot path: project_scene (projection.py:311),
bin_projected (projection.py:379, as CSR of source ids), splat_multilevel
(sparse_splat.py:178) coefficient map + RenderStats, decode (:183),
relevancy_map + mean_filter per level, select_level / localize / segment.
The GPU box has no /root/reference: tests read only these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, "/root/reference/pkg/src")

from splatfield import projection as RP  # noqa: E402
from splatfield import query as RQ  # noqa: E402
from splatfield import sparse_splat as RS  # noqa: E402
from splatfield.core import Codebook, Scene, SceneConfig  # noqa: E402


def random_scene(rng, num_gaussians=50, num_levels=1, L=16, K=4, D=8, image_extent=1.0,
                 opacity_range=(0.2, 0.95)):
    """Same distribution and draw order as the reference's tests/conftest.py:8-50."""
    cfg = SceneConfig(num_levels=num_levels, L=L, K=K, D=D)
    g = num_gaussians
    quats = rng.standard_normal((g, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    idx = np.zeros((num_levels, g, K), dtype=np.uint16)
    val = np.zeros((num_levels, g, K), dtype=np.float32)
    for lv in range(num_levels):
        for i in range(g):
            cols = np.sort(rng.choice(L, size=K, replace=False)).astype(np.uint16)
            raw = rng.random(K).astype(np.float64) + 1e-3
            idx[lv, i] = cols
            val[lv, i] = (raw / raw.sum()).astype(np.float32)
    codebooks = tuple(Codebook(rng.standard_normal((L, D)).astype(np.float32), level=lv)
                      for lv in range(num_levels))
    return Scene(
        positions=(rng.uniform(-image_extent, image_extent, (g, 3)) * np.array([1.0, 1.0, 0.4])).astype(np.float32),
        rotations=quats.astype(np.float32),
        scales=rng.uniform(0.03, 0.15, (g, 3)).astype(np.float32),
        opacities=rng.uniform(*opacity_range, g).astype(np.float32),
        colors=rng.uniform(0, 1, (g, 3)).astype(np.float32),
        coeff_indices=idx, coeff_values=val, codebooks=codebooks, config=cfg)


def camera(w, h, fov=45.0, pos=(0.0, 0.0, -3.0)):
    return RP.Camera.look_at(position=pos, target=(0.0, 0.0, 0.0), fov_y_deg=fov, width=w, height=h)


def dump(name, scene, cam, *, query_seed=None, window=5, with_query=True):
    cfg = scene.config
    d = dict(
        positions=scene.positions, rotations=scene.rotations, scales=scene.scales,
        opacities=scene.opacities, colors=scene.colors, coeff_indices=scene.coeff_indices,
        coeff_values=scene.coeff_values, ids=scene.ids,
        codebooks=np.stack([cb.atoms for cb in scene.codebooks]),
        config=np.array([cfg.num_levels, cfg.L, cfg.K, cfg.D], dtype=np.int64),
        cam_R=cam.rotation, cam_t=cam.translation,
        cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near]),
        cam_size=np.array([cam.width, cam.height], dtype=np.int64),
    )
    proj = RP.project_scene(scene, cam)
    d.update(p_means2d=proj.means2d, p_inv_covs=proj.inv_covs, p_depths=proj.depths,
             p_opacities=proj.opacities, p_source_ids=proj.source_ids, p_rows=proj.rows)
    b = RP.bin_projected(proj, cam)
    lens = np.array([lst.size for lst in b.tile_lists], dtype=np.int64)
    d.update(b_offsets=np.concatenate([[0], np.cumsum(lens)]).astype(np.int64),
             b_source_ids=(np.concatenate([b.projected.source_ids[lst] for lst in b.tile_lists])
                           if lens.sum() else np.zeros(0, np.int64)).astype(np.int64),
             b_canonical_bytes=np.frombuffer(b.canonical_bytes(), dtype=np.uint8))
    cmap, stats = RS.splat_multilevel(scene, cam, with_stats=True)
    d.update(cmap=cmap.data, final_t=stats.final_transmittance,
             pairs=np.int64(stats.pairs_blended), channels=np.int64(stats.channels_per_gaussian))
    fms = RS.decode(cmap, scene.codebooks)
    d.update(features=np.stack(fms.maps))
    if with_query:
        r = np.random.default_rng(query_seed if query_seed is not None else 7)
        qv = r.standard_normal(cfg.D)
        canon = r.standard_normal((4, cfg.D))
        q = RQ.QueryEmbedding(name="q", vector=qv)
        res = RS.query_pipeline(scene, cam, q, canon, window=window, instrument=False)
        seg = RQ.segment(res.chosen)
        raws = np.stack([RQ.relevancy_map(fms.maps[bb], q, canon, level=lv).data
                         for bb, lv in enumerate(cmap.levels)])
        d.update(q_vector=qv, q_canon=canon, q_window=np.int64(window), q_raw=raws,
                 q_filtered=np.stack([m.data for m in res.level_maps]),
                 q_level=np.int64(res.level), q_point=np.array(res.point, dtype=np.int64),
                 q_mask=seg.mask, q_degenerate=np.bool_(seg.degenerate))
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **d)
    return path, os.path.getsize(path)


def fused_fixtures():
    """Shapes on which the blend kernel decodes features itself (sf_decode_fused:
    L = 64, levels * K = 12, D % 32 == 0): ragged image, opaque enough that
    early exit and the fp64 fixup replay occur."""
    made = []
    rng = np.random.default_rng(1005)
    sc = random_scene(rng, num_gaussians=1500, num_levels=3, L=64, K=4, D=64, opacity_range=(0.5, 0.98))
    made.append(dump("fused_s5", sc, camera(37, 29)))
    return made


def dense_fixtures():
    """render_dense (rasterizer.py:206-272): colours, a 20-channel feature array
    (two 16-channel GPU passes) and a background composite, ragged image."""
    from splatfield import rasterizer as RR
    rng = np.random.default_rng(1006)
    sc = random_scene(rng, num_gaussians=400, num_levels=1, L=16, K=4, D=8, opacity_range=(0.3, 0.97))
    cam = camera(45, 37)
    feats = rng.standard_normal((400, 20))
    col, st = RR.render_dense(sc, cam, "color", with_stats=True)
    fe = RR.render_dense(sc, cam, feats)
    bg = RR.render_dense(sc, cam, "color", background=[0.2, 0.4, 0.6])
    d = dict(positions=sc.positions, rotations=sc.rotations, scales=sc.scales, opacities=sc.opacities,
             colors=sc.colors, coeff_indices=sc.coeff_indices, coeff_values=sc.coeff_values, ids=sc.ids,
             codebooks=np.stack([cb.atoms for cb in sc.codebooks]),
             config=np.array([1, 16, 4, 8], dtype=np.int64),
             cam_R=cam.rotation, cam_t=cam.translation,
             cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near]),
             cam_size=np.array([cam.width, cam.height], dtype=np.int64),
             dense_feats=feats, dense_color=col.data, dense_color_t=st.final_transmittance,
             dense_color_pairs=np.int64(st.pairs_blended), dense_feat=fe.data, dense_bg=bg.data)
    path = os.path.join(OUT, "dense_s6.npz")
    np.savez_compressed(path, **d)
    return [(path, os.path.getsize(path))]


def io_fixtures():
    """Reference-written files (io.py): an LSV2 scene (3 levels, K = 4, odd K = 3
    variant), a framebuffer and a query set, for byte-exact format tests."""
    from splatfield import io as RIO
    from splatfield import rasterizer as RR
    from splatfield.query import QueryEmbedding as RQE
    made = []
    for name, (g, nl, L, K, D) in (("io_scene_k4", (300, 3, 16, 4, 8)), ("io_scene_k3", (120, 2, 8, 3, 5))):
        rng = np.random.default_rng(1007 + K)
        sc = random_scene(rng, num_gaussians=g, num_levels=nl, L=L, K=K, D=D)
        path = os.path.join(OUT, name + ".lsv2")
        RIO.save_scene(path, sc)
        made.append((path, os.path.getsize(path)))
    fb = RR.Framebuffer(data=np.random.default_rng(3).random((7, 5, 3)), tag="color")
    path = os.path.join(OUT, "io_frame.fbuf")
    RIO.dump_framebuffer(path, fb)
    made.append((path, os.path.getsize(path)))
    r = np.random.default_rng(4)
    qs = RIO.QuerySet(dim=6, canonicals=r.standard_normal((4, 6)),
                      queries=[RQE(name="chair", vector=r.standard_normal(6)),
                               RQE(name="lamp", vector=r.standard_normal(6))],
                      gt_mask_paths={"lamp": "masks/lamp.fbuf"})
    path = os.path.join(OUT, "io_queries.json")
    RIO.save_query_set(path, qs)
    made.append((path, os.path.getsize(path)))
    return made


def train_fixtures():
    """forward_loss + backward (train.py:201-344) on a small scene: loss, dL/dlogits,
    dL/datoms, with a validity mask and the cosine term, and without either."""
    from splatfield import train as RT
    made = []
    for name, (cosw, use_mask) in (("train_s8", (0.5, True)), ("train_s9", (0.0, False))):
        rng = np.random.default_rng(1008 if use_mask else 1009)
        sc = random_scene(rng, num_gaussians=300, num_levels=2, L=8, K=2, D=8)
        cam = camera(40, 32)
        fld = RT.TrainableField(logits=rng.standard_normal((2, 300, 8)),
                                codebooks=rng.standard_normal((2, 8, 8)))
        targets = rng.standard_normal((2, 32, 40, 8))
        mask = rng.random((32, 40)) > 0.2 if use_mask else None
        batch = RT.TrainingBatch(camera=cam, targets=targets, mask=mask)
        cfg = RT.TrainConfig(cosine_weight=cosw)
        loss, cache = RT.forward_loss(fld, sc, batch, cfg)
        grads = RT.backward(cache)
        d = dict(positions=sc.positions, rotations=sc.rotations, scales=sc.scales, opacities=sc.opacities,
                 colors=sc.colors, coeff_indices=sc.coeff_indices, coeff_values=sc.coeff_values, ids=sc.ids,
                 codebooks=np.stack([cb.atoms for cb in sc.codebooks]),
                 config=np.array([2, 8, 2, 8], dtype=np.int64),
                 cam_R=cam.rotation, cam_t=cam.translation,
                 cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near]),
                 cam_size=np.array([cam.width, cam.height], dtype=np.int64),
                 t_logits=fld.logits, t_codebooks=fld.codebooks, t_targets=targets,
                 t_mask=mask if mask is not None else np.zeros(0, bool), t_cosine=np.float64(cosw),
                 t_loss=np.float64(loss), t_grad_logits=grads.logits, t_grad_codebooks=grads.codebooks,
                 t_coeff_maps=cache.coeff_maps)
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **d)
        made.append((path, os.path.getsize(path)))
    return made


def train_field_fixtures():
    """init_field (k-means seeding) + train_field (train.py:347-518): two batches,
    a holdout, 6 Adam iterations; and the random-codebook init."""
    from splatfield import train as RT
    made = []
    rng = np.random.default_rng(1010)
    sc = random_scene(rng, num_gaussians=400, num_levels=2, L=8, K=2, D=8)
    cams = [camera(40, 32), camera(40, 32, pos=(0.4, 0.1, -3.0)), camera(40, 32, pos=(-0.3, 0.2, -3.0))]
    batches = [RT.TrainingBatch(camera=c, targets=rng.standard_normal((2, 32, 40, 8)),
                                mask=(rng.random((32, 40)) > 0.1) if i == 1 else None)
               for i, c in enumerate(cams)]
    cfg = RT.TrainConfig(lr_logits=0.05, lr_codebook=0.02, cosine_weight=0.25)
    init = RT.init_field(sc, batches[:2], seed=3)
    init_r = RT.init_field(sc, batches[:2], seed=4, codebook_init="random")
    res = RT.train_field(sc, batches[:2], 6, cfg, seed=3, holdout=batches[2])
    d = dict(positions=sc.positions, rotations=sc.rotations, scales=sc.scales, opacities=sc.opacities,
             colors=sc.colors, coeff_indices=sc.coeff_indices, coeff_values=sc.coeff_values, ids=sc.ids,
             codebooks=np.stack([cb.atoms for cb in sc.codebooks]),
             config=np.array([2, 8, 2, 8], dtype=np.int64),
             cam_R=cams[0].rotation, cam_t=cams[0].translation,
             cam_intr=np.array([cams[0].fx, cams[0].fy, cams[0].cx, cams[0].cy, cams[0].near]),
             cam_size=np.array([40, 32], dtype=np.int64),
             cams_pos=np.array([(0.0, 0.0, -3.0), (0.4, 0.1, -3.0), (-0.3, 0.2, -3.0)]),
             t_targets=np.stack([b.targets for b in batches]), t_mask1=batches[1].mask,
             i_logits=init.logits, i_codebooks=init.codebooks, r_codebooks=init_r.codebooks,
             f_curve=np.array(res.loss_curve), f_logits=res.field.logits, f_codebooks=res.field.codebooks,
             f_coeff_indices=res.scene.coeff_indices, f_coeff_values=res.scene.coeff_values,
             f_holdout=np.array([res.holdout_initial, res.holdout_final]))
    path = os.path.join(OUT, "train_field_s10.npz")
    np.savez_compressed(path, **d)
    made.append((path, os.path.getsize(path)))
    return made


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--only-train" in sys.argv:
        for p, sz in train_fixtures() + train_field_fixtures():
            print(f"{os.path.basename(p)}: {sz / 1024:.1f} KiB")
        return
    if "--only-io" in sys.argv:
        for p, sz in io_fixtures():
            print(f"{os.path.basename(p)}: {sz / 1024:.1f} KiB")
        return
    if "--only-dense" in sys.argv:
        for p, sz in dense_fixtures():
            print(f"{os.path.basename(p)}: {sz / 1024:.1f} KiB")
        return
    if "--only-fused" in sys.argv:
        for p, sz in fused_fixtures():
            print(f"{os.path.basename(p)}: {sz / 1024:.1f} KiB")
        return
    made = fused_fixtures() + dense_fixtures() + io_fixtures() + train_fixtures() + train_field_fixtures()
    # 1. reference-test-like scenes (tests/conftest.py distribution)
    for seed, (g, nl, L, K, D, w, h) in enumerate([
        (50, 1, 16, 4, 8, 32, 32),
        (300, 3, 16, 4, 8, 48, 40),
        (1000, 3, 64, 4, 8, 61, 45),
        (200, 2, 8, 8, 8, 40, 40),       # K == L
        (500, 1, 64, 4, 16, 40, 40),     # acceptance-suite L/K/D (test_acceptance.py:48-58)
    ]):
        rng = np.random.default_rng(1000 + seed)
        sc = random_scene(rng, num_gaussians=g, num_levels=nl, L=L, K=K, D=D)
        made.append(dump(f"random_s{seed}", sc, camera(w, h)))
    # 2. permuted, non-contiguous ids (canonical order must come from (depth, id))
    rng = np.random.default_rng(77)
    sc = random_scene(rng, num_gaussians=400, num_levels=3, L=16, K=4, D=8)
    perm = rng.permutation(400)
    sc = sc.permuted(perm)
    sc.ids = (rng.permutation(400) * 7 - 1000).astype(np.int64)
    made.append(dump("permuted_ids", sc, camera(48, 40)))
    # 3. exact depth ties resolved by id (test_projection.py:205-211 pattern)
    rng = np.random.default_rng(5)
    sc = random_scene(rng, num_gaussians=64, num_levels=1, L=16, K=4, D=8)
    sc.positions[:, 2] = np.float32(0.1)  # every Gaussian at the same depth
    sc.ids = rng.permutation(64).astype(np.int64) * 3
    made.append(dump("depth_ties", sc, camera(32, 32)))
    # 4. empty and fully culled scenes
    rng = np.random.default_rng(9)
    sc = random_scene(rng, num_gaussians=0, num_levels=1, L=16, K=4, D=8)
    made.append(dump("empty", sc, camera(20, 12), with_query=True))
    sc = random_scene(rng, num_gaussians=30, num_levels=1, L=16, K=4, D=8)
    sc.positions[:, 2] = np.float32(-10.0)  # behind the camera
    made.append(dump("behind_camera", sc, camera(24, 24)))
    # 5. ragged image (partial edge tiles) with high opacity (early exit exercised)
    rng = np.random.default_rng(11)
    sc = random_scene(rng, num_gaussians=600, num_levels=2, L=16, K=4, D=8, opacity_range=(0.7, 0.98))
    made.append(dump("ragged_opaque", sc, camera(37, 29)))
    # 6. config A (SURVEY 8(d) generator, 10k Gaussians, 256x256, 3 levels, D=512) --
    #    projection + binning + coefficient map only (features would be 800 MB)
    sys.path.insert(0, os.path.join(HERE, ".."))
    from paper_2507_07136_b200 import synthetic
    s = synthetic.make_scene(10_000)
    scA = Scene(positions=s.positions, rotations=s.rotations, scales=s.scales, opacities=s.opacities,
                colors=s.colors, coeff_indices=s.coeff_indices, coeff_values=s.coeff_values,
                codebooks=tuple(Codebook(cb.atoms, level=cb.level) for cb in s.codebooks),
                config=SceneConfig(3, 64, 4, 512))
    camA = camera(256, 256)
    proj = RP.project_scene(scA, camA)
    b = RP.bin_projected(proj, camA)
    lens = np.array([lst.size for lst in b.tile_lists], dtype=np.int64)
    cmap, stats = RS.splat_multilevel(scA, camA, with_stats=True)
    path = os.path.join(OUT, "configA_binning.npz")
    np.savez_compressed(
        path, p_means2d=proj.means2d, p_inv_covs=proj.inv_covs, p_depths=proj.depths,
        p_rows=proj.rows, b_offsets=np.concatenate([[0], np.cumsum(lens)]).astype(np.int64),
        b_source_ids=np.concatenate([b.projected.source_ids[lst] for lst in b.tile_lists]).astype(np.int64),
        pairs=np.int64(stats.pairs_blended),
        cmap_rows=cmap.data[[5, 130]], final_t=stats.final_transmittance[::8].astype(np.float32))
    made.append((path, os.path.getsize(path)))
    for p, sz in made:
        print(f"{os.path.basename(p)}: {sz / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
