"""Config E's tile-band sharding through a real process group: two processes
(gloo, both on cuda:0) run distributed.band_query / band_query_sweep and must
equal the single-process frame bit for bit (the reference's
only parallel axis, its tile thread pool sparse_splat.py:152-159, is what the
band split generalises)."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

_HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    sys.path.insert(0, _HERE)
    from conftest import make_camera, random_scene
    rng = np.random.default_rng(11)
    scene = random_scene(rng, 4000, num_levels=3, L=64, K=4, D=64)
    cam = make_camera(96, 80)
    canon = rng.standard_normal((4, 64))
    prompts = rng.standard_normal((5, 64))
    return scene, cam, canon, prompts


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2507_07136_b200.device import QuerySpec, device_scene
    from paper_2507_07136_b200.distributed import band_query, band_query_sweep
    scene, cam, canon, prompts = _inputs()
    eng = device_scene(scene).engine
    levels = (0, 1, 2)
    bq = band_query(eng, cam, levels, QuerySpec(prompts[0], canon, 11, -1, 0.5), world, rank)
    torch.cuda.synchronize()
    y0, y1 = bq.band.y0, bq.band.y1
    bs = band_query_sweep(eng, cam, levels, prompts, canon, world, rank)
    sel = np.array([[s[0], s[1][0], s[1][1]] for s in bs.selections], dtype=np.int64)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), y0=y0, y1=y1, level=bq.level, point=np.array(bq.point),
             lo=bq.lo, hi=bq.hi, mask=bq.out.mask[y0:y1].cpu().numpy(),
             sweep_sel=sel, sweep_masks=bs.masks[:, y0:y1].cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_band_query_and_sweep_over_a_gloo_group_equal_the_full_frame(tmp_path):
    import torch.multiprocessing as mp

    import paper_2507_07136_b200 as sf
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    scene, cam, canon, prompts = _inputs()
    full = sf.query_pipeline(scene, cam, sf.QueryEmbedding("q0", prompts[0]), canon)
    sweep = sf.query_sweep(scene, cam, [sf.QueryEmbedding(f"q{i}", p) for i, p in enumerate(prompts)], canon)
    rows = 0
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        y0, y1 = int(z["y0"]), int(z["y1"])
        rows += y1 - y0
        # every rank holds the global selection (max-all-reduce of exact keys)
        assert int(z["level"]) == full.level and tuple(z["point"]) == tuple(full.point)
        assert np.array_equal(z["mask"].astype(bool), full.mask[y0:y1])
        for i, res in enumerate(sweep):
            assert tuple(z["sweep_sel"][i]) == (res.level, res.point[0], res.point[1])
            assert np.array_equal(z["sweep_masks"][i].astype(bool), res.mask[y0:y1])
    assert rows == cam.height  # the bands cover the image once
