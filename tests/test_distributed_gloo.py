"""Multi-process host logic of the sharded path on CPU (gloo, world size 2)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_07136_b200.distributed import band_rows, shard_views


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_views_cover_and_balance():
    for n, w in [(64, 8), (10, 3), (1, 4)]:
        shards = [shard_views(n, w, r) for r in range(w)]
        assert sorted(sum(shards, [])) == list(range(n))
        assert max(map(len, shards)) - min(map(len, shards)) <= 1


def test_band_rows_partition_with_halo():
    H = 1080
    bands = [band_rows(H, 8, r) for r in range(8)]
    assert bands[0].y0 == 0 and bands[-1].y1 == H
    for a, b in zip(bands, bands[1:]):
        assert a.y1 == b.y0 and a.y0 % 16 == 0
    for b in bands:
        assert b.render_y0 == max(0, b.y0 - 5) and b.render_y1 == min(H, b.y1 + 5)


def _worker(rank, world, port, results):
    import torch
    import torch.distributed as dist

    from paper_2507_07136_b200.distributed import gather_results, global_selection
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    H, W = 24, 10
    maps = rng.random((3, H, W)) * 0.9 + 0.05
    maps[1, 17, 3] = 0.99          # global max of level 1 ...
    maps[1, 20, 8] = 0.99          # ... tied later in row-major order (lower index must win)
    band = band_rows(H, world, rank, tile=8, halo=0)
    sub = maps[:, band.y0:band.y1]
    lmax = sub.reshape(3, -1).max(axis=1)
    larg = sub.reshape(3, -1).argmax(axis=1)
    rows, cols = np.divmod(larg, W)
    flat = (rows + band.y0) * W + cols
    lmin = sub.reshape(3, -1).min(axis=1)
    level, idx, mn, mx = global_selection(lmax, flat, lmin)
    masks = gather_results(torch.from_numpy((sub[level] > 0.5).astype(np.uint8)).contiguous()
                           if band.y1 - band.y0 == H // world else torch.zeros(1, dtype=torch.uint8))
    results[rank] = (level, idx, mn, mx, masks.shape[0])
    dist.destroy_process_group()


def test_band_sharded_selection_matches_single_process():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    rng = np.random.default_rng(0)
    maps = rng.random((3, 24, 10)) * 0.9 + 0.05
    maps[1, 17, 3] = 0.99
    maps[1, 20, 8] = 0.99
    level = int(np.argmax(maps.reshape(3, -1).max(axis=1)))
    idx = int(np.argmax(maps[level]))
    for r in range(world):
        lv, ix, mn, mx, n = results[r]
        assert lv == level == 1
        assert ix == idx == 17 * 10 + 3
        assert mn == pytest.approx(maps[level].min()) and mx == pytest.approx(maps[level].max())
        assert n == world


def test_combine_selection_rules():
    """Host twin of global_selection: lowest level on ties, first row-major argmax."""
    from paper_2507_07136_b200.distributed import combine_selection
    # band 0 / band 1 of a 3-level, 4x5 image (rows 0-1 / 2-3)
    mx = [[0.5, 0.9, 0.9], [0.7, 0.9, 0.2]]
    am = [[3, 7, 1], [12, 11, 15]]
    mn = [[0.1, 0.2, 0.3], [0.05, 0.25, 0.1]]
    level, idx, lo, hi = combine_selection(mx, am, mn)
    assert level == 1 and idx == 7 and lo == 0.2 and hi == 0.9
    mx = [[0.5, 0.4], [0.5, 0.3]]
    am = [[9, 0], [4, 0]]
    level, idx, _, _ = combine_selection(mx, am, [[0.0, 0.0], [0.0, 0.0]])
    assert level == 0 and idx == 4


def _worker_many(rank, world, port, results):
    import torch.distributed as dist

    from paper_2507_07136_b200.distributed import global_selection_many
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    P, H, W = 5, 24, 10
    maps = rng.random((P, 3, H, W)) * 0.9 + 0.05
    maps[2, 1, 3, 4] = 0.995       # prompt 2: the max of level 1 in band 0 ...
    maps[2, 1, 20, 1] = 0.995      # ... tied in band 1 (the lower flat index wins)
    band = band_rows(H, world, rank, tile=8, halo=0)
    sub = maps[:, :, band.y0:band.y1].reshape(P, 3, -1)
    lmax, lmin = sub.max(axis=2), sub.min(axis=2)
    rows, cols = np.divmod(sub.argmax(axis=2), W)
    flat = (rows + band.y0) * W + cols
    results[rank] = global_selection_many(lmax, flat, lmin)
    dist.destroy_process_group()


def test_band_sharded_selection_many_prompts():
    """global_selection_many (one pair of all-reduces for every prompt of a
    band sweep) equals the single-process selection prompt by prompt."""
    from paper_2507_07136_b200.distributed import combine_selection_many
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker_many, args=(world, port, results), nprocs=world, join=True)
    rng = np.random.default_rng(1)
    P, H, W = 5, 24, 10
    maps = rng.random((P, 3, H, W)) * 0.9 + 0.05
    maps[2, 1, 3, 4] = 0.995
    maps[2, 1, 20, 1] = 0.995
    for p in range(P):
        level = int(np.argmax(maps[p].reshape(3, -1).max(axis=1)))
        idx = int(np.argmax(maps[p, level]))
        for r in range(world):
            lv, ix, mn, mx = results[r][p]
            assert (lv, ix) == (level, idx)
            assert mn == maps[p, level].min() and mx == maps[p, level].max()
    assert results[0][2][:2] == (1, 3 * W + 4)
    # the host twin over per-band statistics gives the same answers
    stats = []
    for r in range(world):
        band = band_rows(H, world, r, tile=8, halo=0)
        sub = maps[:, :, band.y0:band.y1].reshape(P, 3, -1)
        rows, cols = np.divmod(sub.argmax(axis=2), W)
        stats.append((sub.max(axis=2), (rows + band.y0) * W + cols, sub.min(axis=2)))
    mx_b, am_b, mn_b = (np.stack(x) for x in zip(*stats))
    assert combine_selection_many(mx_b, am_b, mn_b) == results[0]


def test_band_rows_rejects_more_ranks_than_tile_rows():
    """Every rank raises before any collective (no empty bands, no hang)."""
    from paper_2507_07136_b200.errors import ValidationError
    for r in range(8):
        with pytest.raises(ValidationError):
            band_rows(64, 8, r)
    assert band_rows(64, 4, 3).y1 == 64
