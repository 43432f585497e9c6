"""File formats (splatfield/io.py) against files the reference itself wrote
(tests/golden/io_*, made by oracle/gen_golden.py), and the device loader."""

import os
import struct

import numpy as np
import pytest

import paper_2507_07136_b200 as sf
from paper_2507_07136_b200 import io
from conftest import GOLDEN, make_camera

SCENES = ["io_scene_k4.lsv2", "io_scene_k3.lsv2"]


@pytest.mark.parametrize("name", SCENES)
def test_scene_round_trip_is_byte_exact(name, tmp_path):
    path = os.path.join(GOLDEN, name)
    scene = io.load_scene(path)
    out = tmp_path / name
    io.save_scene(out, scene)
    assert out.read_bytes() == open(path, "rb").read()


def test_scene_errors(tmp_path):
    raw = open(os.path.join(GOLDEN, SCENES[0]), "rb").read()
    (tmp_path / "magic").write_bytes(b"LSV3" + raw[4:])
    with pytest.raises(sf.FormatError):
        io.load_scene(tmp_path / "magic")
    (tmp_path / "version").write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(sf.FormatError):
        io.load_scene(tmp_path / "version")
    (tmp_path / "trunc").write_bytes(raw[:28 + 100])
    with pytest.raises(sf.TruncatedFileError) as e:
        io.load_scene(tmp_path / "trunc")
    assert e.value.offset == 128
    (tmp_path / "tail").write_bytes(raw[:-10])
    with pytest.raises(sf.TruncatedFileError):
        io.load_scene(tmp_path / "tail")


def test_framebuffer_and_query_set_round_trip(tmp_path):
    fb = io.load_framebuffer(os.path.join(GOLDEN, "io_frame.fbuf"), expect_tag="color", expect_shape=(7, 5, 3))
    io.dump_framebuffer(tmp_path / "f.fbuf", fb)
    assert (tmp_path / "f.fbuf").read_bytes() == open(os.path.join(GOLDEN, "io_frame.fbuf"), "rb").read()
    with pytest.raises(sf.FormatError):
        io.load_framebuffer(os.path.join(GOLDEN, "io_frame.fbuf"), expect_tag="coefficient")
    qs = io.load_query_set(os.path.join(GOLDEN, "io_queries.json"))
    assert qs.names() == ["chair", "lamp"] and qs.gt_mask_paths == {"lamp": "masks/lamp.fbuf"}
    io.save_query_set(tmp_path / "q.json", qs)
    assert (tmp_path / "q.json").read_text() == open(os.path.join(GOLDEN, "io_queries.json")).read()
    with pytest.raises(sf.ValidationError):
        qs.get("sofa")
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(sf.FormatError):
        io.load_query_set(tmp_path / "bad.json")


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_device_loader_equals_host_scene(name):
    """load_scene_device (pinned read -> raw H2D -> sf_lsv2_unpack) gives the
    same resident arrays, and the same frames, as uploading load_scene's."""
    import torch
    from paper_2507_07136_b200.device import DeviceScene
    path = os.path.join(GOLDEN, name)
    host = io.load_scene(path)
    ds = io.load_scene_device(path)
    ref = DeviceScene(host)
    for k in ("positions", "rotations", "scales", "opacities", "colors", "coeff_indices", "coeff_values",
              "codebooks"):
        assert torch.equal(getattr(ds, k), getattr(ref, k)), k
    cam = make_camera(40, 32)
    a = sf.splat_multilevel(ds, cam).data
    b = sf.splat_multilevel(host, cam).data
    assert a.tobytes() == b.tobytes()
    cfg = host.config
    q = sf.QueryEmbedding("q", np.random.default_rng(1).standard_normal(cfg.D))
    canon = np.random.default_rng(2).standard_normal((4, cfg.D))
    r1 = sf.query_pipeline(ds, cam, q, canon)
    r2 = sf.query_pipeline(host, cam, q, canon)
    assert r1.level == r2.level and r1.point == r2.point
    np.testing.assert_array_equal(r1.mask, r2.mask)
    assert np.abs(r1.feature_maps.maps[0] - r2.feature_maps.maps[0]).max() == 0
    assert sf.render_dense(ds, cam).data.tobytes() == sf.render_dense(host, cam).data.tobytes()


@pytest.mark.gpu
def test_device_loader_validation_flags(tmp_path):
    """Corrupt records raise Scene.validate's errors (core.py:285-331) from the device flags."""
    path = os.path.join(GOLDEN, SCENES[0])
    raw = bytearray(open(path, "rb").read())
    rs = 56 + 3 * 6 * 4
    cases = {
        12: (np.float32(2.0), "unit norm"),             # quaternion w of record 0
        28: (np.float32(-1.0), "scales"),               # scale x
        40: (np.float32(1.5), "opacities"),             # opacity
        56 + 8 + 0: (np.float32(0.9), "sum to 1"),      # first value of level 0
    }
    for off, (val, msg) in cases.items():
        bad = bytearray(raw)
        bad[28 + rs + off:28 + rs + off + 4] = val.tobytes()  # record 1
        p = tmp_path / f"bad{off}.lsv2"
        p.write_bytes(bytes(bad))
        with pytest.raises(sf.ValidationError, match=msg):
            io.load_scene_device(p)
    bad = bytearray(raw)
    bad[28 + 56:28 + 58] = np.uint16(99).tobytes()  # index >= L
    (tmp_path / "idx.lsv2").write_bytes(bytes(bad))
    with pytest.raises(sf.ValidationError, match="index >= L"):
        io.load_scene_device(tmp_path / "idx.lsv2")
    with pytest.raises(sf.TruncatedFileError):
        (tmp_path / "t.lsv2").write_bytes(bytes(raw[:-4]))
        io.load_scene_device(tmp_path / "t.lsv2")
