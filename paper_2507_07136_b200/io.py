"""Scene / framebuffer / query-set files (splatfield/io.py:1-246), and the
B200 scene loader.

``save_scene`` / ``load_scene`` / ``dump_framebuffer`` / ``load_framebuffer`` /
``save_query_set`` / ``load_query_set`` read and write the reference's formats
byte for byte (little-endian, magic + version; io.py:7-11, 34-246).

``load_scene_device`` is the serving loader: the LSV2
file is read once into pinned host memory, copied raw to HBM, and
``sf_lsv2_unpack`` (sf_io.cu) de-interleaves the packed records into the SoA
arrays the frame kernels read, with Scene.validate's checks (core.py:285-331)
as device flags -- no per-Gaussian numpy on the way.  It returns a resident
``DeviceScene`` that every API function accepts in place of a ``Scene``.
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .core import Codebook, Scene, SceneConfig
from .errors import FormatError, TruncatedFileError, ValidationError
from .query import QueryEmbedding

SCENE_MAGIC = b"LSV2"
SCENE_VERSION = 1
FRAME_MAGIC = b"FBUF"
FRAME_VERSION = 1
_TAG_CODES = {"color": 0, "dense-feature": 1, "coefficient": 2}
_TAG_NAMES = {v: k for k, v in _TAG_CODES.items()}
_HEADER = 28  # magic + 6 x u32


def _record_dtype(num_levels: int, k: int) -> np.dtype:
    """Packed scene record (io.py:42-53)."""
    fields = [("position", "<f4", (3,)), ("rotation", "<f4", (4,)), ("scale", "<f4", (3,)),
              ("opacity", "<f4"), ("color", "<f4", (3,))]
    for lv in range(num_levels):
        fields.append((f"idx{lv}", "<u2", (k,)))
        fields.append((f"val{lv}", "<f4", (k,)))
    return np.dtype(fields)


def save_scene(path, scene: Scene) -> None:
    """io.py:56-74."""
    scene.validate()
    cfg = scene.config
    g = scene.num_gaussians
    rec = np.zeros(g, dtype=_record_dtype(cfg.num_levels, cfg.K))
    rec["position"] = scene.positions
    rec["rotation"] = scene.rotations
    rec["scale"] = scene.scales
    rec["opacity"] = scene.opacities
    rec["color"] = scene.colors
    for lv in range(cfg.num_levels):
        rec[f"idx{lv}"] = scene.coeff_indices[lv]
        rec[f"val{lv}"] = scene.coeff_values[lv]
    with open(path, "wb") as f:
        f.write(SCENE_MAGIC)
        f.write(struct.pack("<IIIIII", SCENE_VERSION, g, cfg.num_levels, cfg.L, cfg.K, cfg.D))
        f.write(rec.tobytes())
        for cb in scene.codebooks:
            f.write(cb.atoms.astype("<f4").tobytes())


def _read_header(f):
    magic = f.read(4)
    if magic != SCENE_MAGIC:
        raise FormatError(f"bad magic {magic!r}; expected {SCENE_MAGIC!r}")
    header = f.read(24)
    if len(header) != 24:
        raise TruncatedFileError("file truncated in header", 4 + len(header))
    version, g, num_levels, L, K, D = struct.unpack("<IIIIII", header)
    if version != SCENE_VERSION:
        raise FormatError(f"unsupported scene version {version}")
    return g, num_levels, L, K, D


def load_scene(path) -> Scene:
    """io.py:77-124 (host arrays; the same errors at the same byte offsets)."""
    with open(path, "rb") as f:
        g, num_levels, L, K, D = _read_header(f)
        dtype = _record_dtype(num_levels, K)
        body = f.read(g * dtype.itemsize)
        if len(body) != g * dtype.itemsize:
            raise TruncatedFileError(
                f"file truncated mid-record ({len(body) % dtype.itemsize} trailing bytes)", _HEADER + len(body))
        rec = np.frombuffer(body, dtype=dtype)
        codebooks = []
        for lv in range(num_levels):
            block = f.read(L * D * 4)
            if len(block) != L * D * 4:
                raise TruncatedFileError(f"file truncated in codebook block {lv}",
                                         _HEADER + len(body) + lv * L * D * 4 + len(block))
            codebooks.append(Codebook(np.frombuffer(block, dtype="<f4").reshape(L, D).copy(), level=lv))
    cfg = SceneConfig(num_levels=num_levels, L=L, K=K, D=D)
    scene = Scene(
        positions=rec["position"].copy(), rotations=rec["rotation"].copy(), scales=rec["scale"].copy(),
        opacities=rec["opacity"].copy(), colors=rec["color"].copy(),
        coeff_indices=np.stack([rec[f"idx{lv}"] for lv in range(num_levels)]) if g
        else np.zeros((num_levels, 0, K), dtype=np.uint16),
        coeff_values=np.stack([rec[f"val{lv}"] for lv in range(num_levels)]) if g
        else np.zeros((num_levels, 0, K), dtype=np.float32),
        codebooks=tuple(codebooks), config=cfg)
    scene.validate()
    return scene


_FLAG_MESSAGES = [  # SF_LSV2_* bits, in Scene.validate's order (core.py:306-331)
    (1, "non-finite entries"),
    (2, "all quaternions must be unit norm"),
    (4, "all scales must be > 0"),
    (8, "opacities must be in [0, 1]"),
    (16, "coefficient index >= L"),
    (32, "coefficient indices must be strictly increasing"),
    (64, "coefficient values must be >= 0"),
    (128, "coefficient values must sum to 1 per level"),
]


def load_scene_device(path):
    """LSV2 file -> resident DeviceScene: one read into pinned host memory, one
    raw H2D copy, ``sf_lsv2_unpack`` on the device."""
    import ctypes

    import torch

    from . import _native as N
    from .device import DeviceScene, require_cuda, stream_ptr
    dev = require_cuda()
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        g, num_levels, L, K, D = _read_header(f)
        rs = _record_dtype(num_levels, K).itemsize
        body = g * rs
        tail = num_levels * L * D * 4
        if size < _HEADER + body:
            raise TruncatedFileError(f"file truncated mid-record ({(size - _HEADER) % rs} trailing bytes)", size)
        if size < _HEADER + body + tail:
            lv = (size - _HEADER - body) // (L * D * 4)
            raise TruncatedFileError(f"file truncated in codebook block {lv}", size)
        host = torch.empty(body + tail, dtype=torch.uint8, pin_memory=True)
        n = f.readinto(memoryview(host.numpy()))
        if n != body + tail:
            raise TruncatedFileError("file truncated", _HEADER + n)
    raw = host.to(dev, non_blocking=True)
    f32, i16 = torch.float32, torch.int16
    t = dict(positions=torch.empty((g, 3), dtype=f32, device=dev),
             rotations=torch.empty((g, 4), dtype=f32, device=dev),
             scales=torch.empty((g, 3), dtype=f32, device=dev),
             opacities=torch.empty((g,), dtype=f32, device=dev),
             colors=torch.empty((g, 3), dtype=f32, device=dev),
             coeff_indices=torch.empty((num_levels, g, K), dtype=i16, device=dev),
             coeff_values=torch.empty((num_levels, g, K), dtype=f32, device=dev))
    t["codebooks"] = raw[body:].view(f32).reshape(num_levels, L, D).clone() if tail else \
        torch.zeros((0, L, D), dtype=f32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(N.load().sf_lsv2_unpack(N.ptr(raw), g, num_levels, K, L, N.ptr(t["positions"]),
                                    N.ptr(t["rotations"]), N.ptr(t["scales"]), N.ptr(t["opacities"]),
                                    N.ptr(t["colors"]), N.ptr(t["coeff_indices"]), N.ptr(t["coeff_values"]),
                                    N.ptr(flags), stream_ptr()))
    bad = int(flags.item())
    for bit, msg in _FLAG_MESSAGES:
        if bad & bit:
            raise ValidationError(msg)
    host_cb = tuple(Codebook(t["codebooks"][lv].cpu().numpy(), level=lv) for lv in range(num_levels))
    del raw, host
    return DeviceScene.from_device(SceneConfig(num_levels=num_levels, L=L, K=K, D=D), t, host_cb, dev)


def dump_framebuffer(path, fb) -> None:
    """Framebuffer as float32; header stores dims, channels, tag (io.py:127-137)."""
    with open(path, "wb") as f:
        f.write(FRAME_MAGIC)
        f.write(struct.pack("<IIIIB", FRAME_VERSION, fb.height, fb.width, fb.channels, _TAG_CODES[fb.tag]))
        f.write(np.ascontiguousarray(fb.data, dtype="<f4").tobytes())


def load_framebuffer(path, *, expect_tag: str | None = None, expect_shape=None):
    """io.py:140-166."""
    from .rasterizer import Framebuffer
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != FRAME_MAGIC:
            raise FormatError(f"bad magic {magic!r}; expected {FRAME_MAGIC!r}")
        header = f.read(17)
        if len(header) != 17:
            raise TruncatedFileError("file truncated in header", 4 + len(header))
        version, h, w, c, tag_code = struct.unpack("<IIIIB", header)
        if version != FRAME_VERSION:
            raise FormatError(f"unsupported framebuffer version {version}")
        if tag_code not in _TAG_NAMES:
            raise FormatError(f"unknown framebuffer tag code {tag_code}")
        tag = _TAG_NAMES[tag_code]
        if expect_tag is not None and tag != expect_tag:
            raise FormatError(f"framebuffer tag is {tag!r}, expected {expect_tag!r}")
        if expect_shape is not None and (h, w, c) != tuple(expect_shape):
            raise FormatError(f"framebuffer dims {(h, w, c)} do not match expected {tuple(expect_shape)}")
        body = f.read(h * w * c * 4)
        if len(body) != h * w * c * 4:
            raise TruncatedFileError("file truncated in pixel data", 21 + len(body))
    return Framebuffer(data=np.frombuffer(body, dtype="<f4").reshape(h, w, c).copy(), tag=tag)


@dataclass
class QuerySet:
    """Named query embeddings plus the shared canonical set (io.py:169-195)."""

    dim: int
    canonicals: np.ndarray  # (n, D) float32
    queries: list
    gt_mask_paths: dict = field(default_factory=dict)

    def __post_init__(self):
        self.canonicals = np.asarray(self.canonicals, dtype=np.float32)
        if self.canonicals.ndim != 2 or self.canonicals.shape[1] != self.dim:
            raise ValidationError("canonicals must be (n, D)")
        for q in self.queries:
            if q.vector.shape[0] != self.dim:
                raise ValidationError(f"query {q.name!r} has dimension {q.vector.shape[0]} != {self.dim}")

    def names(self) -> list:
        return [q.name for q in self.queries]

    def get(self, name: str):
        for q in self.queries:
            if q.name == name:
                return q
        raise ValidationError(f"unknown query {name!r}; available: {', '.join(self.names())}")


def _float_list(arr) -> list:
    return [float(v) for v in np.asarray(arr, dtype=np.float32)]


def save_query_set(path, qs: QuerySet) -> None:
    """io.py:202-219 (JSON, float32 values)."""
    doc = {"D": qs.dim, "canonicals": [_float_list(c) for c in qs.canonicals],
           "queries": [{"name": q.name, "vector": _float_list(q.vector),
                        **({"gt_mask_path": qs.gt_mask_paths[q.name]} if q.name in qs.gt_mask_paths else {})}
                       for q in qs.queries]}
    Path(path).write_text(json.dumps(doc, indent=1) + "\n")


def load_query_set(path) -> QuerySet:
    """io.py:222-243."""
    try:
        doc = json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise FormatError(f"query set is not valid JSON: {exc}") from exc
    try:
        dim = int(doc["D"])
        canonicals = np.array(doc["canonicals"], dtype=np.float32).reshape(-1, dim)
        queries, masks = [], {}
        for q in doc["queries"]:
            queries.append(QueryEmbedding(name=q["name"], vector=np.array(q["vector"], dtype=np.float32)))
            if "gt_mask_path" in q:
                masks[q["name"]] = q["gt_mask_path"]
    except (KeyError, TypeError, ValueError) as exc:
        raise FormatError(f"malformed query set: {exc}") from exc
    return QuerySet(dim=dim, canonicals=canonicals, queries=queries, gt_mask_paths=masks)
