"""Compositing contract shared by the splat path (splatfield/rasterizer.py:45-272).

The blend itself is the sm_100a kernel behind ``sparse_splat``; this module
keeps the reference's constants, ``RenderStats``, ``Framebuffer``, the
up-front render budget check, and ``render_dense`` -- the dense comparator
(rasterizer.py:206-272), run by the same blend kernel with a dense scatter
plan (channel c of every Gaussian -> accumulator row c), 16 channels per pass.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ResourceLimitError, ValidationError

EARLY_EXIT_T = 1e-4                      # rasterizer.py:45
DEFAULT_MAX_RENDER_ELEMENTS = 1 << 27    # rasterizer.py:46

TAG_COLOR = "color"
TAG_FEATURE = "dense-feature"
TAG_COEFFICIENT = "coefficient"
_TAGS = (TAG_COLOR, TAG_FEATURE, TAG_COEFFICIENT)
DEFAULT_TILE_SIZE = 16
DENSE_CHANNELS_PER_PASS = 16  # channels a Gaussian's scatter plan can hold (kMaxC)


@dataclass
class RenderStats:
    """Instrumentation attached to a render when requested (rasterizer.py:100-107)."""

    final_transmittance: np.ndarray  # (H, W)
    pairs_blended: int               # Gaussian-tile entries processed
    channels_per_gaussian: int       # channel slots each blended Gaussian touches
    workers: int


def check_render_budget(width: int, height: int, channels: int, max_elements: int) -> None:
    """ResourceLimitError before any work (rasterizer.py:197-203)."""
    total = width * height * channels
    if total > max_elements:
        raise ResourceLimitError(
            f"render of {height}x{width}x{channels} = {total} elements exceeds "
            f"the budget of {max_elements}")


@dataclass
class Framebuffer:
    """H x W x C scalar grid with a channel-semantics tag (rasterizer.py:55-86)."""

    data: np.ndarray
    tag: str

    def __post_init__(self):
        self.data = np.asarray(self.data)
        if self.data.ndim != 3:
            raise ValidationError(f"framebuffer data must be H x W x C, got {self.data.shape}")
        if self.tag not in _TAGS:
            raise ValidationError(f"unknown framebuffer tag {self.tag!r}")

    @property
    def height(self) -> int:
        return int(self.data.shape[0])

    @property
    def width(self) -> int:
        return int(self.data.shape[1])

    @property
    def channels(self) -> int:
        return int(self.data.shape[2])

    def validate(self) -> None:
        if not np.all(np.isfinite(self.data)):
            raise ValidationError("framebuffer entries must be finite")
        if self.tag == TAG_COEFFICIENT:
            if np.any(self.data < 0) or np.any(self.data > 1):
                raise ValidationError("coefficient channels must lie in [0, 1]")


def _resolve_channels(scene, channels):
    """'color' or a (num_gaussians, C) array (rasterizer.py:184-195)."""
    if isinstance(channels, str):
        if channels != "color":
            raise ValidationError(f"unknown channel source {channels!r}")
        return np.asarray(scene.colors, dtype=np.float64), TAG_COLOR
    values = np.asarray(channels, dtype=np.float64)
    if values.ndim != 2 or values.shape[0] != scene.num_gaussians:
        raise ValidationError(f"channel array must be (num_gaussians, C), got {values.shape}")
    return values, TAG_FEATURE


def render_dense(scene, cam, channels="color", *, tag: str | None = None,
                 tile_size: int = DEFAULT_TILE_SIZE, early_exit: bool = True, background=None,
                 max_elements: int = DEFAULT_MAX_RENDER_ELEMENTS, workers: int = 1,
                 with_stats: bool = False, engine=None):
    """Dense render of per-Gaussian channel vectors (rasterizer.py:206-272) on the GPU.

    The sm_100a blend kernel runs with a dense scatter plan -- Gaussian g adds
    e * values[g, c] to accumulator channel c -- in passes of 16 channels
    (values are blended in fp32, like the coefficient path).  ``workers`` is
    accepted and echoed; tiles are independent CTAs.  Errors are raised before
    any work, as in the reference."""
    import torch

    from .device import device_scene
    from .device import DeviceScene
    device_rows = isinstance(scene, DeviceScene) and isinstance(channels, str) and channels == "color"
    if device_rows:  # a resident scene's colours, already in device row order
        values, inferred = scene.colors.double().cpu().numpy(), TAG_COLOR
    else:
        values, inferred = _resolve_channels(scene, channels)
    tag = tag or inferred
    c = values.shape[1]
    W, H = int(cam.width), int(cam.height)
    check_render_budget(W, H, c, max_elements)
    bg = None
    if background is not None:
        bg = np.asarray(background, dtype=np.float64)
        if bg.shape != (c,):
            raise ValidationError(f"background must have {c} channels")
    if tile_size != DEFAULT_TILE_SIZE:
        raise ValidationError("the sm_100a kernels are specialised for 16x16 tiles")
    ds = device_scene(scene)
    eng = ds.engine if engine is None else engine
    dev = ds.device
    g = ds.num_gaussians
    vals = values if (ds.orig_rows is None or device_rows) else values[ds.orig_rows.cpu().numpy()]
    vals = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float32)).to(dev)
    out = torch.zeros((H, W, c), dtype=torch.float32, device=dev)
    # every pass blends 16 plan channels (unused ones carry zero values), so the
    # workspace layout is the same for all passes: the first pass projects and
    # bins, the others reuse its tile lists (SfFrame.reuse_lists).  C = 0 still
    # runs one pass: final T and the pair count come from a real frame.
    cc = DENSE_CHANNELS_PER_PASS
    half = (4 * cc + 15) // 16 * 4  # words per record half (chan_val_offset / 4)
    fo = eng.allocate(W, H, (0,), coeff_map=False, final_t=True, mask=False)
    fo.coeff_map = torch.empty((H, W, cc), dtype=torch.float32, device=dev)
    with eng._lock:
        for i, c0 in enumerate(range(0, max(c, 1), cc)):
            n = min(cc, c - c0)
            plan = torch.zeros((max(g, 1), 2 * half), dtype=torch.int32, device=dev)
            plan[:, :cc] = torch.arange(cc, dtype=torch.int32, device=dev) * 516  # accumulator byte offsets
            if g and n > 0:
                plan[:g, half:half + n] = vals[:, c0:c0 + n].contiguous().view(torch.int32)
            eng.run(cam, (0,), fo, early_exit=early_exit, dense=(plan, cc), reuse_lists=i > 0)
            if n > 0:
                out[:, :, c0:c0 + n] = fo.coeff_map[:, :, :n]
    final_t = fo.final_t
    pairs = int(fo.host_stats()[0][1])
    data = out.double()
    if bg is not None:
        data = data + final_t.double()[:, :, None] * torch.from_numpy(bg).to(dev)[None, None, :]
    fb = Framebuffer(data=data.cpu().numpy(), tag=tag)
    if not with_stats:
        return fb
    return fb, RenderStats(final_transmittance=final_t.double().cpu().numpy(), pairs_blended=pairs,
                           channels_per_gaussian=c, workers=workers)
