"""Compositing contract shared by the splat path (splatfield/rasterizer.py:45-203).

The blend itself is the sm_100a kernel behind ``sparse_splat``; this module
keeps the reference's constants, ``RenderStats`` and the up-front render
budget check.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ResourceLimitError

EARLY_EXIT_T = 1e-4                      # rasterizer.py:45
DEFAULT_MAX_RENDER_ELEMENTS = 1 << 27    # rasterizer.py:46

TAG_COLOR = "color"
TAG_FEATURE = "dense-feature"
TAG_COEFFICIENT = "coefficient"


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
