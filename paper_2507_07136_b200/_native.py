"""ctypes binding of libsplatfield_b200.so (the C ABI in include/splatfield_b200.h).

This is the only way the package reaches the GPU: there is no CPU or
PyTorch fallback.  If the library is missing or cannot be loaded the import
of any compute function raises ``SplatfieldError`` immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ResourceLimitError, SplatfieldError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsplatfield_b200.so")

SF_OK, SF_ERR_VALIDATION, SF_ERR_RESOURCE, SF_ERR_CUDA, SF_ERR_WORKSPACE = 0, 1, 2, 3, 4
STAT_VISIBLE, STAT_PAIRS, STAT_OVERFLOW, STAT_LEVEL, STAT_ROW, STAT_COL, STAT_DEGENERATE = range(7)
STAT_FIXUPS, STAT_LEVEL_ARGMAX = 7, 8  # STAT_LEVEL_ARGMAX + b: band-owned first argmax of block b
CHAN_WORD = 129 * 4  # scatter-plan channel word = channel x this (sf_common.cuh kChanWord)
STATF_MIN, STATF_MAX, STATF_LEVEL_MAX = 0, 1, 8  # STATF_LEVEL_MAX + n_levels + b: block b min

P = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f64 = ctypes.c_double
sz = ctypes.c_size_t


class SfCamera(ctypes.Structure):
    _fields_ = [("R", f64 * 9), ("t", f64 * 3), ("fx", f64), ("fy", f64), ("cx", f64),
                ("cy", f64), ("near_plane", f64), ("width", i32), ("height", i32)]


class SfScene(ctypes.Structure):
    _fields_ = [("num_gaussians", i64), ("num_levels", i32), ("L", i32), ("K", i32), ("D", i32),
                ("positions", P), ("rotations", P), ("scales", P), ("opacities", P),
                ("coeff_indices", P), ("coeff_values", P), ("ids", P), ("codebooks", P)]


class SfQuery(ctypes.Structure):
    _fields_ = [("vector", P), ("canonicals", P), ("n_canonicals", i32), ("window", i32),
                ("fixed_level", i32), ("threshold", f64)]


class SfFrame(ctypes.Structure):
    _fields_ = [("host_levels", P), ("n_levels", i32), ("early_exit", i32), ("pair_capacity", i64),
                ("coeff_map", P), ("final_t", P), ("features", P), ("relevancy_raw", P),
                ("relevancy_filtered", P), ("mask", P), ("stats_i64", P), ("stats_f64", P),
                ("events", P * 5), ("chan_by_row", P), ("band_y0", i32), ("band_y1", i32),
                ("dec_image", P), ("grad_coeff_map", P), ("grad_values", P), ("reuse_lists", i32)]


EXPORTS = {
    "sf_fixup_capacity": (i64, [i32, i32]),
    "sf_frame_workspace_bytes": (ctypes.c_int, [i64, i32, i32, i32, i32, i32, i32, i64, ctypes.POINTER(sz)]),
    "sf_render_frame": (ctypes.c_int, [ctypes.POINTER(SfScene), ctypes.POINTER(SfCamera),
                                       ctypes.POINTER(SfQuery), ctypes.POINTER(SfFrame), P, sz, P]),
    "sf_render_frame_split": (ctypes.c_int, [ctypes.POINTER(SfScene), ctypes.POINTER(SfCamera),
                                       ctypes.POINTER(SfQuery), ctypes.POINTER(SfFrame), P, sz, P, P, P]),
    "sf_query_sweep": (ctypes.c_int, [ctypes.POINTER(SfScene), ctypes.POINTER(SfCamera), ctypes.POINTER(SfFrame),
                                      P, i32, P, i32, i32, f64, P, P, P, P, P, sz, P]),
    "sf_frame_tile_lists": (ctypes.c_int, [i64, i32, i32, i32, i32, i32, i32, i64, P, sz, P, P, i64, P]),
    "sf_project_workspace_bytes": (ctypes.c_int, [i64, ctypes.POINTER(sz)]),
    "sf_project": (ctypes.c_int, [ctypes.POINTER(SfScene), ctypes.POINTER(SfCamera), P, P, P, P, P,
                                  P, P, P, sz, P]),
    "sf_project_rows": (ctypes.c_int, [ctypes.POINTER(SfScene), ctypes.POINTER(SfCamera), P, P, P,
                                       P, P, P, P, P, P, sz, P]),
    "sf_bin_workspace_bytes": (ctypes.c_int, [i64, i32, i32, i64, ctypes.POINTER(sz)]),
    "sf_bin": (ctypes.c_int, [i64, P, P, P, P, i32, i32, i64, P, P, P, P, P, sz, P]),
    "sf_channel_plan_bytes": (sz, [i64, i32, i32]),
    "sf_pack_channels": (ctypes.c_int, [ctypes.POINTER(SfScene), P, i32, P, sz, P]),
    "sf_decode_workspace_bytes": (sz, [i32, i32]),
    "sf_decode": (ctypes.c_int, [i64, i32, i32, P, i64, P, P, P, sz, P]),
    "sf_decode_simt": (ctypes.c_int, [i64, i32, i32, P, i64, P, P, P]),
    "sf_relevancy_f32": (ctypes.c_int, [i64, i32, P, P, P, i32, P, P]),
    "sf_relevancy_f64": (ctypes.c_int, [i64, i32, P, P, P, i32, P, P]),
    "sf_mean_filter": (ctypes.c_int, [i32, i32, P, i32, P, P, sz, P]),
    "sf_select_segment_workspace_bytes": (sz, [i32, i32, i32]),
    "sf_select_segment": (ctypes.c_int, [i32, i32, i32, P, i32, f64, P, P, P, P, sz, P]),
    "sf_mask_rows": (ctypes.c_int, [P, i32, i32, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double, i32,
                                    i32, P, P]),
    "sf_event_create": (P, []),
    "sf_event_destroy": (None, [P]),
    "sf_event_elapsed_ms": (ctypes.c_float, [P, P]),
    "sf_last_error": (ctypes.c_char_p, []),
    "sf_abi_version": (ctypes.c_int, []),
    "sf_decode_fused": (ctypes.c_int, [i32, i32, i32, i32]),
    "sf_relevancy_fused": (ctypes.c_int, [i32, i32, i32, i32]),
    "sf_decode_image_bytes": (sz, [i32, i32, i32, i32]),
    "sf_pack_decode_image": (ctypes.c_int, [ctypes.POINTER(SfScene), P, i32, P, sz, P]),
    "sf_train_plan": (ctypes.c_int, [i64, i32, i32, i32, P, P, P]),
    "sf_train_loss_blocks": (i64, [i64]),
    "sf_train_cb_splits": (i32, []),
    "sf_train_residual": (ctypes.c_int, [i64, i32, i32, i32, P, P, P, P, f64, f64, P, P, P, P, P]),
    "sf_train_cbgrad": (ctypes.c_int, [i64, i32, i32, i32, P, P, P, P, P]),
    "sf_train_logit_blocks": (i64, [i64, i32]),
    "sf_train_adam_blocks": (i64, [i64]),
    "sf_train_logits": (ctypes.c_int, [i64, i32, i32, i32, P, P, P, P, P, f64, f64, f64, f64, i64, P, P]),
    "sf_train_adam": (ctypes.c_int, [i64, P, P, P, P, f64, f64, f64, f64, i64, P, P]),
    "sf_train_reduce": (ctypes.c_int, [i64, i32, i32, P, P, P]),
    "sf_lsv2_unpack": (ctypes.c_int, [P, i64, i32, i32, i32, P, P, P, P, P, P, P, P, P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load (once) and return the native library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise SplatfieldError(
                f"native library {LIB_PATH} is missing: run "
                "`python -m paper_2507_07136_b200.build_native` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map an SF_ERR_* status to the reference's exception types."""
    if rc == SF_OK:
        return
    msg = load().sf_last_error().decode(errors="replace")
    if rc == SF_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == SF_ERR_RESOURCE:
        raise ResourceLimitError(msg)
    raise SplatfieldError(f"native error {rc}: {msg}")


def check_fixups(stats, width: int, height: int) -> None:
    """Raise when a frame listed more ambiguous early-exit pixels than the
    exact-replay list holds (only possible with SF_FIXUP_CAPACITY lowered):
    the pixels past the capacity kept an uncertified fp32 decision."""
    n = int(stats[STAT_FIXUPS])
    cap = int(load().sf_fixup_capacity(int(width), int(height)))
    if n > cap:
        raise SplatfieldError(f"exact-replay capacity exceeded: {n} ambiguous pixels > capacity {cap}")


def ptr(t) -> ctypes.c_void_p:
    """Device (or host) pointer of a torch tensor / None."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())
