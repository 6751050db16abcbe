"""ctypes binding of the C ABI in include/gslic.h (libgslic.so, sm_100a).

The product path has no CPU fallback: if the in-tree library is missing (or there is no CUDA
device) every entry point raises.  Structures mirror the header field by field.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DataError, DomainError, NumericalError

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSLIC_LIB: a developer override for A/B builds (tools/gpu_ab.sh); default the in-tree build
LIB_PATH = os.environ.get("GSLIC_LIB") or os.path.join(_HERE, "lib", "libgslic.so")

GS_ROW = 64
GS_NPARAM = 59
GS_TILE = 16
GS_G2D = 20  # int64 words per screen-space gradient row (10 fixed-point (hi, lo) fields)
GS_G2D_FIELDS = 10
GS_LOSS_RING = 64  # per-iteration loss ring of an engine workspace (gs_frame.loss[8:])
GS_SPLAT = 16  # floats per 2D splat record
CNT_ACTIVE, CNT_ENTRIES, CNT_TOUCHED, CNT_OVERFLOW, CNT_ENTRIES_EFF = 0, 1, 2, 3, 4
GS_CNT_SLOTS = 16
GS_BIN_LAZY = 2  # gs_bin cull mode of the iteration engine (tile lists materialised on demand)
GS_PP_LAZY_SH = 1  # gs_preprocess_ex flag of the iteration engine (colours only where blended)
GS_LOSS_TABLES_READY, GS_LOSS_ACCUMULATE, GS_LOSS_DEPTH_GRADS_ZERO = 1, 2, 4  # gs_loss_ex flags
GS_BWD_ROWS_ZERO, GS_BWD_CLEAR_DEPTH_GRADS = 1, 2  # gs_render_bwd_ex flags
GS_FWD_EARLY_STOP, GS_FWD_CLEAR_G2D = 1, 2  # gs_render_fwd_ex flags

# Set by dropin.install: the reference-shaped entry points then return numpy arrays for every
# map (the reference's callers do numpy arithmetic on them, R/cli.py:153-159, R/apps.py:208-223),
# not only for reference-typed (numpy) maps
HOST_ARRAYS = False

P = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f32 = ctypes.c_float


class GsCamera(ctypes.Structure):
    _fields_ = [("width", i32), ("height", i32), ("fx", f32), ("fy", f32), ("cx", f32), ("cy", f32),
                ("rot_cw", f32 * 9), ("trans_cw", f32 * 3), ("center", f32 * 3)]


class GsView(ctypes.Structure):
    _fields_ = [("cam", GsCamera), ("target", P), ("lidar_idx", P), ("lidar_z", P), ("lidar_k", i32),
                ("pad_", i32)]


class GsFrame(ctypes.Structure):
    _fields_ = [("n", i64), ("entry_capacity", i64), ("width", i32), ("height", i32), ("tiles_x", i32),
                ("tiles_y", i32),
                ("splat2d", P), ("cov2d", P), ("rect", P), ("valid", P), ("touched", P), ("touched_list", P),
                ("g2d", P), ("grad_rows", P), ("bias_corr", P), ("keep_bits", P), ("kept", P), ("big_list", P),
                ("big_slot", P), ("cull_queue", P), ("cull_queue_cap", i64),
                ("huge", P), ("huge_mask", P), ("huge_mask_t", P),
                ("tile_scratch", P), ("tile_minkey", P), ("big_bits", P), ("big_bits_words", i64),
                ("keys_a", P), ("keys_b", P),
                ("entry_splat", P), ("tile_offsets", P), ("counters", P),
                ("color", P), ("depth", P), ("opacity", P), ("trans", P), ("n_contrib", P),
                ("g_color", P), ("g_depth", P), ("g_opac", P), ("loss_parts", P), ("loss", P),
                ("loss_blocks", i64), ("pose_acc", P), ("ssim_g", P)]


_lib = None


def lib():
    """Load libgslic.so; raise loudly if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2507_04004_b200.build` "
                           "(the sm_100a kernels are the only implementation; there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    sigs = {
        "gs_workspace_size": (ctypes.c_size_t, [i64, i32, i32, i64]),
        "gs_frame_layout": (ctypes.c_int, [i64, i32, i32, i64, P, ctypes.c_size_t, ctypes.POINTER(GsFrame)]),
        "gs_camera_init": (None, [ctypes.POINTER(GsCamera)]),
        "gs_last_error": (ctypes.c_char_p, []),
        "gs_version": (ctypes.c_int, []),
        "gs_preprocess": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P]),
        "gs_preprocess_ex": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, i32, P]),
        "gs_bin": (ctypes.c_int, [ctypes.POINTER(GsFrame), i32, P]),
        "gs_render_fwd": (ctypes.c_int, [ctypes.POINTER(GsFrame), i32, P]),
        "gs_render_fwd_ex": (ctypes.c_int, [ctypes.POINTER(GsFrame), i32, P]),
        "gs_loss": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, f32, f32, P]),
        "gs_loss_ex": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, f32, f32, i32, P]),
        "gs_render_bwd_ex": (ctypes.c_int, [ctypes.POINTER(GsFrame), i32, P]),
        "gs_render_bwd": (ctypes.c_int, [ctypes.POINTER(GsFrame), P]),
        "gs_chain_adam": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P, P, P, P, P]),
        "gs_chain_adam_part": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P, P, P, P, i32, i32, i32, P]),
        "gs_p2p_reduce_adam": (ctypes.c_int, [i32, i32, P, P, P, P, ctypes.c_uint64, i64, P, P, P, P, P, P, P, P, P, P,
                                              P, P]),
        "gs_ipc_export": (ctypes.c_int, [P, P, ctypes.POINTER(i64)]),
        "gs_ipc_import": (ctypes.c_int, [P, i64, ctypes.POINTER(P), ctypes.POINTER(P)]),
        "gs_ipc_close": (ctypes.c_int, [P]),
        "gs_chain": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P, P, P]),
        "gs_chain_pose": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P, P, P, P]),
        "gs_project_points": (ctypes.c_int, [P, i64, P, P, P, f32, P, P, P, P, P, P, P, P]),
        "gs_zbuffer": (ctypes.c_int, [P, i64, P, i32, i32, P, P, P]),
        "gs_init_rows": (ctypes.c_int, [P, P, P, i64, f32, P, P]),
        "gs_decode_u8": (ctypes.c_int, [P, P, i64, P]),
        "gs_track_mask": (ctypes.c_int, [P, i32, i32, f32, P, P]),
        "gs_track_grad": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, f32, P]),
        "gs_pose_adam": (ctypes.c_int, [P, P, P, f32, P]),
        "gs_adam": (ctypes.c_int, [P, P, P, P, P, P, i64, P, P]),
        "gs_lidar_compact": (ctypes.c_int, [P, i32, i32, P, P, P, P]),
        "gs_project": (ctypes.c_int, [P, i64, P, P, P, P, P, P, P, P, P, P, P]),
        "gs_eval_sh": (ctypes.c_int, [P, P, P, i64, P, P, P]),
        "gs_pack_splats": (ctypes.c_int, [ctypes.POINTER(GsFrame), P, P, P, P, P, P, P, P]),
        "gs_compact_flags": (ctypes.c_int, [P, i64, P, P, P, P]),
        "gs_gather_rows": (ctypes.c_int, [P, P, P, i64, P, P]),
        "gs_adam_packed": (ctypes.c_int, [P, P, P, P, P, P, P, i64, i64, P, P, P, P]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = ["gs_workspace_size", "gs_frame_layout", "gs_camera_init", "gs_last_error", "gs_version",
            "gs_preprocess", "gs_preprocess_ex", "gs_bin", "gs_render_fwd", "gs_render_fwd_ex", "gs_loss", "gs_loss_ex", "gs_render_bwd", "gs_render_bwd_ex", "gs_chain_adam",
            "gs_chain_adam_part", "gs_chain", "gs_chain_pose", "gs_adam", "gs_lidar_compact", "gs_project", "gs_eval_sh", "gs_pack_splats",
            "gs_project_points", "gs_zbuffer", "gs_init_rows", "gs_decode_u8", "gs_track_mask", "gs_track_grad", "gs_pose_adam",
            "gs_compact_flags", "gs_gather_rows", "gs_adam_packed", "gs_p2p_reduce_adam", "gs_ipc_export",
            "gs_ipc_import", "gs_ipc_close"]


def check(rc: int, what: str) -> None:
    """Map C-ABI status codes onto the reference's error taxonomy (R/errors.py)."""
    if rc == 0:
        return
    msg = f"{what}: {lib().gs_last_error().decode(errors='replace')}"
    if rc in (1, 2):
        raise DomainError(msg)
    if rc in (3, 4):
        raise DataError(msg)
    raise NumericalError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
