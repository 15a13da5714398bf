"""ctypes binding of libartemis.so (the C ABI declared in include/artemis.h).

This is the only place the Python layer touches native code. The library
is built in-tree by ``build_lib.py``; if it is missing, or no sm_100 device
is visible, every product call raises ``ExtensionMissing`` -- there is no
CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (ContractViolation, DeviceError, DuplicateMortonError, ExtensionMissing)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ARTEMIS_LIB_PATH") or os.path.join(HERE, "libartemis.so")

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
INT = C.c_int
DBL = C.c_double
SZ = C.c_size_t

OK, ERR_ARG, ERR_RANGE, ERR_EMPTY, ERR_DUP, ERR_OOM, ERR_CUDA, ERR_WS, ERR_NODEV = range(9)
(ASSET_TRUNC_HEADER, ASSET_BAD_MAGIC, ASSET_BAD_VERSION, ASSET_ZERO_COUNT, ASSET_TRUNC_LEAVES,
 ASSET_TRUNC_FLUT, ASSET_RIG_OFFSET, ASSET_TRUNC_RIG, ASSET_TRAILING) = range(20, 29)


class BrickMap(C.Structure):
    _fields_ = [("table", P), ("recs", P), ("aabb", P), ("org", I32 * 3), ("dims", I32 * 3)]


class TreeView(C.Structure):
    _fields_ = [("nodes", P), ("leaves", P), ("n_leaves", I64), ("n_leaves_dev", P),
                ("coord_max", DBL), ("bricks", C.POINTER(BrickMap))]


class Shading(C.Structure):
    _fields_ = [("coef", P), ("sigma", P), ("rot_index", P), ("rot_inv", P), ("degree", INT),
                ("channels", INT), ("coef_stride", INT)]


class Rays(C.Structure):
    _fields_ = [("origins_g", P), ("dirs_g", P), ("dirs_w", P), ("n_rays", I64),
                ("t_min", DBL), ("t_max", DBL), ("fast_div", I32)]


class Camera(C.Structure):
    _fields_ = [("R", DBL * 9), ("origin", DBL * 3), ("fx", DBL), ("fy", DBL), ("cx", DBL),
                ("cy", DBL), ("width", I32), ("height", I32), ("lo", DBL * 3),
                ("cell", DBL * 3), ("tile_start", I32), ("tile_stride", I32)]


class Asset(C.Structure):
    _fields_ = [("n_voxels", I64), ("resolution", I32), ("slots", I32), ("max_joints", I32),
                ("degree", I32), ("channels", I32), ("lo", DBL * 3), ("hi", DBL * 3),
                ("cells", P), ("joint_idx", P), ("weights", P), ("coef", P), ("sigma", P)]


class AssetInfo(C.Structure):
    _fields_ = [("version", C.c_uint32), ("resolution", C.c_uint32), ("count", I64),
                ("degree", I32), ("channels", I32), ("width", I32), ("lo", DBL * 3),
                ("hi", DBL * 3), ("rig_offset", I64), ("leaf_offset", I64),
                ("flut_offset", I64), ("flut_end", I64)]


class AssetRig(C.Structure):
    _fields_ = [("n_joints", I32), ("k_max", I32), ("name_bytes", I64), ("end", I64)]


class FrameTree(C.Structure):
    _fields_ = [("codes", P), ("code_bytes", I32), ("flut_idx", P), ("left", P), ("right", P),
                ("box_min", P), ("box_size", P), ("rotation_joint", P), ("n_live_dev", P),
                ("n_in_dev", P)]


_SIGS = {
    "artemis_version": (C.c_char_p, []),
    "artemis_status_string": (C.c_char_p, [INT]),
    "artemis_last_cuda_error": (C.c_char_p, []),
    "artemis_device_ok": (INT, []),
    "artemis_morton_encode": (INT, [P, I64, P, P, P]),
    "artemis_morton_decode": (INT, [P, I64, P, P]),
    "artemis_sort_workspace_bytes": (SZ, [I64, INT, INT]),
    "artemis_sort_pairs_u64": (INT, [P, P, P, P, I64, INT, P, SZ, P]),
    "artemis_sort_pairs_u32": (INT, [P, P, P, P, I64, INT, P, SZ, P]),
    "artemis_build_tree": (INT, [P, I64, P, P, P, P, P, P]),
    "artemis_pack_tree": (INT, [P, P, I64, I32, P, P, P, P, P, P, P, P, P]),
    "artemis_flut_split_f64": (INT, [P, I64, INT, P, P, P]),
    "artemis_flut_split_f32": (INT, [P, I64, INT, P, P, P]),
    "artemis_render_rays": (INT, [C.POINTER(TreeView), C.POINTER(Shading), C.POINTER(Rays), DBL,
                                  DBL, INT, P, P, P, P]),
    "artemis_count_hits": (INT, [C.POINTER(TreeView), C.POINTER(Rays), P, P]),
    "artemis_forward_fit": (INT, [C.POINTER(TreeView), C.POINTER(Shading), C.POINTER(Rays), P, P,
                                  P, P, P, P, P]),
    "artemis_camera_rays": (INT, [C.POINTER(Camera), P, P, P, P]),
    "artemis_warp": (INT, [P, I64, INT, P, P, P, INT, P, P, INT, P, P, P, P, P]),
    "artemis_resolve_workspace_bytes": (SZ, [I64]),
    "artemis_resolve_u64": (INT, [P, P, I64, P, P, P, P, P, P, P, SZ, P]),
    "artemis_frame_create": (INT, [C.POINTER(Asset), C.POINTER(P)]),
    "artemis_frame_destroy": (INT, [P]),
    "artemis_frame_run": (INT, [P, P, P, INT, C.POINTER(Camera), DBL, DBL, INT, P, P, P, P]),
    "artemis_frame_counts": (INT, [P, C.POINTER(I64), C.POINTER(I64), P]),
    "artemis_frame_get_tree": (INT, [P, C.POINTER(FrameTree)]),
    "artemis_frame_launches": (INT, [P]),
    "artemis_frame_set_tile_order": (INT, [P, INT, INT, P]),
    "artemis_frame_set_output_peer": (INT, [P, P, P, P, I64, INT]),
    "artemis_frame_run_views": (INT, [P, P, P, INT, P, INT, DBL, DBL, INT, P, P, P, P]),
    "artemis_copy_to_host": (INT, [P, P, SZ, P]),
    "artemis_frame_profile": (INT, [P, INT]),
    "artemis_brickmap_bytes": (SZ, [I64, P]),
    "artemis_brickmap_build": (INT, [P, I64, P, P, P, SZ, C.POINTER(BrickMap), P]),
    "artemis_frame_stage_ms": (INT, [P, C.POINTER(C.c_float)]),
    "artemis_backward_workspace_bytes": (SZ, [I64, I64]),
    "artemis_backward_rays": (INT, [P, I64, P, P, P, I64, P, P, P, P, I64, INT, P, P, INT, INT,
                                    INT, INT, P, P, SZ, P]),
    "artemis_over_background": (INT, [P, P, INT, I64, INT, P, P, P]),
    "artemis_composite": (INT, [P, P, P, INT, I64, INT, P, P, P, P]),
    "artemis_straight_rgba": (INT, [P, P, INT, I64, P, P]),
    "artemis_rgba8": (INT, [P, P, INT, I64, P, P]),
    "artemis_asset_probe": (INT, [P, SZ, C.POINTER(AssetInfo)]),
    "artemis_asset_decode_leaves": (INT, [P, I64, P, P, SZ, P, P]),
    "artemis_asset_decode_rig": (INT, [P, SZ, C.POINTER(AssetInfo), C.POINTER(AssetRig), P, P,
                                       P, P, P, P]),
    "artemis_compact_workspace_bytes": (SZ, [I64]),
    "artemis_frame_compact": (INT, [P, P, P, INT, I64, INT, P, P, P, SZ, P]),
    "artemis_host_expand": (INT, [P, I64, INT, P, I64, P, P, P, P, INT]),
    "artemis_frame_bbox": (INT, [P, P, INT, INT, INT, P, P]),
    "artemis_copy_rect_d2h": (INT, [P, P, SZ, SZ, SZ, I64, I64, P]),
    "artemis_views_bbox": (INT, [P, P, INT, INT, INT, INT, P, P]),
    "artemis_views_copy_union_d2h": (INT, [INT, P, P, P, P, INT, INT, INT, INT, P, P]),
    "artemis_l1_grads": (INT, [P, P, P, P, I64, INT, P, P, P, P, P]),
    "artemis_mark_touched": (INT, [P, I64, P, P]),
    "artemis_vrt_workspace_bytes": (SZ, [I64, I64]),
    "artemis_vrt_grads": (INT, [P, I64, INT, P, I64, DBL, P, P, P, SZ, P]),
    "artemis_sparse_adam": (INT, [P, P, P, P, P, I64, INT, DBL, DBL, DBL, DBL, DBL, DBL, P]),
    "artemis_tiles_shard_floats": (I64, [INT, INT, INT, INT, INT]),
    "artemis_tiles_pack": (INT, [P, P, P, INT, INT, INT, INT, INT, P, P]),
    "artemis_tiles_unpack": (INT, [P, INT, INT, INT, INT, INT, P, P, P, P]),
    "artemis_host_checksum": (INT, [P, SZ, INT, P]),
    "artemis_host_widen_f32": (INT, [P, I64, I64, I64, P, I64, INT]),
    "artemis_host_pose_tables": (INT, [INT, P, P, P, P, P, P, P, P, P, P, P]),
    "artemis_debug_set_render_blocks": (INT, [INT]),
    "artemis_debug_set_flut_l2_resident": (INT, [INT]),
    "artemis_debug_division_selftest": (INT, [I64, C.c_uint64, P, P]),
}

EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen libartemis.so and declare every exported symbol (no device
    needed). Raises ExtensionMissing when the file is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ExtensionMissing(
                f"{path} is not built; run `python -m paper_2202_05628_b200.build_lib`")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_device_checked = False


def lib():
    """The library, after checking an sm_100 device is present."""
    global _device_checked
    L = load_library()
    if not _device_checked:
        if not L.artemis_device_ok():
            raise ExtensionMissing("no CUDA device of compute capability 10.x is visible; "
                                   "the ARTEMIS path has no CPU fallback")
        _device_checked = True
    return L


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    L = load_library()
    msg = L.artemis_status_string(status).decode()
    if status == ERR_CUDA or status == ERR_OOM:
        msg += " (" + L.artemis_last_cuda_error().decode() + ")"
    if status == ERR_RANGE:
        raise ValueError(f"{what}: {msg}")
    if status == ERR_EMPTY:
        raise ValueError(f"{what}: {msg}")
    if status == ERR_DUP:
        raise DuplicateMortonError(f"{what}: {msg}")
    if status == ERR_ARG:
        raise ContractViolation(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg}")
