"""ctypes view of the C-ABI in include/rlcuts_b200.h.

Loads the in-tree ``librlcuts_b200.so`` (built by ``__graft_entry__.build()``).
There is no fallback: a missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RLC_LIB_PATH") or os.path.join(HERE, "librlcuts_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "rlcuts_b200.h")

RLC_OK = 0
RLC_ERR_INVALID_ARGUMENT = 1
RLC_ERR_OUT_OF_RANGE = 2
RLC_ERR_CUDA = 3
RLC_ERR_NO_DEVICE = 4
RLC_ERR_INTERNAL = 5
RLC_ERR_IO = 6
RLC_ERR_PARSE = 7


class CutConfigC(C.Structure):
    _fields_ = [("cut_size", C.c_uint32), ("iterations", C.c_uint32), ("alpha", C.c_double),
                ("split_threshold", C.c_double), ("eps_q", C.c_double),
                ("alpha_schedule", C.c_uint32), ("_pad", C.c_uint32)]


class HashConfigC(C.Structure):
    _fields_ = [("capacity", C.c_uint32), ("probe_limit", C.c_uint32),
                ("normal_bits", C.c_uint32), ("_pad", C.c_uint32),
                ("base_tile", C.c_double), ("jitter_scale", C.c_double)]


class RenderConfigC(C.Structure):
    _fields_ = [("spp", C.c_uint32), ("passes", C.c_uint32), ("max_depth", C.c_uint32),
                ("sampler", C.c_uint32), ("cut", CutConfigC), ("hash", HashConfigC),
                ("seed", C.c_uint64), ("workers", C.c_uint32), ("_pad", C.c_uint32)]


class SceneDescC(C.Structure):
    _fields_ = [("num_triangles", C.c_uint32), ("num_materials", C.c_uint32),
                ("vertices", C.POINTER(C.c_double)), ("material_ids", C.POINTER(C.c_uint32)),
                ("materials", C.POINTER(C.c_double)), ("cam_origin", C.c_double * 3),
                ("cam_look_at", C.c_double * 3), ("cam_up", C.c_double * 3),
                ("vfov_degrees", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class CellKeyC(C.Structure):
    _fields_ = [("qx", C.c_int32), ("qy", C.c_int32), ("qz", C.c_int32),
                ("qn", C.c_uint32), ("level", C.c_uint32)]


class RenderResultC(C.Structure):
    _fields_ = [("wall_ms", C.c_double), ("occupied_cells", C.c_uint32),
                ("num_passes", C.c_uint32), ("lookups", C.c_uint64),
                ("fallback_hits", C.c_uint64), ("sc_changes", C.POINTER(C.c_uint32))]


class GridStatsC(C.Structure):
    _fields_ = [("occupied", C.c_uint32), ("cut_size", C.c_uint32), ("lookups", C.c_uint64),
                ("fallback_hits", C.c_uint64), ("pending_lookups", C.c_uint64),
                ("new_keys", C.c_uint64)]


class ContextInfoC(C.Structure):
    _fields_ = [("num_triangles", C.c_uint32), ("num_emitters", C.c_uint32),
                ("bvh_nodes", C.c_uint32), ("light_tree_nodes", C.c_uint32),
                ("base_tile", C.c_double), ("shadow_eps", C.c_double),
                ("device_bytes", C.c_uint64)]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)

# name -> (restype, argtypes)
SIGNATURES = {
    "rlc_last_error": (C.c_char_p, []),
    "rlc_abi_version": (C.c_int, []),
    "rlc_kernel_launches": (C.c_uint64, []),
    "rlc_render_config_default": (C.c_int, [C.POINTER(RenderConfigC)]),
    "rlc_context_create": (C.c_int, [C.POINTER(SceneDescC), C.POINTER(RenderConfigC), C.c_int, _PP]),
    "rlc_context_destroy": (C.c_int, [_P]),
    "rlc_context_info_get": (C.c_int, [_P, C.POINTER(ContextInfoC)]),
    "rlc_context_set_stream": (C.c_int, [_P, _P]),
    "rlc_context_synchronize": (C.c_int, [_P]),
    "rlc_context_enable_timing": (C.c_int, [_P, C.c_int]),
    "rlc_context_stage_times": (C.c_int, [_P, _dp, _u32p]),
    "rlc_context_stage_marks": (C.c_int, [_P, C.c_uint32, _dp, _u32p]),
    "rlc_occluded_batch": (C.c_int, [_P, C.c_uint32, _dp, _dp, C.POINTER(C.c_uint8)]),
    "rlc_libm_variant": (C.c_int, [C.POINTER(C.c_int32)]),
    "rlc_libm_sincos": (C.c_int, [_P, C.c_uint32, _dp, _dp, _dp]),
    "rlc_libm_sincos_host": (C.c_int, [C.c_int32, C.c_uint64, _dp, _dp, _dp]),
    "rlc_intersect_batch": (C.c_int, [_P, C.c_uint32, _dp, _dp, C.c_double, _dp,
                                      C.POINTER(C.c_int32)]),
    "rlc_debug_trav_stats": (C.c_int, [C.c_int32, C.POINTER(C.c_uint64)]),
    "rlc_work_counters": (C.c_int, [C.c_int32, C.POINTER(C.c_uint64)]),
    "rlc_context_count_work": (C.c_int, [_P, C.c_int]),
    "rlc_debug_host_bvh": (C.c_int, [C.POINTER(SceneDescC), C.c_uint32, _dp, _u32p]),
    "rlc_measure_l2_bandwidth": (C.c_int, [C.c_int, _dp]),
    "rlc_render_passes_async": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, C.c_uint32,
                                          _P, _P]),
    "rlc_grid_slots": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                 C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_uint32)]),
    "rlc_intersect_batch_sah": (C.c_int, [_P, C.c_uint32, _dp, _dp, C.c_double, _dp,
                                          C.POINTER(C.c_int32)]),
    "rlc_grid_create": (C.c_int, [_P, C.POINTER(RenderConfigC), _PP]),
    "rlc_grid_destroy": (C.c_int, [_P]),
    "rlc_grid_stats_get": (C.c_int, [_P, C.POINTER(GridStatsC)]),
    "rlc_grid_export": (C.c_int, [_P, C.c_uint32, C.POINTER(CellKeyC), _u32p, _u32p, _dp, _dp,
                                  _u32p, _u32p]),
    "rlc_grid_template": (C.c_int, [_P, _u32p, _u32p, _dp, _dp, _u32p, _dp]),
    "rlc_framebuffer_create": (C.c_int, [_P, C.c_int32, C.c_int32, _PP]),
    "rlc_framebuffer_destroy": (C.c_int, [_P]),
    "rlc_framebuffer_clear": (C.c_int, [_P]),
    "rlc_framebuffer_download": (C.c_int, [_P, _dp, _u64p]),
    "rlc_framebuffer_resolve": (C.c_int, [_P, _dp]),
    "rlc_render_pass": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, _P]),
    "rlc_render_pass_rows": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, _P,
                                       C.c_uint32, C.c_uint32]),
    "rlc_end_of_pass_update": (C.c_int, [_P, _P, C.POINTER(CutConfigC), _u32p]),
    "rlc_render_pass_async": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, _P]),
    "rlc_end_of_pass_update_async": (C.c_int, [_P, _P, C.POINTER(CutConfigC)]),
    "rlc_grid_last_changes": (C.c_int, [_P, _u32p]),
    "rlc_shard_trace": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, C.c_uint32,
                                  C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), _u64p]),
    "rlc_shard_fold": (C.c_int, [_P, C.POINTER(RenderConfigC), _P, _P, C.c_uint32, C.c_uint32,
                                 C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _u64p]),
    "rlc_shard_trace_to": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, C.c_uint32,
                                     C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(C.c_void_p),
                                     C.c_uint32]),
    "rlc_comm_enable_peer_exchange": (C.c_int, [_P, C.c_uint64, C.c_int]),
    "rlc_shard_entry_arrays": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _u64p]),
    "rlc_shard_finish": (C.c_int, [_P, _P, _P, C.c_uint32, C.c_int]),
    "rlc_shard_sync": (C.c_int, [_P, _P]),
    "rlc_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "rlc_comm_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8), _PP]),
    "rlc_comm_destroy": (C.c_int, [_P]),
    "rlc_shard_frame": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, _P, _P, _P, C.c_uint32,
                                  C.c_uint32, C.c_uint64, C.c_int]),
    "rlc_shard_frames": (C.c_int, [_P, C.POINTER(RenderConfigC), C.c_uint32, C.c_uint32, _P, _P, _P,
                                   C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_int]),
    "rlc_render_frame": (C.c_int, [_P, C.POINTER(RenderConfigC), _dp, C.POINTER(RenderResultC)]),
    "rlc_context_enable_sample_export": (C.c_int, [_P, C.c_int]),
    "rlc_context_set_pdf_mode": (C.c_int, [_P, C.c_int]),
    "rlc_pass_samples": (C.c_int, [_P, C.c_uint64, C.c_void_p, _u64p]),
    "rlc_context_update_scene": (C.c_int, [_P, C.POINTER(SceneDescC)]),
    "rlc_context_prepare_scene": (C.c_int, [_P, C.POINTER(SceneDescC), _u64p]),
    "rlc_context_commit_scene": (C.c_int, [_P, C.c_uint64]),
    "rlc_render_frame_scored": (C.c_int, [_P, C.POINTER(RenderConfigC), _dp, C.c_int32, C.c_int32,
                                          _dp, C.POINTER(RenderResultC), _dp]),
    "rlc_image_write_pfm": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_char_p]),
    "rlc_image_read_pfm": (C.c_int, [C.c_char_p, _dp, C.c_uint64, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]),
    "rlc_image_write_ppm": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_char_p]),
    "rlc_image_mse": (C.c_int, [_dp, C.c_int32, C.c_int32, _dp, C.c_int32, C.c_int32, _dp]),
    "rlc_image_relative_mse": (C.c_int, [_dp, C.c_int32, C.c_int32, _dp, C.c_int32, C.c_int32,
                                         _dp]),
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library (no fallback: raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (the CUDA path has no "
            "CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def declared_functions() -> list[str]:
    """Function names declared in include/rlcuts_b200.h."""
    import re
    text = open(HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rlc_[a-z0-9_]+)\s*\(", text)))
