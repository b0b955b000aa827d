"""TEST INFRASTRUCTURE: ctypes driver of the compiled reference library
(oracle/_ref/librlcuts_ref.so, see oracle/ref_capi.cpp)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1911_10217_b200 import _lib
from paper_1911_10217_b200.rlcuts import RenderConfig
from paper_1911_10217_b200.scenes import Scene

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "librlcuts_ref.so")

_P = C.c_void_p
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_lib_ref = None

_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_mix64": (C.c_uint64, [C.c_uint64]),
    "ref_rng_draws": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _dp]),
    "ref_run_create": (_P, [C.POINTER(_lib.SceneDescC), C.POINTER(_lib.RenderConfigC),
                            C.POINTER(C.c_int)]),
    "ref_run_destroy": (None, [_P]),
    "ref_run_pass": (C.c_int64, [_P, C.c_uint32, _dp]),
    "ref_run_render_only": (C.c_int, [_P, C.c_uint32]),
    "ref_run_framebuffer": (None, [_P, _dp, _u64p]),
    "ref_run_stats": (None, [_P, _u64p]),
    "ref_run_info": (None, [_P, _dp, _u32p]),
    "ref_run_export": (C.c_uint32, [_P, C.c_uint32, C.POINTER(_lib.CellKeyC), _u32p, _u32p, _dp,
                                    _dp, _u32p]),
    "ref_run_template": (None, [_P, _u32p, _u32p, _dp, _dp, _u32p, _dp]),
    "ref_run_occluded": (None, [_P, C.c_uint32, _dp, _dp, C.POINTER(C.c_uint8)]),
    "ref_run_intersect": (None, [_P, C.c_uint32, _dp, _dp, C.c_double, _dp, _i32p]),
    "ref_render_frame": (C.c_double, [C.POINTER(_lib.SceneDescC), C.POINTER(_lib.RenderConfigC),
                                      _dp, _u64p, _u32p, _dp, _dp]),
    "ref_run_update_scene": (C.c_int, [_P, C.POINTER(_lib.SceneDescC)]),
    "ref_image_write_pfm": (C.c_int, [_dp, C.c_int, C.c_int, C.c_char_p]),
    "ref_image_read_pfm": (C.c_int, [C.c_char_p, _dp, C.c_uint64, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]),
    "ref_image_write_ppm": (C.c_int, [_dp, C.c_int, C.c_int, C.c_char_p]),
    "ref_image_mse": (C.c_int, [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_int, _dp]),
    "ref_light_tree": (C.c_uint32, [C.c_uint32, _dp, _dp, _u32p, _i32p, _dp]),
    "ref_init_cut": (C.c_uint32, [C.c_uint32, _dp, _dp, C.c_uint32, C.c_double, _u32p, _u32p, _dp,
                                  _dp, _u32p, _dp]),
    "ref_split_collapse": (C.c_int64, [C.c_uint32, _dp, _dp, C.c_uint32, C.c_double, _dp, _u32p,
                                       C.c_double, C.c_uint32, _u32p, _u32p, _dp, _dp, _u32p]),
    "ref_update_q_seq": (C.c_int, [C.c_uint32, _dp, _u32p, C.c_double, C.c_double, C.c_uint32,
                                   C.c_uint32, _u32p, _dp, _dp]),
    "ref_sample_cluster": (None, [C.c_uint32, _dp, _dp, C.c_uint32, _dp, _u32p, _dp]),
    "ref_level_for_footprint": (C.c_int, [C.c_uint32, _dp, C.c_double, _u32p]),
    "ref_make_key": (C.c_int, [C.c_uint32, _dp, _dp, _u32p, _dp, _dp, C.c_double, C.c_uint32,
                               C.c_double, C.POINTER(_lib.CellKeyC), _u64p]),
    "ref_octa_encode": (None, [C.c_uint32, _dp, _dp]),
    "ref_run_slots": (C.c_uint32, [_P, C.c_uint32, _u32p, _u32p]),
    "ref_run_grid_views": (C.c_uint32, [C.c_void_p, C.c_char_p, C.c_uint32, _u64p, _u32p,
                                        C.c_uint32]),
}


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> C.CDLL:
    global _lib_ref
    if _lib_ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle ref` where "
                               "/root/reference is mounted")
        lib = C.CDLL(REF_LIB)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib_ref = lib
    return _lib_ref


def dp(a):
    return a.ctypes.data_as(_dp)


def up(a):
    return a.ctypes.data_as(_u32p)


def raise_ref(status: int):
    msg = ref_lib().ref_last_error().decode()
    if status == _lib.RLC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _lib.RLC_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


class RefRun:
    """One reference run: build_context + HashGrid + Framebuffer, passes
    driven one at a time (the loop body of render_frame, render.cpp:219-224)."""

    def __init__(self, scene: Scene, config: RenderConfig):
        lib = ref_lib()
        self.scene = scene
        self._desc = scene.desc()
        self._cfg = config.c()
        st = C.c_int()
        self.h = lib.ref_run_create(C.byref(self._desc), C.byref(self._cfg), C.byref(st))
        if not self.h:
            raise_ref(st.value)

    def update_scene(self, scene: Scene):
        """ctx' = build_context(scene, cfg) with the creation light tree
        (the semantics of rlc_context_update_scene)."""
        desc = scene.desc()
        st = ref_lib().ref_run_update_scene(self.h, C.byref(desc))
        if st:
            raise_ref(st)
        self.scene, self._desc = scene, desc

    def run_pass(self, pass_index: int) -> tuple[int, float]:
        ms = C.c_double()
        r = ref_lib().ref_run_pass(self.h, pass_index, C.byref(ms))
        if r < 0:
            raise_ref(-r)
        return int(r), ms.value

    def framebuffer(self):
        cam = self.scene.camera
        s = np.zeros((cam.height, cam.width, 3), np.float64)
        c = np.zeros((cam.height, cam.width), np.uint64)
        ref_lib().ref_run_framebuffer(self.h, dp(s), c.ctypes.data_as(_u64p))
        return s, c

    def stats(self) -> dict:
        o = np.zeros(4, np.uint64)
        ref_lib().ref_run_stats(self.h, o.ctypes.data_as(_u64p))
        return {"occupied": int(o[0]), "lookups": int(o[1]), "fallback_hits": int(o[2]),
                "cut_size": int(o[3])}

    def info(self) -> dict:
        d = np.zeros(2, np.float64)
        u = np.zeros(4, np.uint32)
        ref_lib().ref_run_info(self.h, dp(d), up(u))
        return {"base_tile": d[0], "shadow_eps": d[1], "num_triangles": int(u[0]),
                "num_emitters": int(u[1]), "bvh_nodes": int(u[2]), "light_tree_nodes": int(u[3])}

    def render_only(self, pass_index: int):
        """render_pass alone (no end_of_pass_update): the touched slots stay set."""
        st = ref_lib().ref_run_render_only(self.h, pass_index)
        if st:
            raise_ref(st)

    def grid_views(self) -> tuple[str, int, list]:
        """HashGrid::dump_stats text, memory_records and the CellKeys of
        touched_slots() in slot order."""
        buf = C.create_string_buffer(1 << 16)
        mem = np.zeros(1, np.uint64)
        cap = max(self.stats()["occupied"], 1)
        keys = np.zeros(5 * cap, np.uint32)
        n = ref_lib().ref_run_grid_views(self.h, buf, len(buf), mem.ctypes.data_as(_u64p),
                                         up(keys), cap)
        k = keys.view(np.int32).reshape(-1, 5)
        touched = [(int(k[i, 0]), int(k[i, 1]), int(k[i, 2]), int(keys[5 * i + 3]),
                    int(keys[5 * i + 4])) for i in range(min(n, cap))]
        return buf.value.decode(), int(mem[0]), touched

    def slots(self) -> list:
        """Occupied slots in slot order: (slot, CellKey)."""
        n = max(self.stats()["occupied"], 1)
        slot = np.zeros(n, np.uint32)
        keys = np.zeros(5 * n, np.uint32)
        got = ref_lib().ref_run_slots(self.h, n, up(slot), up(keys))
        k = keys.view(np.int32).reshape(-1, 5)
        return [(int(slot[i]), (int(k[i, 0]), int(k[i, 1]), int(k[i, 2]), int(keys[5 * i + 3]),
                                int(keys[5 * i + 4]))) for i in range(min(got, n))]

    def export(self) -> dict:
        st = self.stats()
        n, m = st["occupied"], st["cut_size"]
        keys = (_lib.CellKeyC * max(n, 1))()
        node = np.zeros((max(n, 1), m), np.uint32)
        ends = np.zeros_like(node)
        vis = np.zeros_like(node)
        q = np.zeros((max(n, 1), m), np.float64)
        cdf = np.zeros_like(q)
        got = ref_lib().ref_run_export(self.h, n, keys, up(node), up(ends), dp(q), dp(cdf), up(vis))
        assert got == n, (got, n)
        out = {}
        for i in range(n):
            k = keys[i]
            out[(k.qx, k.qy, k.qz, k.qn, k.level)] = {
                "node_ids": node[i], "ends": ends[i], "q": q[i], "cdf": cdf[i], "visits": vis[i]}
        return out

    def occluded(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(a.shape[0], np.uint8)
        ref_lib().ref_run_occluded(self.h, a.shape[0], dp(a), dp(b),
                                   out.ctypes.data_as(C.POINTER(C.c_uint8)))
        return out.astype(bool)

    def intersect(self, org: np.ndarray, d: np.ndarray, t_min: float = 0.0):
        org = np.ascontiguousarray(org, np.float64)
        d = np.ascontiguousarray(d, np.float64)
        t = np.zeros(org.shape[0], np.float64)
        tri = np.zeros(org.shape[0], np.int32)
        ref_lib().ref_run_intersect(self.h, org.shape[0], dp(org), dp(d), t_min, dp(t),
                                    tri.ctypes.data_as(_i32p))
        return t, tri

    def close(self):
        if self.h:
            ref_lib().ref_run_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_render_frame(scene: Scene, config: RenderConfig, reference=None):
    """The stock reference render_frame (render.cpp:202-240), optionally
    scored against `reference` (h x w x 3) after every pass."""
    cam = scene.camera
    img = np.zeros((cam.height, cam.width, 3), np.float64)
    stats = np.zeros(3, np.uint64)
    ch = np.zeros(max(config.passes, 1), np.uint32)
    pm = np.zeros(max(config.passes, 1))
    desc = scene.desc()
    cfg = config.c()
    ref = None if reference is None else np.ascontiguousarray(reference, np.float64)
    ms = ref_lib().ref_render_frame(C.byref(desc), C.byref(cfg), dp(img),
                                    stats.ctypes.data_as(_u64p), up(ch),
                                    None if ref is None else dp(ref),
                                    None if ref is None else dp(pm))
    if ms < 0:
        raise RuntimeError(ref_lib().ref_last_error().decode())
    return {"image": img, "wall_ms": ms, "occupied": int(stats[0]), "lookups": int(stats[1]),
            "fallback_hits": int(stats[2]), "sc_changes": ch[:config.passes].tolist(),
            "pass_mse": pm[:config.passes].tolist() if ref is not None else []}


def _img_status(r: int):
    if r:
        raise RuntimeError(f"reference image call failed ({r}): "
                           + ref_lib().ref_last_error().decode())


def ref_write_pfm(image, path):
    im = np.ascontiguousarray(image, np.float64)
    _img_status(ref_lib().ref_image_write_pfm(dp(im), im.shape[1], im.shape[0], str(path).encode()))


def ref_read_pfm(path):
    w, h = C.c_int(), C.c_int()
    _img_status(ref_lib().ref_image_read_pfm(str(path).encode(), None, 0, C.byref(w), C.byref(h)))
    img = np.zeros((h.value, w.value, 3))
    _img_status(ref_lib().ref_image_read_pfm(str(path).encode(), dp(img), w.value * h.value,
                                             C.byref(w), C.byref(h)))
    return img


def ref_write_ppm(image, path):
    im = np.ascontiguousarray(image, np.float64)
    _img_status(ref_lib().ref_image_write_ppm(dp(im), im.shape[1], im.shape[0], str(path).encode()))


def ref_mse(a, b, relative=False):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    out = C.c_double()
    _img_status(ref_lib().ref_image_mse(dp(a), a.shape[1], a.shape[0], dp(b), b.shape[1],
                                        b.shape[0], int(relative), C.byref(out)))
    return out.value
