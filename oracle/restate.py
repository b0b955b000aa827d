"""TEST INFRASTRUCTURE: ctypes driver of the CPU restatement
(oracle/rlc_oracle.cpp -> oracle/librlc_oracle.so)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1911_10217_b200 import _lib
from paper_1911_10217_b200.rlcuts import RenderConfig
from paper_1911_10217_b200.scenes import Scene

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "librlc_oracle.so")

_P = C.c_void_p
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)
_lib_orc = None

_SIGS = {
    "orc_last_error": (C.c_char_p, []),
    "orc_mix64": (C.c_uint64, [C.c_uint64]),
    "orc_rng_draws": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _dp]),
    "orc_run_create": (_P, [C.POINTER(_lib.SceneDescC), C.POINTER(_lib.RenderConfigC),
                            C.POINTER(C.c_int)]),
    "orc_run_destroy": (None, [_P]),
    "orc_run_pass": (C.c_int64, [_P, C.c_uint32]),
    "orc_run_framebuffer": (None, [_P, _dp, _u64p]),
    "orc_run_stats": (None, [_P, _u64p]),
    "orc_run_export": (C.c_uint32, [_P, C.c_uint32, C.POINTER(_lib.CellKeyC), _u32p, _u32p, _dp,
                                    _dp, _u32p]),
    "orc_run_samples": (C.c_uint32, [_P, C.c_uint32, _u32p, _dp]),
    "orc_run_trav_stats": (None, [_P, _u64p]),
    "orc_run_trace": (C.c_int64, [_P, C.c_uint32, C.c_uint32, C.c_uint32]),
    "orc_run_records": (None, [_P, _P]),
    "orc_run_fold": (C.c_int, [_P, _P, _u64p, C.c_uint32, C.c_uint32, C.c_uint64]),
    "orc_run_end_of_pass": (C.c_int64, [_P]),
    "orc_run_occluded": (None, [_P, C.c_uint32, _dp, _dp, C.POINTER(C.c_uint8)]),
    "orc_light_tree": (C.c_uint32, [C.c_uint32, _dp, _dp, _u32p, _i32p, _dp]),
    "orc_init_cut": (C.c_uint32, [C.c_uint32, _dp, _dp, C.c_uint32, C.c_double, _u32p, _u32p, _dp,
                                  _dp, _u32p, _dp]),
    "orc_split_collapse": (C.c_int64, [C.c_uint32, _dp, _dp, C.c_uint32, C.c_double, _dp, _u32p,
                                       C.c_double, C.c_uint32, _u32p, _u32p, _dp, _dp, _u32p]),
    "orc_update_q_seq": (C.c_int, [C.c_uint32, _dp, _u32p, C.c_double, C.c_double, C.c_uint32,
                                   C.c_uint32, _u32p, _dp, _dp]),
    "orc_sample_cluster": (None, [C.c_uint32, _dp, _dp, C.c_uint32, _dp, _u32p, _dp]),
    "orc_level_for_footprint": (C.c_int, [C.c_uint32, _dp, C.c_double, _u32p]),
    "orc_make_key": (C.c_int, [C.c_uint32, _dp, _dp, _u32p, _dp, _dp, C.c_double, C.c_uint32,
                               C.c_double, C.POINTER(_lib.CellKeyC), _u64p]),
    "orc_octa_encode": (None, [C.c_uint32, _dp, _dp]),
}


def oracle_lib() -> C.CDLL:
    global _lib_orc
    if _lib_orc is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle oracle`")
        lib = C.CDLL(ORACLE_LIB)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib_orc = lib
    return _lib_orc


def _dp_(a):
    return a.ctypes.data_as(_dp)


def _up_(a):
    return a.ctypes.data_as(_u32p)


def _raise(status: int):
    msg = oracle_lib().orc_last_error().decode()
    if status == _lib.RLC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _lib.RLC_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


class OracleRun:
    """Restated render_pass + end_of_pass_update as the deferred fold."""

    def __init__(self, scene: Scene, config: RenderConfig):
        self.scene = scene
        self._desc = scene.desc()
        self._cfg = config.c()
        st = C.c_int()
        self.h = oracle_lib().orc_run_create(C.byref(self._desc), C.byref(self._cfg), C.byref(st))
        if not self.h:
            _raise(st.value)

    def run_pass(self, pass_index: int) -> int:
        r = oracle_lib().orc_run_pass(self.h, pass_index)
        if r < 0:
            _raise(-r)
        return int(r)

    def framebuffer(self):
        cam = self.scene.camera
        s = np.zeros((cam.height, cam.width, 3), np.float64)
        c = np.zeros((cam.height, cam.width), np.uint64)
        oracle_lib().orc_run_framebuffer(self.h, _dp_(s), c.ctypes.data_as(_u64p))
        return s, c

    def stats(self) -> dict:
        o = np.zeros(4, np.uint64)
        oracle_lib().orc_run_stats(self.h, o.ctypes.data_as(_u64p))
        return {"occupied": int(o[0]), "lookups": int(o[1]), "fallback_hits": int(o[2]),
                "cut_size": int(o[3])}

    def export(self) -> dict:
        st = self.stats()
        n, m = st["occupied"], st["cut_size"]
        keys = (_lib.CellKeyC * max(n, 1))()
        node = np.zeros((max(n, 1), m), np.uint32)
        ends = np.zeros_like(node)
        vis = np.zeros_like(node)
        q = np.zeros((max(n, 1), m), np.float64)
        cdf = np.zeros_like(q)
        oracle_lib().orc_run_export(self.h, n, keys, _up_(node), _up_(ends), _dp_(q), _dp_(cdf),
                                    _up_(vis))
        return {(keys[i].qx, keys[i].qy, keys[i].qz, keys[i].qn, keys[i].level):
                {"node_ids": node[i], "ends": ends[i], "q": q[i], "cdf": cdf[i], "visits": vis[i]}
                for i in range(n)}

    def samples(self) -> dict:
        """Light samples of the last pass in canonical order."""
        n = oracle_lib().orc_run_samples(self.h, 0, None, None)
        u = np.zeros((max(n, 1), 4), np.uint32)
        f = np.zeros((max(n, 1), 6), np.float64)
        oracle_lib().orc_run_samples(self.h, n, _up_(u), _dp_(f))
        return {"pixel": u[:n, 0], "cluster": u[:n, 1], "emitter": u[:n, 2],
                "fallback": u[:n, 3].astype(bool), "q_before": f[:n, 0], "v": f[:n, 1],
                "radiance": f[:n, 2:5], "total": f[:n, 5]}

    # ---- sharded pass (CPU model of the replicated rlc_shard_* protocol) ----
    def trace(self, pass_index: int, rows: tuple) -> int:
        r = oracle_lib().orc_run_trace(self.h, pass_index, rows[0], rows[1])
        if r < 0:
            _raise(-r)
        self._n = int(r)
        return self._n

    def records(self) -> np.ndarray:
        from paper_1911_10217_b200.rlcuts import RECORD_DTYPE
        out = np.zeros(self._n, RECORD_DTYPE)
        oracle_lib().orc_run_records(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def fold(self, all_records: np.ndarray, counts, rank: int, stride: int):
        c = np.ascontiguousarray(counts, np.uint64)
        buf = np.ascontiguousarray(all_records)
        st = oracle_lib().orc_run_fold(self.h, buf.ctypes.data_as(C.c_void_p),
                                       c.ctypes.data_as(_u64p), len(c), rank, stride)
        if st:
            _raise(st)

    def end_of_pass(self) -> int:
        return int(oracle_lib().orc_run_end_of_pass(self.h))

    def trav_stats(self) -> dict:
        """Mean nodes / triangles tested per primary and per shadow ray so far
        (reference BVH and traversal order)."""
        o = np.zeros(6, np.uint64)
        oracle_lib().orc_run_trav_stats(self.h, o.ctypes.data_as(_u64p))
        pr, sr = max(int(o[0]), 1), max(int(o[3]), 1)
        return {"primary_rays": int(o[0]), "primary_nodes": int(o[1]) / pr,
                "primary_tris": int(o[2]) / pr, "shadow_rays": int(o[3]),
                "shadow_nodes": int(o[4]) / sr, "shadow_tris": int(o[5]) / sr}

    def occluded(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(a.shape[0], np.uint8)
        oracle_lib().orc_run_occluded(self.h, a.shape[0], _dp_(a), _dp_(b),
                                      out.ctypes.data_as(C.POINTER(C.c_uint8)))
        return out.astype(bool)

    def close(self):
        if self.h:
            oracle_lib().orc_run_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- unit-level wrappers shared with the reference driver (oracle.ref) ----

def unit_api(lib, prefix: str):
    """Uniform Python wrappers over the ``<prefix>_*`` unit entry points of
    either the restatement (prefix 'orc') or the reference wrapper ('ref')."""
    f = lambda name: getattr(lib, f"{prefix}_{name}")  # noqa: E731
    err = f("last_error")

    def check(status):
        if status != 0:
            msg = err().decode()
            if status == _lib.RLC_ERR_INVALID_ARGUMENT:
                raise ValueError(msg)
            if status == _lib.RLC_ERR_OUT_OF_RANGE:
                raise IndexError(msg)
            raise RuntimeError(msg)

    def light_tree(centroids, energies):
        c = np.ascontiguousarray(centroids, np.float64).reshape(-1, 3)
        e = np.ascontiguousarray(energies, np.float64)
        n = len(e)
        order = np.zeros(max(n, 1), np.uint32)
        nodes = np.zeros((max(2 * n - 1, 1), 5), np.int32)
        en = np.zeros(max(2 * n - 1, 1), np.float64)
        k = f("light_tree")(n, _dp_(c), _dp_(e), _up_(order), nodes.ctypes.data_as(_i32p), _dp_(en))
        if k == 0:
            raise ValueError(err().decode())
        return order[:n], nodes[:k], en[:k]

    def init_cut(centroids, energies, M, eps=-1.0):
        c = np.ascontiguousarray(centroids, np.float64).reshape(-1, 3)
        e = np.ascontiguousarray(energies, np.float64)
        m = max(min(M, len(e)), 1)
        node, ends, vis = (np.zeros(m, np.uint32) for _ in range(3))
        q, cdf = np.zeros(m), np.zeros(m)
        eo = C.c_double()
        k = f("init_cut")(len(e), _dp_(c), _dp_(e), M, eps, _up_(node), _up_(ends), _dp_(q),
                          _dp_(cdf), _up_(vis), C.byref(eo))
        if k == 0:
            raise ValueError(err().decode())
        return {"node_ids": node, "ends": ends, "q": q, "cdf": cdf, "visits": vis,
                "eps_q": eo.value}

    def split_collapse(centroids, energies, M, q_in, threshold, iterations, eps=-1.0,
                       visits_in=None):
        c = np.ascontiguousarray(centroids, np.float64).reshape(-1, 3)
        e = np.ascontiguousarray(energies, np.float64)
        qi = np.ascontiguousarray(q_in, np.float64)
        m = len(qi)
        vi = None if visits_in is None else _up_(np.ascontiguousarray(visits_in, np.uint32))
        node, ends, vis = (np.zeros(m, np.uint32) for _ in range(3))
        q, cdf = np.zeros(m), np.zeros(m)
        ch = f("split_collapse")(len(e), _dp_(c), _dp_(e), M, eps, _dp_(qi), vi, threshold,
                                 iterations, _up_(node), _up_(ends), _dp_(q), _dp_(cdf), _up_(vis))
        if ch < 0:
            check(-ch)
        return int(ch), {"node_ids": node, "ends": ends, "q": q, "cdf": cdf, "visits": vis}

    def update_q_seq(q, visits, eps, alpha, schedule, s, v):
        q = np.array(q, np.float64)
        visits = np.array(visits, np.uint32)
        s = np.ascontiguousarray(s, np.uint32)
        v = np.ascontiguousarray(v, np.float64)
        qb = np.zeros(max(len(s), 1))
        check(f("update_q_seq")(len(q), _dp_(q), _up_(visits), eps, alpha, schedule, len(s),
                                _up_(s), _dp_(v), _dp_(qb)))
        return q, visits, qb[:len(s)]

    def sample_cluster(q, cdf, u):
        q = np.ascontiguousarray(q, np.float64)
        cdf = np.ascontiguousarray(cdf, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        s = np.zeros(len(u), np.uint32)
        p = np.zeros(len(u))
        f("sample_cluster")(len(q), _dp_(q), _dp_(cdf), len(u), _dp_(u), _up_(s), _dp_(p))
        return s, p

    def level_for_footprint(area_pdf, base_tile):
        a = np.ascontiguousarray(np.atleast_1d(area_pdf), np.float64)
        out = np.zeros(len(a), np.uint32)
        check(f("level_for_footprint")(len(a), _dp_(a), base_tile, _up_(out)))
        return out

    def make_key(pos, nrm, level, ju1, ju2, base_tile, normal_bits=4, jitter_scale=0.0):
        pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
        nrm = np.ascontiguousarray(nrm, np.float64).reshape(-1, 3)
        n = pos.shape[0]
        level = np.ascontiguousarray(np.broadcast_to(level, n), np.uint32)
        ju1 = np.ascontiguousarray(np.broadcast_to(ju1, n), np.float64)
        ju2 = np.ascontiguousarray(np.broadcast_to(ju2, n), np.float64)
        keys = (_lib.CellKeyC * max(n, 1))()
        h = np.zeros(n, np.uint64)
        check(f("make_key")(n, _dp_(pos), _dp_(nrm), _up_(level), _dp_(ju1), _dp_(ju2), base_tile,
                            normal_bits, jitter_scale, keys, h.ctypes.data_as(_u64p)))
        return [(k.qx, k.qy, k.qz, k.qn, k.level) for k in keys[:n]], h

    def octa_encode(nrm):
        nrm = np.ascontiguousarray(nrm, np.float64).reshape(-1, 3)
        uv = np.zeros((nrm.shape[0], 2))
        f("octa_encode")(nrm.shape[0], _dp_(nrm), _dp_(uv))
        return uv

    def rng_draws(seed, a, b=0, c=0, n=8):
        out = np.zeros(n)
        f("rng_draws")(seed, a, b, c, n, _dp_(out))
        return out

    return dict(light_tree=light_tree, init_cut=init_cut, split_collapse=split_collapse,
                update_q_seq=update_q_seq, sample_cluster=sample_cluster,
                level_for_footprint=level_for_footprint, make_key=make_key,
                octa_encode=octa_encode, rng_draws=rng_draws, mix64=f("mix64"))


def oracle_units() -> dict:
    return unit_api(oracle_lib(), "orc")
