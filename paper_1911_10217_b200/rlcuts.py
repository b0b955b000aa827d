"""Python mirror of the reference's public render API (proj/include/rlcuts/)
over the C-ABI (include/rlcuts_b200.h).

Same names, argument meaning and error behaviour as the reference:
``std::invalid_argument`` -> ``ValueError``, ``std::out_of_range`` ->
``IndexError``.  Every call runs on the B200 through librlcuts_b200.so; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .scenes import Scene


class NoDeviceError(RuntimeError):
    pass


class DeviceError(RuntimeError):
    pass


class ImageIoError(RuntimeError):
    """ImageIoError (image.hpp:15-28); .code is "io_error" or "parse_error"."""

    def __init__(self, msg: str, code: str):
        super().__init__(msg)
        self.code = code


def _check(status: int):
    if status == _lib.RLC_OK:
        return
    msg = _lib.load().rlc_last_error().decode(errors="replace")
    if status == _lib.RLC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == _lib.RLC_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if status == _lib.RLC_ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    if status in (_lib.RLC_ERR_IO, _lib.RLC_ERR_PARSE):
        raise ImageIoError(msg, "io_error" if status == _lib.RLC_ERR_IO else "parse_error")
    raise DeviceError(msg)


class SamplerKind(enum.IntEnum):  # estimators.hpp:16-20
    uniform = 0
    energy = 1
    rl_lightcuts = 2


class AlphaSchedule(enum.IntEnum):  # cut.hpp:16-19
    fixed = 0
    harmonic = 1


@dataclass
class CutConfig:  # cut.hpp:21-28
    cut_size: int = 128
    alpha: float = 0.2
    split_threshold: float = 4.0
    eps_q: float = -1.0
    iterations: int = 1
    alpha_schedule: AlphaSchedule = AlphaSchedule.fixed

    def c(self) -> _lib.CutConfigC:
        return _lib.CutConfigC(self.cut_size, self.iterations, self.alpha, self.split_threshold,
                               self.eps_q, int(self.alpha_schedule), 0)


@dataclass
class HashConfig:  # hash_grid.hpp:17-23
    capacity: int = 1 << 16
    base_tile: float = 0.0
    probe_limit: int = 32
    normal_bits: int = 4
    jitter_scale: float = 0.0

    def c(self) -> _lib.HashConfigC:
        return _lib.HashConfigC(self.capacity, self.probe_limit, self.normal_bits, 0,
                                self.base_tile, self.jitter_scale)


@dataclass
class RenderConfig:  # render.hpp:17-26
    spp: int = 16
    passes: int = 4
    max_depth: int = 1
    sampler: SamplerKind = SamplerKind.uniform
    cut: CutConfig = field(default_factory=CutConfig)
    hash: HashConfig = field(default_factory=HashConfig)
    seed: int = 1
    workers: int = 1

    def c(self) -> _lib.RenderConfigC:
        return _lib.RenderConfigC(self.spp, self.passes, self.max_depth, int(self.sampler),
                                  self.cut.c(), self.hash.c(), self.seed, self.workers, 0)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _uptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


class RenderContext:
    """build_context (proj/src/render.cpp:143-157), device resident."""

    def __init__(self, scene: Scene, config: RenderConfig, device: int = 0):
        lib = _lib.load()
        self.scene = scene
        self._desc = scene.desc()
        self._cfg = config.c()
        h = C.c_void_p()
        _check(lib.rlc_context_create(C.byref(self._desc), C.byref(self._cfg), device, C.byref(h)))
        self.handle = h

    def info(self) -> dict:
        i = _lib.ContextInfoC()
        _check(_lib.load().rlc_context_info_get(self.handle, C.byref(i)))
        return {k: getattr(i, k) for k, _ in _lib.ContextInfoC._fields_}

    def update_scene(self, scene: Scene):
        """Dynamic emitters (rlc_context_update_scene): render `scene` from now
        on with the light tree of this context's creation, so the learned cuts
        of its hash grids stay valid.  Vertices and camera pose may change."""
        desc = scene.desc()
        _check(_lib.load().rlc_context_update_scene(self.handle, C.byref(desc)))
        self.scene, self._desc = scene, desc

    def prepare_scene(self, scene: Scene) -> int:
        """Start the host build of a later frame's scene (rlc_context_prepare_scene);
        returns the token commit_scene takes."""
        desc = scene.desc()
        tok = C.c_uint64()
        _check(_lib.load().rlc_context_prepare_scene(self.handle, C.byref(desc), C.byref(tok)))
        return tok.value

    def commit_scene(self, token: int, scene: Scene | None = None):
        """Make a prepared scene the context's (rlc_context_commit_scene)."""
        _check(_lib.load().rlc_context_commit_scene(self.handle, token))
        if scene is not None:
            self.scene = scene

    @property
    def base_tile(self) -> float:
        return self.info()["base_tile"]

    def set_stream(self, stream_ptr: int | None):
        _check(_lib.load().rlc_context_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))

    STAGES = ("primary", "sample", "sort", "fold", "accumulate", "split_collapse", "shadow",
              "insert", "compact", "exchange_keys")

    def count_work(self, on: bool = True):
        """k_shadow's counting instance on/off (rlc_context_count_work)."""
        _check(_lib.load().rlc_context_count_work(self.handle, 1 if on else 0))

    def enable_timing(self, on: bool = True):
        _check(_lib.load().rlc_context_enable_timing(self.handle, 1 if on else 0))

    def stage_times(self) -> dict:
        """{stage: (total_ms, launches)} since the last call (CUDA events)."""
        ms = np.zeros(len(self.STAGES), np.float64)
        cnt = np.zeros(len(self.STAGES), np.uint32)
        _check(_lib.load().rlc_context_stage_times(self.handle, _dptr(ms), _uptr(cnt)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.STAGES)}

    def stage_marks(self) -> list:
        """[(stage name, start ms, end ms)] of every timed stage launch since
        the last stage_times() (read before calling it), from the first."""
        lib = _lib.load()
        n = C.c_uint32()
        _check(lib.rlc_context_stage_marks(self.handle, 0, None, C.byref(n)))
        out = np.zeros(3 * max(n.value, 1))
        _check(lib.rlc_context_stage_marks(self.handle, n.value, _dptr(out), C.byref(n)))
        return [(self.STAGES[int(out[3 * i])], out[3 * i + 1], out[3 * i + 2])
                for i in range(n.value)]

    def libm_sincos(self, x: np.ndarray):
        """The bounce sampler's sin/cos on the device (rlc_libm.h)."""
        x = np.ascontiguousarray(x, np.float64).ravel()
        s, c = np.empty_like(x), np.empty_like(x)
        _check(_lib.load().rlc_libm_sincos(self.handle, x.size, _dptr(x), _dptr(s), _dptr(c)))
        return s, c

    def occluded(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """occluded() (bvh.hpp:38-40) for n segments (n x 3 endpoints)."""
        a = np.ascontiguousarray(a, np.float64).reshape(-1, 3)
        b = np.ascontiguousarray(b, np.float64).reshape(-1, 3)
        out = np.zeros(a.shape[0], np.uint8)
        _check(_lib.load().rlc_occluded_batch(self.handle, a.shape[0], _dptr(a), _dptr(b),
                                              out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out.astype(bool)

    def intersect(self, origins: np.ndarray, dirs: np.ndarray, t_min: float = 0.0,
                  sah_only: bool = False):
        """intersect() (bvh.hpp:35-36): (t, triangle id), -1 on a miss.  With
        sah_only, the SAH tree's decision alone (-2: deferred to the ordered
        traversal)."""
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        t = np.zeros(o.shape[0], np.float64)
        tri = np.zeros(o.shape[0], np.int32)
        fn = _lib.load().rlc_intersect_batch_sah if sah_only else _lib.load().rlc_intersect_batch
        _check(fn(self.handle, o.shape[0], _dptr(o), _dptr(d),
                                               t_min, _dptr(t),
                                               tri.ctypes.data_as(C.POINTER(C.c_int32))))
        return t, tri

    def synchronize(self):
        _check(_lib.load().rlc_context_synchronize(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rlc_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_context(scene: Scene, config: RenderConfig, device: int = 0) -> RenderContext:
    return RenderContext(scene, config, device)


class HashGrid:
    """HashGrid(hash, init_cut(tree, M, eps)) (proj/src/render.cpp:211-216)."""

    def __init__(self, ctx: RenderContext, config: RenderConfig):
        self.ctx = ctx
        self._cfg = config.c()
        h = C.c_void_p()
        _check(_lib.load().rlc_grid_create(ctx.handle, C.byref(self._cfg), C.byref(h)))
        self.handle = h

    def stats(self) -> dict:
        s = _lib.GridStatsC()
        _check(_lib.load().rlc_grid_stats_get(self.handle, C.byref(s)))
        return {"occupied": s.occupied, "cut_size": s.cut_size, "lookups": s.lookups,
                "fallback_hits": s.fallback_hits}

    def insertion_stats(self) -> dict:
        """Lookups that missed the table at the start of their pass, and the
        distinct keys among them (inserted in canonical order or refused)."""
        s = _lib.GridStatsC()
        _check(_lib.load().rlc_grid_stats_get(self.handle, C.byref(s)))
        return {"pending_lookups": s.pending_lookups, "new_keys": s.new_keys}

    def occupied_count(self) -> int:
        return self.stats()["occupied"]

    def lookup_count(self) -> int:
        return self.stats()["lookups"]

    def fallback_hits(self) -> int:
        return self.stats()["fallback_hits"]

    def export(self) -> dict:
        """Per-cell cut state keyed by CellKey (qx, qy, qz, qn, level)."""
        st = self.stats()
        n, m = st["occupied"], st["cut_size"]
        keys = (_lib.CellKeyC * max(n, 1))()
        node = np.zeros((max(n, 1), m), np.uint32)
        ends = np.zeros_like(node)
        vis = np.zeros_like(node)
        q = np.zeros((max(n, 1), m), np.float64)
        cdf = np.zeros_like(q)
        got = C.c_uint32()
        _check(_lib.load().rlc_grid_export(self.handle, n, keys, _uptr(node), _uptr(ends), _dptr(q),
                                           _dptr(cdf), _uptr(vis), C.byref(got)))
        out = {}
        for i in range(n):
            k = keys[i]
            out[(k.qx, k.qy, k.qz, k.qn, k.level)] = {
                "node_ids": node[i], "ends": ends[i], "q": q[i], "cdf": cdf[i], "visits": vis[i]}
        return out

    def slots(self) -> list:
        """Occupied slots in slot order: (slot, dense cell, CellKey, touched)."""
        lib = _lib.load()
        n = C.c_uint32()
        _check(lib.rlc_grid_slots(self.handle, 0, None, None, None, None, C.byref(n)))
        m = max(n.value, 1)
        slot = np.zeros(m, np.uint32)
        cell = np.zeros(m, np.uint32)
        touched = np.zeros(m, np.uint8)
        keys = (_lib.CellKeyC * m)()
        _check(lib.rlc_grid_slots(self.handle, m, _uptr(slot), _uptr(cell), keys,
                                  touched.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(n)))
        return [(int(slot[i]), int(cell[i]),
                 (keys[i].qx, keys[i].qy, keys[i].qz, keys[i].qn, keys[i].level), bool(touched[i]))
                for i in range(min(n.value, m))]

    def key_of(self, slot: int):
        """HashGrid::key_of (hash_grid.hpp:90): the CellKey in `slot` (None: empty)."""
        for s, _, k, _ in self.slots():
            if s == slot:
                return k
        return None

    def touched_slots(self) -> list:
        """HashGrid::touched_slots (hash_grid.cpp:157-170): ready and touched
        slots in slot order (between render_pass and end_of_pass_update)."""
        return [s for s, _, _, t in self.slots() if t]

    def memory_records(self) -> int:
        """HashGrid::memory_records (hash_grid.cpp:179-187): the sum of cut
        sizes over occupied slots (every cut keeps the template's size)."""
        st = self.stats()
        return st["occupied"] * st["cut_size"]

    def dump_stats(self) -> str:
        """HashGrid::dump_stats (hash_grid.cpp:189-202): CSV header and value
        rows -- occupancy, lookups, fallback hits, per-level occupied counts."""
        st = self.stats()
        hist = [0] * 17
        for _, _, k, _ in self.slots():
            hist[min(k[4], 16)] += 1
        head = "occupied,lookups,fallback_hits" + "".join(f",level_{l}" for l in range(17))
        row = f"{st['occupied']},{st['lookups']},{st['fallback_hits']}" + \
            "".join(f",{h}" for h in hist)
        return head + "\n" + row + "\n"

    def fallback_cut(self) -> dict:
        """HashGrid::fallback_cut: the template cut, sampled on overflow and
        never adapted (hash_grid.cpp:102-111, 136-140)."""
        return self.template()

    def template(self) -> dict:
        m = self.stats()["cut_size"]
        node = np.zeros(m, np.uint32)
        ends = np.zeros(m, np.uint32)
        vis = np.zeros(m, np.uint32)
        q = np.zeros(m, np.float64)
        cdf = np.zeros(m, np.float64)
        eps = C.c_double()
        _check(_lib.load().rlc_grid_template(self.handle, _uptr(node), _uptr(ends), _dptr(q),
                                             _dptr(cdf), _uptr(vis), C.byref(eps)))
        return {"node_ids": node, "ends": ends, "q": q, "cdf": cdf, "visits": vis,
                "eps_q": eps.value}

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rlc_grid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Framebuffer:
    """Framebuffer (proj/include/rlcuts/image.hpp:47-63), device resident."""

    def __init__(self, ctx: RenderContext, width: int | None = None, height: int | None = None):
        self.ctx = ctx
        self.width = int(width if width is not None else ctx.scene.camera.width)
        self.height = int(height if height is not None else ctx.scene.camera.height)
        h = C.c_void_p()
        _check(_lib.load().rlc_framebuffer_create(ctx.handle, self.width, self.height, C.byref(h)))
        self.handle = h

    def download(self) -> tuple[np.ndarray, np.ndarray]:
        s = np.zeros((self.height, self.width, 3), np.float64)
        c = np.zeros((self.height, self.width), np.uint64)
        _check(_lib.load().rlc_framebuffer_download(
            self.handle, _dptr(s), c.ctypes.data_as(C.POINTER(C.c_uint64))))
        return s, c

    def resolve(self) -> np.ndarray:
        img = np.zeros((self.height, self.width, 3), np.float64)
        _check(_lib.load().rlc_framebuffer_resolve(self.handle, _dptr(img)))
        return img

    def clear(self):
        _check(_lib.load().rlc_framebuffer_clear(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rlc_framebuffer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def render_pass(ctx: RenderContext, config: RenderConfig, pass_index: int,
                grid: HashGrid | None, framebuffer: Framebuffer, rows: tuple | None = None,
                sync: bool = True):
    """render_pass (proj/src/render.cpp:159-183)."""
    lib = _lib.load()
    cfg = config.c()
    g = grid.handle if grid is not None else None
    if rows is not None:
        _check(lib.rlc_render_pass_rows(ctx.handle, C.byref(cfg), pass_index, g,
                                        framebuffer.handle, rows[0], rows[1]))
    elif sync:
        _check(lib.rlc_render_pass(ctx.handle, C.byref(cfg), pass_index, g, framebuffer.handle))
    else:
        _check(lib.rlc_render_pass_async(ctx.handle, C.byref(cfg), pass_index, g,
                                         framebuffer.handle))


def render_passes(ctx: RenderContext, config: RenderConfig, first_pass: int, count: int,
                  grid: HashGrid | None, framebuffer: Framebuffer):
    """render_frame's pass loop (proj/src/render.cpp:218-224) for passes
    [first_pass, first_pass + count): render_pass and, with the learned
    sampler, end_of_pass_update per pass, enqueued asynchronously (CUDA-graph
    replays for launch-bound frames).  ctx.synchronize() waits for it."""
    cfg = config.c()
    _check(_lib.load().rlc_render_passes_async(ctx.handle, C.byref(cfg), first_pass, count,
                                               grid.handle if grid is not None else None,
                                               framebuffer.handle))


def end_of_pass_update(grid: HashGrid, ctx: RenderContext, config: CutConfig,
                       sync: bool = True) -> int | None:
    """end_of_pass_update (proj/src/render.cpp:185-200); returns the change count."""
    lib = _lib.load()
    cut = config.c()
    if not sync:
        _check(lib.rlc_end_of_pass_update_async(grid.handle, ctx.handle, C.byref(cut)))
        return None
    ch = C.c_uint32()
    _check(lib.rlc_end_of_pass_update(grid.handle, ctx.handle, C.byref(cut), C.byref(ch)))
    return ch.value


RECORD_DTYPE = np.dtype([("qx", "<i4"), ("qy", "<i4"), ("qz", "<i4"), ("qn", "<u4"),
                         ("level", "<u4"), ("cluster", "<u4"), ("v", "<f8")])  # rlc_update_record


SAMPLE_DTYPE = np.dtype([("vertex", "<u4"), ("cluster", "<u4"), ("emitter", "<u4"),
                         ("flags", "<u4"), ("q_before", "<f8"), ("v", "<f8"), ("total", "<f8"),
                         ("radiance", "<f8", (3,))])  # rlc_sample_record
SAMPLE_VALID, SAMPLE_FALLBACK, SAMPLE_RAY, SAMPLE_NONZERO, SAMPLE_LEARNED = 1, 2, 4, 8, 16
SAMPLE_FROZEN = 32
PDF_LIVE_Q, PDF_FROZEN_CDF = 0, 1


def set_pdf_mode(ctx: RenderContext, mode: int) -> None:
    """rlc_context_set_pdf_mode: PDF_LIVE_Q (the reference's estimator,
    bit-exact) or PDF_FROZEN_CDF (unbiased, non-parity)."""
    _check(_lib.load().rlc_context_set_pdf_mode(ctx.handle, int(mode)))


def enable_sample_export(ctx: RenderContext, enable: bool = True) -> None:
    """File the selected emitter index of every light sample from now on
    (rlc_context_enable_sample_export; needed by pass_samples)."""
    _check(_lib.load().rlc_context_enable_sample_export(ctx.handle, int(bool(enable))))


def pass_samples(ctx: RenderContext, config: RenderConfig, row_begin: int = 0) -> dict:
    """The light samples of the context's last pass in canonical order
    (pixel, sample, depth) -- sample_light's selection (cluster, emitter),
    the live q_before of its pdf, v, the frozen total and the radiance
    (rlc_pass_samples), in the layout of the oracle's OracleRun.samples()."""
    lib = _lib.load()
    n = C.c_uint64()
    _check(lib.rlc_pass_samples(ctx.handle, 0, None, C.byref(n)))
    rec = np.zeros(n.value, SAMPLE_DTYPE)
    if n.value:
        _check(lib.rlc_pass_samples(ctx.handle, n.value, rec.ctypes.data_as(C.c_void_p),
                                    C.byref(n)))
    rec = rec[(rec["flags"] & SAMPLE_VALID) != 0]
    per_pixel = (config.spp // config.passes) * max(config.max_depth, 1)
    pixel = (rec["vertex"] // per_pixel + row_begin * ctx.scene.camera.width).astype(np.uint32)
    return {"pixel": pixel, "cluster": rec["cluster"], "emitter": rec["emitter"],
            "fallback": (rec["flags"] & SAMPLE_FALLBACK) != 0, "q_before": rec["q_before"],
            "v": rec["v"], "radiance": rec["radiance"], "total": rec["total"],
            "ray": (rec["flags"] & SAMPLE_RAY) != 0, "nonzero": (rec["flags"] & SAMPLE_NONZERO) != 0,
            "learned": (rec["flags"] & SAMPLE_LEARNED) != 0,
            "frozen": (rec["flags"] & SAMPLE_FROZEN) != 0}


def shard_trace(ctx: RenderContext, config: RenderConfig, pass_index: int, grid: HashGrid,
                rows: tuple, cap_records: int) -> tuple[int, int]:
    """rlc_shard_trace: trace a band and file its update records into the
    context's record block.  Returns (device pointer, bytes) of the block."""
    cfg = config.c()
    ptr = C.c_void_p()
    n = C.c_uint64()
    _check(_lib.load().rlc_shard_trace(ctx.handle, C.byref(cfg), pass_index, grid.handle,
                                       rows[0], rows[1], cap_records, C.byref(ptr), C.byref(n)))
    return int(ptr.value or 0), int(n.value)


def shard_trace_to(ctx: RenderContext, config: RenderConfig, pass_index: int, grid: HashGrid,
                   rows: tuple, cap_records: int, rank: int, dst_ptrs: list) -> None:
    """rlc_shard_trace_to: the band's records stored straight into every
    destination buffer (device pointers) at block `rank`."""
    cfg = config.c()
    arr = (C.c_void_p * len(dst_ptrs))(*dst_ptrs)
    _check(_lib.load().rlc_shard_trace_to(ctx.handle, C.byref(cfg), pass_index, grid.handle,
                                          rows[0], rows[1], cap_records, rank, arr, len(dst_ptrs)))


def shard_fold(ctx: RenderContext, config: RenderConfig, grid: HashGrid, blocks_ptr: int,
               nranks: int, rank: int, owner_fold: bool) -> tuple[int, int, int]:
    """rlc_shard_fold over the all-gathered blocks (device memory, rank-major,
    valid until shard_finish).  Returns (q_before doubles, entry-count
    uint32s, count): the device arrays per exchange slot that owner mode
    sums over the ranks."""
    cfg = config.c()
    ptr = C.c_void_p()
    seg = C.c_void_p()
    n = C.c_uint64()
    _check(_lib.load().rlc_shard_fold(ctx.handle, C.byref(cfg), grid.handle, C.c_void_p(blocks_ptr),
                                      nranks, rank, int(owner_fold), C.byref(ptr), C.byref(seg),
                                      C.byref(n)))
    return int(ptr.value or 0), int(seg.value or 0), int(n.value)


def shard_entry_arrays(ctx: RenderContext) -> tuple[int, int, int]:
    """rlc_shard_entry_arrays: (final-q doubles, count uint32s, entries) of
    owner mode's entry exchange after shard_fold; (0, 0, 0) in per-slot mode."""
    q = C.c_void_p()
    n = C.c_void_p()
    cnt = C.c_uint64()
    _check(_lib.load().rlc_shard_entry_arrays(ctx.handle, C.byref(q), C.byref(n), C.byref(cnt)))
    return int(q.value or 0), int(n.value or 0), int(cnt.value)


def shard_finish(ctx: RenderContext, grid: HashGrid, framebuffer: Framebuffer, rank: int,
                 owner_fold: bool):
    _check(_lib.load().rlc_shard_finish(ctx.handle, grid.handle, framebuffer.handle, rank,
                                        int(owner_fold)))


def shard_sync(ctx: RenderContext, grid: HashGrid):
    _check(_lib.load().rlc_shard_sync(ctx.handle, grid.handle))


class Comm:
    """NCCL communicator of one rank (rlc_comm_*); rank 0's unique id is
    shared by the caller (e.g. torch.distributed.broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(_lib.load().rlc_comm_unique_id(buf))
        return bytes(buf)

    def enable_peer_exchange(self, cap_records: int, enable: bool = True):
        """Collective: rlc_shard_frame moves records by peer memory (CUDA IPC)
        instead of ncclAllGather."""
        _check(_lib.load().rlc_comm_enable_peer_exchange(self.handle, cap_records, int(enable)))

    def __init__(self, device: int, nranks: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(_lib.load().rlc_comm_create(device, nranks, rank, buf, C.byref(h)))
        self.handle, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().rlc_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_frame(ctx: RenderContext, config: RenderConfig, pass_index: int, grid: HashGrid,
                framebuffer: Framebuffer, comm: Comm, rows: tuple, cap_records: int,
                owner_fold: bool = True):
    """rlc_shard_frame: this rank's band of one frame with the exchange over
    NCCL, enqueued without a host synchronization."""
    cfg = config.c()
    _check(_lib.load().rlc_shard_frame(ctx.handle, C.byref(cfg), pass_index, grid.handle,
                                       framebuffer.handle, comm.handle, rows[0], rows[1],
                                       cap_records, int(owner_fold)))


def shard_frames(ctx: RenderContext, config: RenderConfig, first_pass: int, count: int,
                 grid: HashGrid, framebuffer: Framebuffer, comm: Comm, rows: tuple,
                 cap_records: int, owner_fold: bool = True, graph: bool = True):
    """rlc_shard_frames: `count` frames of shard_frame, replayed from a CUDA
    graph of two frames (kernels and NCCL collectives) when `graph`."""
    cfg = config.c()
    _check(_lib.load().rlc_shard_frames(ctx.handle, C.byref(cfg), first_pass, count, grid.handle,
                                        framebuffer.handle, comm.handle, rows[0], rows[1],
                                        cap_records, int(owner_fold), int(graph)))


@dataclass
class RenderResult:  # render.hpp:56-64
    image: np.ndarray
    wall_ms: float
    occupied_cells: int
    lookups: int
    fallback_hits: int
    sc_changes: list
    pass_mse: list = field(default_factory=list)  # vs the reference image; empty without one


def render_frame(ctx: RenderContext, config: RenderConfig,
                 reference: np.ndarray | None = None) -> RenderResult:
    """render_frame (proj/src/render.cpp:202-240); with `reference` (h x w x 3
    linear RGB) the accumulated image is scored after every pass."""
    cam = ctx.scene.camera
    img = np.zeros((cam.height, cam.width, 3), np.float64)
    changes = (C.c_uint32 * max(config.passes, 1))()
    res = _lib.RenderResultC()
    res.sc_changes = C.cast(changes, C.POINTER(C.c_uint32))
    cfg = config.c()
    if reference is None:
        _check(_lib.load().rlc_render_frame(ctx.handle, C.byref(cfg), _dptr(img), C.byref(res)))
        pm = []
    else:
        ref = np.ascontiguousarray(reference, np.float64)
        if ref.ndim != 3 or ref.shape[2] != 3:
            raise ValueError("mse: image dimensions disagree")
        out = np.zeros(max(config.passes, 1))
        _check(_lib.load().rlc_render_frame_scored(ctx.handle, C.byref(cfg), _dptr(ref),
                                                   ref.shape[1], ref.shape[0], _dptr(img),
                                                   C.byref(res), _dptr(out)))
        pm = out[:config.passes].tolist()
    return RenderResult(img, res.wall_ms, res.occupied_cells, res.lookups, res.fallback_hits,
                        list(changes)[:config.passes], pm)


# ---- image module (proj/include/rlcuts/image.hpp:65-78) -------------------
def _img(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float64)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError("image must be h x w x 3")
    return a


def write_pfm(image: np.ndarray, path: str) -> None:
    """write_pfm (image.cpp:43-60): float32 RGB, little-endian, bottom row first."""
    im = _img(image)
    _check(_lib.load().rlc_image_write_pfm(_dptr(im), im.shape[1], im.shape[0],
                                           str(path).encode()))


def read_pfm(path: str) -> np.ndarray:
    """read_pfm (image.cpp:62-94)."""
    w, h = C.c_int32(), C.c_int32()
    lib = _lib.load()
    _check(lib.rlc_image_read_pfm(str(path).encode(), None, 0, C.byref(w), C.byref(h)))
    img = np.zeros((h.value, w.value, 3), np.float64)
    _check(lib.rlc_image_read_pfm(str(path).encode(), _dptr(img), img.shape[0] * img.shape[1],
                                  C.byref(w), C.byref(h)))
    return img


def write_ppm(image: np.ndarray, path: str) -> None:
    """write_ppm (image.cpp:96-112): 8-bit gamma-2.2 preview."""
    im = _img(image)
    _check(_lib.load().rlc_image_write_ppm(_dptr(im), im.shape[1], im.shape[0],
                                           str(path).encode()))


def mse(a: np.ndarray, b: np.ndarray) -> float:
    """mse (image.cpp:114-124), the reference's sequential sum."""
    a, b = _img(a), _img(b)
    out = C.c_double()
    _check(_lib.load().rlc_image_mse(_dptr(a), a.shape[1], a.shape[0], _dptr(b), b.shape[1],
                                     b.shape[0], C.byref(out)))
    return out.value


def relative_mse(a: np.ndarray, b: np.ndarray) -> float:
    """relative_mse (image.cpp:126-136); b is the reference."""
    a, b = _img(a), _img(b)
    out = C.c_double()
    _check(_lib.load().rlc_image_relative_mse(_dptr(a), a.shape[1], a.shape[0], _dptr(b),
                                              b.shape[1], b.shape[0], C.byref(out)))
    return out.value


# ---- the stats CSV of the reference CLI (tools/main.cpp:224-258) ----------
STATS_HEADER = (
    "scene,sampler,spp,passes,width,height,seed,depth,workers,cut_size,alpha,"
    "threshold_T,eps_q,iterations,base_tile,capacity,probe_limit,normal_bits,"
    "jitter_scale,alpha_schedule,wall_ms,mse,relative_mse,pass_mse_series,"
    "sc_changes_per_pass,occupied_cells,lookups,fallback_hits,fallback_rate,error")

_SAMPLER_NAMES = {0: "uniform", 1: "energy", 2: "rl"}


def _g(v: float, prec: int = 6) -> str:
    """std::ostream << double at precision `prec` (%g-style, no trailing zeros)."""
    return f"{v:.{prec}g}"


def csv_escape(field_: str) -> str:
    if not any(c in field_ for c in ',"\n\r'):
        return field_
    return '"' + field_.replace('"', '""') + '"'


def stats_row(scene_id: str, config: RenderConfig, width: int, height: int, base_tile: float,
              result: RenderResult | None = None, error_mse: float | None = None,
              error_rel: float | None = None, error_message: str = "") -> str:
    """write_stats_row (tools/main.cpp:230-258): one CSV row, newline-terminated.
    `config` carries the CLI flags (RenderConfig fields); `base_tile` is the
    resolved one (RenderContext.base_tile)."""
    c = config
    schedule = "harmonic" if int(c.cut.alpha_schedule) == 1 else "fixed"
    parts = [csv_escape(scene_id), _SAMPLER_NAMES[int(c.sampler)], str(c.spp), str(c.passes),
             str(width), str(height), str(c.seed), str(c.max_depth), str(c.workers),
             str(c.cut.cut_size), _g(c.cut.alpha), _g(c.cut.split_threshold), _g(c.cut.eps_q),
             str(c.cut.iterations), _g(base_tile), str(c.hash.capacity), str(c.hash.probe_limit),
             str(c.hash.normal_bits), _g(c.hash.jitter_scale), schedule]
    if result is not None:
        rate = result.fallback_hits / result.lookups if result.lookups > 0 else 0.0
        parts += [_g(result.wall_ms, 17),
                  _g(error_mse, 17) if error_mse is not None else "",
                  _g(error_rel, 17) if error_rel is not None else "",
                  csv_escape(";".join(_g(v, 17) for v in result.pass_mse)),
                  csv_escape(";".join(str(v) for v in result.sc_changes)),
                  str(result.occupied_cells), str(result.lookups), str(result.fallback_hits),
                  _g(rate, 17)]
    else:
        parts += [""] * 9
    parts.append(csv_escape(error_message))
    return ",".join(parts) + "\n"


def libm_variant() -> int:
    """Host libm build the bounce sampler restates: 1 glibc FMA, 0 SSE2, -1 unknown."""
    v = C.c_int32()
    _check(_lib.load().rlc_libm_variant(C.byref(v)))
    return v.value


def libm_sincos_host(x: np.ndarray, variant: int):
    """Host run of the restated libm sin/cos (no device needed)."""
    x = np.ascontiguousarray(x, np.float64).ravel()
    s, c = np.empty_like(x), np.empty_like(x)
    _check(_lib.load().rlc_libm_sincos_host(variant, x.size, _dptr(x), _dptr(s), _dptr(c)))
    return s, c


def kernel_launches() -> int:
    return int(_lib.load().rlc_kernel_launches())


def work_counters(reset: bool = True) -> dict:
    """k_shadow's own work since the last reset (rlc_work_counters): rays
    traversed by its tree, node steps, triangle tests."""
    out = np.zeros(4, np.uint64)
    _check(_lib.load().rlc_work_counters(1 if reset else 0,
                                         out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return {"shadow_rays": int(out[0]), "shadow_nodes": int(out[1]), "shadow_tris": int(out[2]),
            "shadow_rays_queued": int(out[3])}


def measure_l2_bandwidth(device: int = 0) -> float:
    """Measured L2 read bandwidth of the device, GB/s (rlc_measure_l2_bandwidth)."""
    out = C.c_double()
    _check(_lib.load().rlc_measure_l2_bandwidth(device, C.byref(out)))
    return out.value


def trav_stats(reset: bool = True) -> dict:
    """Traversal counters of a -DRLC_TRAV_STATS build (zeros otherwise)."""
    out = (C.c_uint64 * 8)()
    _check(_lib.load().rlc_debug_trav_stats(1 if reset else 0, out))
    v = list(out)
    return {"shadow_rays": v[0], "shadow_nodes": v[1], "shadow_tris": v[2],
            "closest_rays": v[3], "closest_nodes": v[4], "closest_tris": v[5],
            "shadow_overflows": v[6], "closest_deferred": v[7]}
