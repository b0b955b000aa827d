"""Synthetic scenes for the BASELINE.json configurations.

Scenes are plain float64 arrays in the layout of ``rlcuts::Scene``
(proj/include/rlcuts/scene.hpp:53-67): the CUDA path and the reference
oracle consume the byte-identical object.  Generators are restatements of
the reference's fixtures (proj/src/scene_gen.cpp:27-147) plus the maze the
survey defines for C3/C4/C5; they are scene *inputs*, not part of the path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """splitmix64 finalizer, proj/include/rlcuts/rng.hpp:12-17."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


class RandomSequence:
    """Counter RNG, proj/include/rlcuts/rng.hpp:26-43 (scalar, for fixtures)."""

    def __init__(self, seed: int, a: int, b: int = 0, c: int = 0):
        k = mix64(seed)
        for v in (a, b, c):
            k = mix64(k ^ mix64(v))
        self.key = k
        self.dim = 0

    def next(self) -> float:
        self.dim += 1
        bits = mix64((self.key + 0x9E3779B97F4A7C15 * self.dim) & M64)
        return float(bits >> 11) * 2.0 ** -53


@dataclass
class Camera:
    origin: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    vfov_degrees: float = 45.0
    width: int = 128
    height: int = 128


@dataclass
class Scene:
    vertices: np.ndarray      # (n, 3, 3) float64: p0, p1, p2
    material_ids: np.ndarray  # (n,) uint32
    materials: np.ndarray     # (m, 6) float64: albedo rgb, emission rgb
    camera: Camera = field(default_factory=Camera)
    name: str = "scene"

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).reshape(-1, 3, 3)
        self.material_ids = np.ascontiguousarray(self.material_ids, dtype=np.uint32)
        self.materials = np.ascontiguousarray(self.materials, dtype=np.float64).reshape(-1, 6)

    @property
    def num_triangles(self) -> int:
        return int(self.vertices.shape[0])

    def emitter_ids(self) -> np.ndarray:
        """derive_emitters (proj/src/scene.cpp:33-37)."""
        e = self.materials[:, 3:6]
        lum = 0.2126 * e[:, 0] + 0.7152 * e[:, 1] + 0.0722 * e[:, 2]
        return np.nonzero(lum[self.material_ids] > 0)[0].astype(np.uint32)

    def with_resolution(self, width: int, height: int) -> "Scene":
        cam = Camera(self.camera.origin, self.camera.look_at, self.camera.up,
                     self.camera.vfov_degrees, int(width), int(height))
        return Scene(self.vertices, self.material_ids, self.materials, cam, self.name)

    def desc(self) -> "_lib.SceneDescC":
        """rlc_scene_desc view; the arrays stay owned by this Scene."""
        d = _lib.SceneDescC()
        d.num_triangles = self.num_triangles
        d.num_materials = int(self.materials.shape[0])
        d.vertices = self.vertices.ctypes.data_as(C.POINTER(C.c_double))
        d.material_ids = self.material_ids.ctypes.data_as(C.POINTER(C.c_uint32))
        d.materials = self.materials.ctypes.data_as(C.POINTER(C.c_double))
        for i in range(3):
            d.cam_origin[i] = float(self.camera.origin[i])
            d.cam_look_at[i] = float(self.camera.look_at[i])
            d.cam_up[i] = float(self.camera.up[i])
        d.vfov_degrees = float(self.camera.vfov_degrees)
        d.width = int(self.camera.width)
        d.height = int(self.camera.height)
        return d


class _Builder:
    def __init__(self):
        self.tris: list[np.ndarray] = []
        self.mats: list[np.ndarray] = []
        self.materials: list[list[float]] = []

    def material(self, albedo, emission) -> int:
        self.materials.append([*albedo, *emission])
        return len(self.materials) - 1

    def quad(self, a, b, c, d, mat):
        """add_quad, proj/src/scene_gen.cpp:15-19: (a,b,c) and (a,c,d)."""
        a, b, c, d = (np.asarray(v, dtype=np.float64) for v in (a, b, c, d))
        self.tris.append(np.stack([np.stack([a, b, c]), np.stack([a, c, d])]))
        self.mats.append(np.array([mat, mat], dtype=np.uint32))

    def tessellated_quad(self, a, b, c, d, mat, nu: int, nv: int):
        """Quad (a,b,c,d) split into nu x nv sub-quads, same winding."""
        a, b, c, d = (np.asarray(v, dtype=np.float64) for v in (a, b, c, d))
        us = np.arange(nu + 1) / nu
        vs = np.arange(nv + 1) / nv

        def at(u, v):  # bilinear over (a, b, c, d)
            return ((1 - u) * (1 - v))[..., None] * a + (u * (1 - v))[..., None] * b + \
                   (u * v)[..., None] * c + ((1 - u) * v)[..., None] * d
        U, V = np.meshgrid(us, vs, indexing="ij")
        P = at(U, V)  # (nu+1, nv+1, 3)
        qa, qb, qc, qd = P[:-1, :-1], P[1:, :-1], P[1:, 1:], P[:-1, 1:]
        t1 = np.stack([qa, qb, qc], axis=-2).reshape(-1, 3, 3)
        t2 = np.stack([qa, qc, qd], axis=-2).reshape(-1, 3, 3)
        tris = np.stack([t1, t2], axis=1).reshape(-1, 3, 3)
        self.tris.append(tris)
        self.mats.append(np.full(tris.shape[0], mat, dtype=np.uint32))

    def add(self, tris: np.ndarray, mats: np.ndarray):
        self.tris.append(np.asarray(tris, dtype=np.float64).reshape(-1, 3, 3))
        self.mats.append(np.asarray(mats, dtype=np.uint32).reshape(-1))

    def scene(self, camera: Camera, name: str) -> Scene:
        return Scene(np.concatenate([t.reshape(-1, 3, 3) for t in self.tris]),
                     np.concatenate(self.mats), np.array(self.materials, dtype=np.float64),
                     camera, name)


def _normalize(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _dome(center, radius, requested):
    """append_dome, proj/src/scene_gen.cpp:27-76 (inward-facing shell)."""
    subdiv = min(range(8), key=lambda s: abs(8.0 * 4.0 ** s - requested))
    top = np.array([0.0, 1.0, 0.0])
    eq = [np.array(v, dtype=np.float64) for v in
          ([1, 0, 0], [0, 0, 1], [-1, 0, 0], [0, 0, -1], [1, 0, 0])]
    tris = []
    for i in range(4):
        mid = _normalize(eq[i] + eq[i + 1])
        tris.append((top, eq[i], mid))
        tris.append((top, mid, eq[i + 1]))
    T = np.array([np.stack(t) for t in tris])
    for _ in range(subdiv):
        a, b, c = T[:, 0], T[:, 1], T[:, 2]
        ab, bc, ca = _normalize(a + b), _normalize(b + c), _normalize(c + a)
        T = np.stack([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                      np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3, 3)
    center = np.asarray(center, dtype=np.float64)
    W = center + T * radius
    n = np.cross(W[:, 1] - W[:, 0], W[:, 2] - W[:, 0])
    out = (np.einsum("ij,ij->i", n, W.mean(axis=1) - center) > 0)
    W[out, 1], W[out, 2] = W[out, 2].copy(), W[out, 1].copy()
    return W


def cornell_grid(k: int, seed: int = 1, dome_triangles: int = 512, *, light_tess=None,
                 dome: bool = True, width: int = 128, height: int = 128) -> Scene:
    """k x k open-top Cornell boxes, each with its own area light
    (gen_cornell_grid, proj/src/scene_gen.cpp:78-147).  ``light_tess=(nu, nv)``
    tessellates each light into nu*nv*2 emissive triangles;
    ``dome=False`` drops the sky dome."""
    if k < 1:
        raise ValueError("gen_cornell_grid: k must be >= 1")
    b = _Builder()
    b.material((0.73, 0.73, 0.73), (0, 0, 0))
    b.material((0.62, 0.06, 0.06), (0, 0, 0))
    b.material((0.11, 0.45, 0.09), (0, 0, 0))
    pitch = 1.25
    extent = pitch * k - 0.25
    for iz in range(k):
        for ix in range(k):
            o = np.array([pitch * ix, 0.0, pitch * iz])
            rng = RandomSequence(seed, iz * k + ix)
            emission = (11.0 + 5.0 * rng.next(), 10.0 + 4.0 * rng.next(), 7.0 + 3.0 * rng.next())
            light = b.material((0, 0, 0), emission)
            P = lambda x, y, z: o + np.array([x, y, z], dtype=np.float64)  # noqa: E731
            b.quad(P(0, 0, 0), P(1, 0, 0), P(1, 0, 1), P(0, 0, 1), 0)  # floor
            b.quad(P(0, 0, 0), P(0, 0, 1), P(0, 1, 1), P(0, 1, 0), 1)  # left, red
            b.quad(P(1, 0, 0), P(1, 1, 0), P(1, 1, 1), P(1, 0, 1), 2)  # right, green
            b.quad(P(0, 0, 1), P(1, 0, 1), P(1, 1, 1), P(0, 1, 1), 0)  # back
            b.quad(P(0, 0, 0), P(0, 1, 0), P(1, 1, 0), P(1, 0, 0), 0)  # front
            la, lb, lc, ld = P(.3, .93, .3), P(.7, .93, .3), P(.7, .93, .7), P(.3, .93, .7)
            if light_tess is None:
                b.quad(la, lb, lc, ld, light)
            else:
                b.tessellated_quad(la, lb, lc, ld, light, *light_tess)
    origin = (extent * 0.5, 2.6 * extent + 2.0, -(0.55 * extent + 0.6))
    look = (extent * 0.5, 0.0, extent * 0.45)
    dist = math.dist(origin, look)
    half_span = 0.52 * extent + 0.1
    cam = Camera(origin, look, (0.0, 0.0, 1.0),
                 2.0 * math.atan2(half_span, dist) * 180.0 / math.pi, width, height)
    gc = np.array([extent * 0.5, 0.0, extent * 0.5])
    radius = max(6.0, 3.0 * extent, 1.3 * math.dist(origin, tuple(gc)))
    hg = 0.95 * radius
    b.quad(gc + [-hg, -1e-3, -hg], gc + [hg, -1e-3, -hg], gc + [hg, -1e-3, hg],
           gc + [-hg, -1e-3, hg], 0)
    if dome:
        dm = b.material((0, 0, 0), (0.035, 0.0425, 0.055))
        W = _dome(gc, radius, dome_triangles)
        b.add(W, np.full(W.shape[0], dm))
    return b.scene(cam, f"cornell_grid_k{k}")


def maze(n_emitters: int = 1_000_000, n_walls: int = 400, seed: int = 5, *,
         width: int = 1920, height: int = 1080) -> Scene:
    """Procedural maze lit by many small ceiling emitters:
    floor [-1,11]^2; ``n_walls`` diffuse wall panels of height 1 on randomly
    chosen edges of a 24 x 24 grid of 0.5 m cells; ``n_emitters`` randomly
    jittered, randomly sized, downward-facing emissive triangles just below
    y = 4 with 16 emission levels; camera (5,3.8,-1) -> (5,0,5), vfov 60."""
    rng = np.random.default_rng(seed)
    b = _Builder()
    floor = b.material((0.6, 0.6, 0.6), (0, 0, 0))
    wall = b.material((0.7, 0.7, 0.7), (0, 0, 0))
    b.quad((-1, 0, -1), (-1, 0, 11), (11, 0, 11), (11, 0, -1), floor)
    g, pitch, h = 24, 0.5, 1.0
    edges = [(i, j, 0) for i in range(g) for j in range(g + 1)] + \
            [(i, j, 1) for i in range(g + 1) for j in range(g)]
    pick = rng.choice(len(edges), size=min(n_walls, len(edges)), replace=False)
    E = np.array([edges[k] for k in np.sort(pick)], dtype=np.float64).reshape(-1, 3)
    along_x = E[:, 2] == 0
    x0 = -1.0 + np.where(along_x, E[:, 0], E[:, 0]) * pitch
    z0 = -1.0 + np.where(along_x, E[:, 1], E[:, 1]) * pitch
    x1 = x0 + np.where(along_x, pitch, 0.0)
    z1 = z0 + np.where(along_x, 0.0, pitch)
    nw = E.shape[0]
    A = np.stack([x0, np.zeros(nw), z0], 1)
    B = np.stack([x1, np.zeros(nw), z1], 1)
    Cc = np.stack([x1, np.full(nw, h), z1], 1)
    D = np.stack([x0, np.full(nw, h), z0], 1)
    walls = np.stack([np.stack([A, B, Cc], 1), np.stack([A, Cc, D], 1)], 1).reshape(-1, 3, 3)
    b.add(walls, np.full(walls.shape[0], wall))
    levels = 16
    first = len(b.materials)
    for i in range(levels):
        s = 1.0 + i / (levels - 1)  # emission 2 .. 4
        b.material((0, 0, 0), (2.0 * s, 2.0 * s, 2.0 * s))
    g = int(math.ceil(math.sqrt(n_emitters)))
    cell = 12.0 / g
    idx = np.arange(n_emitters)
    cx = -1.0 + (idx % g + rng.uniform(0.15, 0.85, n_emitters)) * cell
    cz = -1.0 + (idx // g + rng.uniform(0.15, 0.85, n_emitters)) * cell
    cy = 4.0 - rng.uniform(0.0, 0.01, n_emitters)
    size = cell * rng.uniform(0.2, 0.6, n_emitters)
    a = np.stack([cx - size / 2, cy, cz - size / 2], 1)
    p1 = a + np.stack([size, np.zeros_like(size), np.zeros_like(size)], 1)
    p2 = a + np.stack([np.zeros_like(size), np.zeros_like(size), size], 1)
    em = np.stack([a, p1, p2], 1)  # (a, a+x, a+z): normal -y, faces the floor
    b.add(em, first + rng.integers(0, levels, n_emitters))
    cam = Camera((5.0, 3.8, -1.0), (5.0, 0.0, 5.0), (0.0, 1.0, 0.0), 60.0, width, height)
    return b.scene(cam, f"maze_{n_emitters}")


def _mix64_np(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def displace_emitters(scene: Scene, frame: int, seed: int = 7, amplitude: float = 0.02) -> Scene:
    """C4's moving emitters: every emissive triangle of `scene`
    translated in x and z by amplitude * (u - 1/2), u a counter hash of
    (seed, frame, emitter index, axis); frame 0 is the scene itself.  Same
    triangle order, materials and camera, so the result is a valid
    rlc_context_update_scene input."""
    if frame == 0:
        return scene
    emissive = (scene.materials[:, 3:] @ np.array([0.2126, 0.7152, 0.0722])) > 0
    idx = np.nonzero(emissive[scene.material_ids])[0]
    v = scene.vertices.copy()
    with np.errstate(over="ignore"):
        base = _mix64_np(np.array([seed], np.uint64))[0] ^ _mix64_np(np.array([frame], np.uint64))[0]
        key = _mix64_np(np.uint64(base) ^ _mix64_np(np.arange(len(idx), dtype=np.uint64)))
        ux = (_mix64_np(key ^ np.uint64(1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        uz = (_mix64_np(key ^ np.uint64(2)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    v[idx, :, 0] += (amplitude * (ux - 0.5))[:, None]
    v[idx, :, 2] += (amplitude * (uz - 0.5))[:, None]
    return Scene(v, scene.material_ids, scene.materials, scene.camera, f"{scene.name}_f{frame}")


# ---- BASELINE.json configurations ---------------------------

def config_scene(name: str) -> tuple[Scene, dict]:
    """Scene plus render settings of a named configuration.

    c1: 1 Cornell box, light -> 1,024 tris, 256^2, 16 spp / 16 passes, base_tile 1/16
    c2: 4x4 boxes, 16 lights x 1,024 tris, 1280x720, 64 spp / 16 passes
    c3: maze with 1M emitters, 1920x1080, 64 spp / 64 passes (1 spp per frame)
    c4: maze with 64K emitters, 1920x1080, 1 spp per frame
    c5: maze with 4M emitters, 3840x2160, 64 spp / 16 passes
    """
    if name == "c1":
        s = cornell_grid(1, 1, light_tess=(16, 32), dome=False, width=256, height=256)
        return s, dict(spp=16, passes=16, base_tile=1.0 / 16.0)
    if name == "c2":
        s = cornell_grid(4, 1, light_tess=(16, 32), dome=False, width=1280, height=720)
        return s, dict(spp=64, passes=16, base_tile=0.0)
    if name == "c3":
        return maze(1_000_000), dict(spp=64, passes=64, base_tile=0.0)
    if name == "c4":
        return maze(65_536, seed=7), dict(spp=64, passes=64, base_tile=0.0)
    if name == "c5":
        return maze(4_000_000, seed=11, width=3840, height=2160), dict(spp=64, passes=16,
                                                                        base_tile=0.0)
    raise KeyError(name)
