"""Adversarial near-grazing visibility ("assumption shared
with item 3"): segments and rays built in or near the planes of scene
triangles -- in-plane, or tilted by 1e-12 to 1e-6 rad, through points just
inside and just outside the edges, from origins up to ~1e3 scene extents
away, in scenes offset by up to 3e7 -- where Moller-Trumbore's fp64 t is
least accurate relative to the conservative fp32 tree boxes.  rlc_occluded_batch
and rlc_intersect_batch must equal the reference's occluded / intersect
(proj/src/bvh.cpp:124-188) bit for bit: 1.2e7 segments and 3e6 rays."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes
from paper_1911_10217_b200.scenes import Scene

pytestmark = pytest.mark.gpu


def soup(count, seed, extent, offset):
    rng = np.random.default_rng(seed)
    base = rng.uniform(0, extent, (count, 1, 3))
    size = np.exp(rng.uniform(np.log(0.05), np.log(2.0), (count, 1, 1)))
    v = base + size * rng.uniform(-0.5, 0.5, (count, 3, 3)) + offset
    mats = np.array([[0.5, 0.5, 0.5, 0, 0, 0], [0, 0, 0, 1, 1, 1]], float)
    c = (offset, offset, offset - 5)
    return Scene(v, (np.arange(count) % 2).astype(np.uint32), mats,
                 scenes.Camera(c, (offset,) * 3, (0, 1, 0), 45, 8, 8), "grazing_soup")


def grazing(scene, n, seed):
    """n segments (a, b) and directions grazing random scene triangles."""
    rng = np.random.default_rng(seed)
    v = scene.vertices
    t = rng.integers(0, len(v), n)
    p0, e1, e2 = v[t, 0], v[t, 1] - v[t, 0], v[t, 2] - v[t, 0]
    nrm = np.cross(e1, e2)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    u = e1 / np.linalg.norm(e1, axis=1, keepdims=True)
    w = np.cross(nrm, u)
    # a point of the plane just inside or outside the triangle's edges
    ab = rng.uniform(-0.15, 1.15, (n, 2))
    q = p0 + ab[:, :1] * e1 + ab[:, 1:] * e2
    # tilt out of the plane: exactly 0 for a quarter, else 1e-12 .. 1e-6 rad
    tilt = np.exp(rng.uniform(np.log(1e-12), np.log(1e-6), n)) * rng.choice([-1.0, 1.0], n)
    tilt[rng.random(n) < 0.25] = 0.0
    phi = rng.uniform(0, 2 * np.pi, n)
    d = (np.cos(tilt)[:, None] * (np.cos(phi)[:, None] * u + np.sin(phi)[:, None] * w)
         + np.sin(tilt)[:, None] * nrm)
    # and a hair off the plane along the normal
    q = q + nrm * (rng.uniform(-1e-9, 1e-9, n) * np.abs(q).max(axis=1))[:, None]
    s1 = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), n))
    s2 = np.exp(rng.uniform(np.log(1e-3), np.log(10.0), n))
    return q - s1[:, None] * d, q + s2[:, None] * d, d


@pytest.mark.parametrize("offset", [0.0, 1e3, 3e7])
def test_occluded_near_grazing(ref, offset):
    scene = soup(3000, 5, 8.0, offset)
    cfg = rlcuts.RenderConfig()
    ctx, rr = rlcuts.build_context(scene, cfg), ref.RefRun(scene, cfg)
    hits = 0
    for chunk in range(4):
        a, b, _ = grazing(scene, 1_000_000, 100 + chunk)
        got, want = ctx.occluded(a, b), rr.occluded(a, b)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, f"{bad.size} segments differ, first {bad[:5]}"
        hits += int(want.sum())
    assert 0.05 * 4e6 < hits < 0.95 * 4e6


@pytest.mark.parametrize("offset", [0.0, 1e3, 3e7])
def test_intersect_near_grazing(ref, offset):
    scene = soup(3000, 6, 8.0, offset)
    cfg = rlcuts.RenderConfig()
    ctx, rr = rlcuts.build_context(scene, cfg), ref.RefRun(scene, cfg)
    a, _, d = grazing(scene, 1_000_000, 7)
    t, tri = ctx.intersect(a, d)
    rt, rtri = rr.intersect(a, d)
    assert np.array_equal(tri, rtri), f"{np.count_nonzero(tri != rtri)} triangle ids differ"
    assert np.array_equal(t, rt)
    assert (tri >= 0).mean() > 0.2
