"""GPU visibility kernels against the reference's own BVH queries
(proj/src/bvh.cpp:124-188), mirroring tests/test_scene.cpp:181-231 of the
reference: random triangle soups plus axis-aligned grazing segments.  The
shadow kernel traverses a conservative fp32 4-wide tree and accepts hits only
after the exact fp64 ancestor check, so its booleans must equal the
reference's bit for bit; closest hits must agree in triangle id and exact t."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes
from paper_1911_10217_b200.scenes import RandomSequence, Scene

pytestmark = pytest.mark.gpu


def random_soup(count, seed, extent, tri_size):
    """test_scene.cpp:58-73: random triangles, every other one emissive."""
    rng = RandomSequence(seed, 0)
    v = np.zeros((count, 3, 3))
    for i in range(count):
        base = np.array([extent * rng.next() for _ in range(3)])
        e1 = np.array([tri_size * (rng.next() - 0.5) for _ in range(3)])
        e2 = np.array([tri_size * (rng.next() - 0.5) for _ in range(3)])
        v[i] = [base, base + e1, base + e2]
    mats = np.array([[0.5, 0.5, 0.5, 0, 0, 0], [0, 0, 0, 1, 1, 1]], float)
    return Scene(v, (np.arange(count) % 2).astype(np.uint32), mats,
                 scenes.Camera((0, 0, -5), (0, 0, 0), (0, 1, 0), 45, 8, 8), "soup")


@pytest.fixture(params=["tris", "tris-128B", "leaves", "reference"], autouse=True)
def shadow_tree(request, monkeypatch):
    """All shadow-ray trees: the SAH tree over single triangles (default,
    64-byte quantized nodes; "-128B": the unquantized nodes), the SAH tree over
    the reference leaves, and the reference tree collapsed to 4-wide."""
    tree, _, variant = request.param.partition("-")
    monkeypatch.setenv("RLC_SHADOW_TREE", tree)
    monkeypatch.setenv("RLC_SHADOW_QUANT", "0" if variant == "128B" else "1")
    return request.param


def both(ref, scene):
    cfg = rlcuts.RenderConfig()
    return rlcuts.build_context(scene, cfg), ref.RefRun(scene, cfg)


def test_occluded_random_soup(ref):
    scene = random_soup(2000, 13, 6.0, 0.6)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(78)
    a = rng.uniform(0, 6, (20000, 3))
    b = rng.uniform(0, 6, (20000, 3))
    got, want = ctx.occluded(a, b), rr.occluded(a, b)
    assert np.array_equal(got, want)
    assert 100 < want.sum() < len(want)


def test_intersect_random_soup(ref):
    scene = random_soup(10000, 31, 10.0, 0.8)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(77)
    o = rng.uniform(0, 10, (5000, 3))
    d = rng.normal(size=(5000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t, tri = ctx.intersect(o, d)
    rt, rtri = rr.intersect(o, d)
    assert np.array_equal(tri, rtri)
    assert np.array_equal(t, rt)
    assert (tri >= 0).sum() > 2500


def test_occluded_grazing_axis_aligned(ref):
    """Segments lying in / along the box walls of the Cornell grid: zero
    direction components (inf inverse), NaN slab terms and edge hits."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=32)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(5)
    grid = np.array([0.0, 0.25, 0.5, 0.93, 1.0, 1.25, 1.5, 2.0, 2.25])
    n = 30000
    a = rng.choice(grid, (n, 3))
    b = rng.choice(grid, (n, 3))
    # keep one or two coordinates equal so segments run along planes
    same = rng.random((n, 3)) < 0.4
    b = np.where(same, a, b)
    a[:, 1] = np.clip(a[:, 1], 0, 1.0)
    got, want = ctx.occluded(a, b), rr.occluded(a, b)
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]
    assert 0 < want.sum() < n


def test_occluded_many_emitter_maze(ref):
    """Dense small emitters (the c3 ceiling) at reduced count."""
    scene = scenes.maze(20000, seed=3, width=8, height=8)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(9)
    n = 20000
    a = np.stack([rng.uniform(-1, 11, n), rng.uniform(0, 1.2, n), rng.uniform(-1, 11, n)], 1)
    b = np.stack([rng.uniform(-1, 11, n), rng.uniform(3.9, 4.0, n), rng.uniform(-1, 11, n)], 1)
    got, want = ctx.occluded(a, b), rr.occluded(a, b)
    assert np.array_equal(got, want)
    assert 0 < want.sum() < n


def _check_sah(ctx, rr, o, d, t_min=0.0):
    """Full intersect and the SAH decision alone against the reference: every
    decided ray (tri != -2) must already be the reference's answer."""
    t, tri = ctx.intersect(o, d, t_min)
    rt, rtri = rr.intersect(o, d, t_min)
    assert np.array_equal(tri, rtri) and np.array_equal(t, rt)
    st, stri = ctx.intersect(o, d, t_min, sah_only=True)
    dec = stri != -2
    assert np.array_equal(stri[dec], rtri[dec]) and np.array_equal(st[dec], rt[dec])
    return dec, rtri


def test_intersect_sah_decisions_and_tmin(ref, shadow_tree):
    """Bounce-like queries: origins on the soup's triangles, t_min > 0."""
    scene = random_soup(6000, 17, 8.0, 0.7)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(11)
    v = scene.vertices
    pick = rng.integers(0, v.shape[0], 8000)
    u = rng.random((8000, 2))
    u = np.where(u.sum(1, keepdims=True) > 1, 1 - u, u)
    o = v[pick, 0] + u[:, :1] * (v[pick, 1] - v[pick, 0]) + u[:, 1:] * (v[pick, 2] - v[pick, 0])
    d = rng.normal(size=(8000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dec, rtri = _check_sah(ctx, rr, o, d, t_min=1e-3)
    assert (rtri >= 0).sum() > 3000
    # the SAH closest hit runs on the quantized tree (absent with the 128-byte nodes)
    assert dec.mean() > 0.9 if shadow_tree != "tris-128B" else not dec.any()


def test_intersect_exact_ties_defer_to_reference_order(ref):
    """Every triangle twice (identical Moller-Trumbore t): the reference keeps
    the first one its leaf scan meets; the SAH traversal must defer."""
    base = random_soup(3000, 23, 8.0, 0.8)
    v = base.vertices
    mats_idx = np.arange(2 * v.shape[0]) % 2
    scene = Scene(np.concatenate([v, v[::-1]]), mats_idx.astype(np.uint32),
                  np.array([[0.5, 0.5, 0.5, 0, 0, 0], [0, 0, 0, 1, 1, 1]], float),
                  scenes.Camera((0, 0, -5), (0, 0, 0), (0, 1, 0), 45, 8, 8), "dup")
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(12)
    o = rng.uniform(0, 8, (6000, 3))
    d = rng.normal(size=(6000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dec, rtri = _check_sah(ctx, rr, o, d)
    hits = rtri >= 0
    assert hits.sum() > 1000 and not dec[hits].any()  # every hit is a tie


@pytest.mark.parametrize("limit", ["3", "5"])
def test_occluded_stack_overflow_finishes_exactly(ref, monkeypatch, limit):
    """A shadow ray that would overflow k_shadow's shared-memory stack is
    finished on the exact fp64 path: forced here with a tiny stack."""
    monkeypatch.setenv("RLC_SHADOW_STACK_LIMIT", limit)
    scene = random_soup(3000, 21, 6.0, 0.8)
    ctx, rr = both(ref, scene)
    rng = np.random.default_rng(79)
    a = rng.uniform(0, 6, (20000, 3))
    b = rng.uniform(0, 6, (20000, 3))
    got, want = ctx.occluded(a, b), rr.occluded(a, b)
    assert np.array_equal(got, want)
    assert 100 < want.sum() < len(want)
