"""GPU parity of the whole per-pass path against the compiled reference
(oracle/_ref): same scene arrays, same config, workers = 1 (the reference's
only deterministic mode).  Bit-exact: light selection (through the cut
state it produces), cut topology, learnt q / cdf / visits, framebuffer sums
and counts, split-collapse change counts and grid statistics."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu

RL = rlcuts.SamplerKind.rl_lightcuts


def run_both(ref, scene, cfg):
    ctx = rlcuts.build_context(scene, cfg)
    grid = rlcuts.HashGrid(ctx, cfg) if cfg.sampler == RL else None
    fb = rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene, cfg)
    info, rinfo = ctx.info(), rr.info()
    for k in ("base_tile", "shadow_eps", "num_emitters", "light_tree_nodes", "bvh_nodes"):
        assert info[k] == rinfo[k], k
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut) if grid else 0
        rch, _ = rr.run_pass(p)
        assert ch == rch, f"pass {p}: split-collapse changes {ch} vs reference {rch}"
    return ctx, grid, fb, rr


def assert_same_state(grid, fb, rr):
    s, c = fb.download()
    rs, rc = rr.framebuffer()
    assert np.array_equal(c, rc)
    bad = np.argwhere(s != rs)
    assert bad.size == 0, f"{len(bad)} radiance mismatches, max |d| {np.abs(s - rs).max()}"
    if grid is None:
        return
    st, rst = grid.stats(), rr.stats()
    assert st == rst
    cells, rcells = grid.export(), rr.export()
    assert set(cells) == set(rcells)
    for k, v in cells.items():
        for f in ("node_ids", "ends", "q", "cdf", "visits"):
            assert np.array_equal(v[f], rcells[k][f]), (k, f)


def test_cornell2_rl_bit_exact(ref):
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=64, height=48)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL)
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    assert grid.fallback_hits() == 0 and grid.occupied_count() > 100


def test_c1_analog_rl_bit_exact(ref):
    scene, st = scenes.config_scene("c1")
    scene = scene.with_resolution(64, 64)
    cfg = rlcuts.RenderConfig(spp=8, passes=8, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


def test_harmonic_multi_iteration_small_cut(ref):
    scene = scenes.cornell_grid(2, 3, dome_triangles=512, width=40, height=40)
    cfg = rlcuts.RenderConfig(
        spp=6, passes=3, sampler=RL, seed=9,
        cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0, iterations=3,
                             alpha_schedule=rlcuts.AlphaSchedule.harmonic))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


def test_jittered_keys_and_fine_normals(ref):
    scene = scenes.cornell_grid(1, 2, dome_triangles=128, width=48, height=48)
    cfg = rlcuts.RenderConfig(spp=4, passes=2, sampler=RL,
                              hash=rlcuts.HashConfig(jitter_scale=1.0, normal_bits=6))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


@pytest.mark.parametrize("sampler", [rlcuts.SamplerKind.uniform, rlcuts.SamplerKind.energy])
def test_baseline_samplers_bit_exact(ref, sampler):
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=40)
    cfg = rlcuts.RenderConfig(spp=2, passes=2, sampler=sampler)
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


@pytest.mark.parametrize("depth,sampler", [(2, RL), (3, RL), (5, RL),
                                           (2, rlcuts.SamplerKind.uniform),
                                           (3, rlcuts.SamplerKind.energy)])
def test_multi_bounce_bit_exact(ref, depth, sampler):
    """max_depth > 1 (render.cpp:71-136): cosine-hemisphere bounces with the
    host libm's sin/cos, closest hits from t_min = shadow_eps, NEE and
    update_q records at every vertex, throughput-weighted radiance."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=40, height=32)
    cfg = rlcuts.RenderConfig(spp=4, passes=2, max_depth=depth, sampler=sampler)
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


def test_multi_bounce_c1_analog_learns(ref):
    scene, st = scenes.config_scene("c1")
    scene = scene.with_resolution(48, 48)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, max_depth=3, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    assert grid.lookup_count() > 48 * 48 * 4 * 1.5  # the bounces reached learned vertices


def test_zero_depth_adds_empty_samples(ref):
    scene = scenes.cornell_grid(1, 1, dome_triangles=8, width=16, height=16)
    cfg = rlcuts.RenderConfig(spp=2, passes=2, max_depth=0, sampler=RL)
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


def test_render_frame_matches_reference(ref):
    """render_frame reuses the context's grid/framebuffer cache: repeated
    calls, and calls with another config, must each equal a fresh reference
    render_frame (render.cpp:202-240)."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=32, width=32, height=32)
    cfg = rlcuts.RenderConfig(spp=4, passes=2, sampler=RL)
    cfg2 = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, seed=4,
                               cut=rlcuts.CutConfig(cut_size=16))
    cfg3 = rlcuts.RenderConfig(spp=4, passes=2, sampler=RL, max_depth=3)
    ctx = rlcuts.build_context(scene, cfg)
    for c in (cfg, cfg, cfg2, cfg3, cfg):
        res = rlcuts.render_frame(ctx, c)
        rres = ref.ref_render_frame(scene, c)
        assert np.array_equal(res.image, rres["image"])
        assert res.sc_changes == rres["sc_changes"]
        assert (res.occupied_cells, res.lookups, res.fallback_hits) == (
            rres["occupied"], rres["lookups"], rres["fallback_hits"])


def test_render_frame_repeated_c3_matches_reference(ref):
    """render_frame called back to back on the c3 scene (full-size tables,
    the next pass's primary rays overlapping each pass's tail): every call
    resets the cached grid on the main stream, and the first pass's primary
    rays (side stream) must see the reset table -- each call equals a fresh
    reference render_frame."""
    scene, st = scenes.config_scene("c3")
    scene = scene.with_resolution(320, 180)
    cfg = rlcuts.RenderConfig(spp=3, passes=3, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    ctx = rlcuts.build_context(scene, cfg)
    rres = ref.ref_render_frame(scene, cfg)
    for _ in range(4):
        res = rlcuts.render_frame(ctx, cfg)
        assert np.array_equal(res.image, rres["image"])
        assert res.sc_changes == rres["sc_changes"]
        assert (res.occupied_cells, res.lookups, res.fallback_hits) == (
            rres["occupied"], rres["lookups"], rres["fallback_hits"])


@pytest.mark.parametrize("depth", [1, 2])
def test_async_passes_bit_exact(ref, depth):
    """Passes enqueued back to back without host synchronisation (as the
    bench and render_frame drive them): the next pass's primary rays overlap
    the previous pass's tail on side streams; state must still equal the
    reference after every pass sequence."""
    scene, st = scenes.config_scene("c1")
    scene = scene.with_resolution(96, 80)
    cfg = rlcuts.RenderConfig(spp=8, passes=8, sampler=RL, max_depth=depth,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb, sync=False)
        rlcuts.end_of_pass_update(grid, ctx, cfg.cut, sync=False)
        rr.run_pass(p)
    ctx.synchronize()
    assert_same_state(grid, fb, rr)


@pytest.mark.parametrize("m", [4096, 8192])
def test_large_cuts_bit_exact(ref, m):
    """Cut sizes whose split-collapse rows no longer fit in shared memory
    (32 M bytes per warp > 200 KB) take k_split's global-memory rows."""
    scene = scenes.maze(16384, seed=3, width=40, height=32)
    cfg = rlcuts.RenderConfig(spp=2, passes=2, sampler=RL, cut=rlcuts.CutConfig(cut_size=m),
                              hash=rlcuts.HashConfig(capacity=4096, base_tile=0.1))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)


@pytest.mark.parametrize("case", ["looks_away", "one_pixel", "odd_raster"])
def test_degenerate_frames_bit_exact(ref, case):
    """No hits at all (every stage runs on empty work), a 1x1 image and an
    odd raster that fills no 8x4 tile completely."""
    scene = scenes.cornell_grid(1, 1, dome_triangles=8, width=21, height=13)
    cam = scene.camera
    if case == "looks_away":
        scene = scenes.Scene(scene.vertices, scene.material_ids, scene.materials,
                             scenes.Camera((0.5, 0.5, -50.0), (0.5, 0.5, -100.0), (0.0, 1.0, 0.0),
                                           cam.vfov_degrees, 16, 16))
    elif case == "one_pixel":
        scene = scene.with_resolution(1, 1)
    cfg = rlcuts.RenderConfig(spp=3, passes=3, sampler=RL, max_depth=2)
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    if case == "looks_away":
        assert grid.occupied_count() == 0


def test_nan_rays_follow_the_reference(ref):
    """A camera whose up vector is parallel to the view direction makes every
    camera ray NaN.  The reference's slab and Moller-Trumbore tests pass NaN,
    so it reports NaN-distance hits and then level_for_footprint rejects the
    NaN area pdf; the device path must do the same (and the batch intersect
    must return the reference's last-tested triangle)."""
    scene = scenes.cornell_grid(1, 1, dome_triangles=8, width=21, height=13)
    cam = scene.camera
    scene = scenes.Scene(scene.vertices, scene.material_ids, scene.materials,
                         scenes.Camera((0.5, 0.5, -50.0), (0.5, 0.5, -100.0), cam.up,
                                       cam.vfov_degrees, 16, 16))
    cfg = rlcuts.RenderConfig(spp=1, passes=1, sampler=RL)
    ctx = rlcuts.build_context(scene, cfg)
    rr = ref.RefRun(scene, cfg)
    o = np.array([[0.5, 0.5, -50.0]] * 2)
    d = np.array([[np.nan, np.nan, np.nan], [np.nan, 0.2, -1.0]])
    t, tri = ctx.intersect(o, d)
    rt, rtri = rr.intersect(o, d)
    assert np.array_equal(tri, rtri) and np.array_equal(np.isnan(t), np.isnan(rt))
    with pytest.raises(ValueError, match="area pdf must be positive"):
        rr.run_pass(0)
    with pytest.raises(ValueError, match="area pdf must be positive"):
        rlcuts.render_pass(ctx, cfg, 0, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx))


@pytest.mark.parametrize("scale,offset", [(3e8, 0.0), (1.0, 2e8), (1e-12, 0.0)])
def test_extreme_coordinates_bit_exact(ref, scale, offset):
    """Coordinates beyond the fp32 decision range (|x| > 1e8: the exact fp64
    traversals run) and a tiny scene (fp32 terms near their underflow slack)."""
    base = scenes.cornell_grid(2, 1, dome_triangles=32, width=32, height=24)
    cam = base.camera
    sc = scenes.Scene(base.vertices * scale + offset, base.material_ids, base.materials,
                      scenes.Camera(tuple(np.array(cam.origin) * scale + offset),
                                    tuple(np.array(cam.look_at) * scale + offset), cam.up,
                                    cam.vfov_degrees, cam.width, cam.height))
    cfg = rlcuts.RenderConfig(spp=2, passes=2, sampler=RL, max_depth=2)
    _, grid, fb, rr = run_both(ref, sc, cfg)
    assert_same_state(grid, fb, rr)


def test_degenerate_emitter_raises_like_the_reference(ref):
    """A zero-area emissive triangle: sample_triangle_point (scene.cpp:49-51)
    throws when it is drawn; the device path reports the same error."""
    base = scenes.cornell_grid(1, 1, dome_triangles=8, width=16, height=16)
    v = base.vertices.copy()
    emissive = np.nonzero((base.materials[:, 3:].sum(axis=1) > 0)[base.material_ids])[0]
    v[emissive[0], 2] = v[emissive[0], 1]  # collapse one emitter to a segment
    sc = scenes.Scene(v, base.material_ids, base.materials, base.camera)
    cfg = rlcuts.RenderConfig(spp=8, passes=1, sampler=rlcuts.SamplerKind.uniform)
    ctx = rlcuts.build_context(sc, cfg)
    rr = ref.RefRun(sc, cfg)
    with pytest.raises(ValueError) as want:
        rr.run_pass(0)
    with pytest.raises(ValueError) as got:
        rlcuts.render_pass(ctx, cfg, 0, None, rlcuts.Framebuffer(ctx))
    assert str(got.value) == str(want.value)


def test_errors_match_reference_exceptions(ref):
    scene = scenes.cornell_grid(1, 1, dome_triangles=8, width=8, height=8)
    cfg = rlcuts.RenderConfig(spp=3, passes=2, sampler=RL)
    ctx = rlcuts.build_context(scene, cfg)
    fb = rlcuts.Framebuffer(ctx)
    grid = rlcuts.HashGrid(ctx, cfg)
    with pytest.raises(ValueError, match="divisible"):
        rlcuts.render_pass(ctx, cfg, 0, grid, fb)
    cfg2 = rlcuts.RenderConfig(spp=2, passes=2, sampler=RL)
    with pytest.raises(ValueError, match="hash grid"):
        rlcuts.render_pass(ctx, cfg2, 0, None, fb)
    with pytest.raises(ValueError, match="capacity"):
        rlcuts.HashGrid(ctx, rlcuts.RenderConfig(sampler=RL, hash=rlcuts.HashConfig(capacity=0)))
    with pytest.raises(ValueError, match="cut size"):
        rlcuts.HashGrid(ctx, rlcuts.RenderConfig(sampler=RL, cut=rlcuts.CutConfig(cut_size=0)))


@pytest.mark.parametrize("name,res,passes", [("c3", (192, 108), 3), ("c5", (96, 54), 2)])
def test_full_size_scene_bit_exact(ref, name, res, passes):
    """The bench scenes themselves (1M / 4M emitters: full-size traversal
    trees, light tree and cuts) at a reduced raster, against the reference."""
    scene, st = scenes.config_scene(name)
    scene = scene.with_resolution(*res)
    spp_pp = st["spp"] // st["passes"]
    cfg = rlcuts.RenderConfig(spp=spp_pp * passes, passes=passes, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    assert grid.fallback_hits() == 0 and grid.lookup_count() > 0.5 * res[0] * res[1] * spp_pp


def test_full_resolution_c3_properties():
    """c3 at its bench size (1920x1080, 1M emitters), where the reference is too
    slow to run in a test: size-independent invariants of the learned state
    after a few frames -- every pixel sampled once per frame, light samples
    counted once each, cdf rows exact prefix sums of q, cut leaves a
    partition of the emitter range, no fallback cells."""
    scene, st = scenes.config_scene("c3")
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rlcuts.render_passes(ctx, cfg, 0, cfg.passes, grid, fb)
    ctx.synchronize()
    s, c = fb.download()
    assert (c == cfg.passes).all()
    assert np.isfinite(s).all() and (s >= 0).all()
    stats = grid.stats()
    assert stats["fallback_hits"] == 0 and stats["occupied"] > 1000
    n_emit = ctx.info()["num_emitters"]
    cells = grid.export()
    rng = np.random.default_rng(0)
    for k in rng.choice(len(cells), size=200, replace=False):
        v = list(cells.values())[k]
        q, cdf, ends = v["q"], v["cdf"], v["ends"]
        assert np.array_equal(cdf, np.cumsum(q))  # serial left-to-right sum, as rebuild_cdf
        assert (np.diff(ends.astype(np.int64)) > 0).all() and ends[-1] == n_emit
        assert (q > 0).all() and (v["visits"] >= 1).all()


def test_hash_grid_host_views_match_reference(ref):
    """HashGrid's host accessors (hash_grid.hpp:87-110) served from the device
    grid: dump_stats text, memory_records, the touched slots between
    render_pass and end_of_pass_update, key_of, fallback_cut.  New keys go in
    in the reference's canonical insertion order, so slot positions are the
    reference's too."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=64, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=3, passes=3, sampler=RL,
                              cut=rlcuts.CutConfig(cut_size=32))
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene, cfg)
    for p in range(2):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
        rr.run_pass(p)
    rlcuts.render_pass(ctx, cfg, 2, grid, fb)  # touched slots set, not yet cleared
    rr.render_only(2)
    text, mem, touched = rr.grid_views()
    assert grid.dump_stats() == text
    assert grid.memory_records() == mem
    got = [grid.key_of(s) for s in grid.touched_slots()]
    assert got == touched and len(got) > 50
    assert [(s, k) for s, _, k, _ in grid.slots()] == rr.slots()
    assert grid.key_of(2**31) is None
    tmpl = grid.fallback_cut()
    assert tmpl["q"].shape == (32,) and tmpl["visits"].min() == 1
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    assert grid.touched_slots() == []


@pytest.mark.parametrize("capacity,probe_limit,jitter", [(256, 32, 0.0), (700, 4, 1.0), (97, 97, 0.0)])
def test_hash_grid_overflow_matches_reference(ref, capacity, probe_limit, jitter):
    """A table far too small for the scene's cells: which keys are refused
    (the fallback cut: sampled from, never updated) depends on the order keys
    are inserted in (hash_grid.cpp:113-141).  The GPU inserts each pass's new
    keys in canonical lookup order, so fallback hits, the slot layout, the
    learned cuts and the image all equal the reference's."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=64, height=48)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(capacity=capacity, probe_limit=probe_limit,
                                                     jitter_scale=jitter),
                              cut=rlcuts.CutConfig(cut_size=32))
    ctx, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    st = grid.stats()
    assert st["fallback_hits"] > 1000 and st["occupied"] >= 0.9 * capacity
    assert [(s, k) for s, _, k, _ in grid.slots()] == rr.slots()


@pytest.mark.parametrize("depth", [2, 3])
def test_hash_grid_overflow_multi_bounce(ref, depth):
    """Overflow with several vertices per path: the canonical insertion order
    is (pixel, sample, depth), across the bounce launches."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=40)
    cfg = rlcuts.RenderConfig(spp=2, passes=2, sampler=RL, max_depth=depth,
                              hash=rlcuts.HashConfig(capacity=300, probe_limit=8),
                              cut=rlcuts.CutConfig(cut_size=16))
    _, grid, fb, rr = run_both(ref, scene, cfg)
    assert_same_state(grid, fb, rr)
    assert grid.fallback_hits() > 100
    assert [(s, k) for s, _, k, _ in grid.slots()] == rr.slots()
