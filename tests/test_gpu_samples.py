"""Per-sample parity (the north star's "selected light indices bit-exact"):
every light sample of a pass -- selected cut entry and emitter index, the
fallback flag, the live q_before the reference's pdf reads
(proj/src/cut.cpp:97-106), v and the per-sample radiance
(proj/src/estimators.cpp:50-106) -- exported by rlc_pass_samples and compared
with `==` against the oracle's per-sample dump, pass by pass.  The oracle
(oracle/rlc_oracle.cpp) is itself pinned to the reference (tests/test_oracle.py);
the framebuffer and the learned state are compared with the compiled reference
as well, so selection, learning and image agree three ways."""
import numpy as np
import pytest

from oracle.restate import OracleRun
from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu
RL = rlcuts.SamplerKind.rl_lightcuts
FIELDS = ("pixel", "cluster", "emitter", "fallback", "q_before", "v", "total", "radiance")


def assert_same_samples(got, want, where):
    assert len(got["pixel"]) == len(want["pixel"]), (where, len(got["pixel"]), len(want["pixel"]))
    for f in FIELDS:
        a, b = got[f], want[f]
        bad = np.flatnonzero(np.any((a != b).reshape(len(a), -1), axis=1)) if len(a) else []
        assert len(bad) == 0, f"{where}: {f} differs at {len(bad)} samples, first {bad[:5]}"


def run_sampled(scene, cfg, passes=None, ref=None):
    """GPU passes with the per-sample export on, each checked against the
    oracle's samples; optionally the whole state against the reference."""
    ctx = rlcuts.build_context(scene, cfg)
    rlcuts.enable_sample_export(ctx)
    grid = rlcuts.HashGrid(ctx, cfg) if cfg.sampler == RL else None
    fb = rlcuts.Framebuffer(ctx)
    orc = OracleRun(scene, cfg)
    rr = ref.RefRun(scene, cfg) if ref is not None else None
    n = 0
    for p in range(cfg.passes if passes is None else passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        got = rlcuts.pass_samples(ctx, cfg)
        ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut) if grid else 0
        och = orc.run_pass(p)
        assert_same_samples(got, orc.samples(), f"pass {p}")
        assert ch == och
        if rr is not None:
            rch, _ = rr.run_pass(p)
            assert ch == rch
        n += len(got["pixel"])
    if rr is not None:
        s, c = fb.download()
        rs, rc = rr.framebuffer()
        assert np.array_equal(c, rc) and np.array_equal(s, rs)
        if grid is not None:
            assert grid.stats() == rr.stats()
            cells, rcells = grid.export(), rr.export()
            assert cells.keys() == rcells.keys()
            for k, v in rcells.items():
                for f in v:
                    assert np.array_equal(cells[k][f], v[f]), (k, f)
    return n, grid


def test_c1_samples_bit_exact(ref):
    """c1 at its bench size (256 x 256, 1,024 emitters), 6 of its 16 frames."""
    scene, st = scenes.config_scene("c1")
    cfg = rlcuts.RenderConfig(spp=st["spp"], passes=st["passes"], sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    n, _ = run_sampled(scene, cfg, passes=6, ref=ref)
    assert n > 6 * 40000


def test_c3_samples_bit_exact(ref):
    """The headline scene (1M emitters) at 320 x 180, 4 frames."""
    scene, st = scenes.config_scene("c3")
    scene = scene.with_resolution(320, 180)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    n, _ = run_sampled(scene, cfg, ref=ref)
    assert n > 4 * 30000


@pytest.mark.parametrize("sampler", [rlcuts.SamplerKind.uniform, rlcuts.SamplerKind.energy])
def test_baseline_sampler_samples_bit_exact(sampler):
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=40)
    cfg = rlcuts.RenderConfig(spp=4, passes=2, sampler=sampler)
    run_sampled(scene, cfg)


@pytest.mark.parametrize("depth", [2, 3])
def test_multi_bounce_samples_bit_exact(depth):
    scene = scenes.cornell_grid(2, 2, dome_triangles=128, width=40, height=32)
    cfg = rlcuts.RenderConfig(spp=4, passes=2, sampler=RL, max_depth=depth,
                              cut=rlcuts.CutConfig(cut_size=32))
    run_sampled(scene, cfg)


def test_overflow_samples_bit_exact(ref):
    """A table too small for the scene: the fallback flag of every sample
    (and so its cut, its q_before and whether it updates) as the reference's
    canonical insertion order decides."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=64, height=48)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(capacity=256, probe_limit=8),
                              cut=rlcuts.CutConfig(cut_size=32))
    _, grid = run_sampled(scene, cfg, ref=ref)
    assert grid.fallback_hits() > 1000


def test_c3_full_resolution_two_frames(ref):
    """c3 exactly as benched (1920 x 1080, 1 spp per frame, 1M emitters):
    two frames against the reference (workers = 1) and the oracle's
    per-sample selections."""
    scene, st = scenes.config_scene("c3")
    cfg = rlcuts.RenderConfig(spp=st["spp"], passes=st["passes"], sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    n, grid = run_sampled(scene, cfg, passes=2, ref=ref)
    assert n > 2 * 1_400_000 and grid.fallback_hits() == 0


def test_c3_learning_schedule_64_frames(ref):
    """c3's whole real-time learning schedule (64 frames at 1 spp) at
    480 x 270 against the reference: image, learned cuts, split-collapse
    counts every frame."""
    scene, st = scenes.config_scene("c3")
    scene = scene.with_resolution(480, 270)
    cfg = rlcuts.RenderConfig(spp=st["spp"], passes=st["passes"], sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    assert cfg.passes == 64
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
        rch, _ = rr.run_pass(p)
        assert ch == rch, p
    s, c = fb.download()
    rs, rc = rr.framebuffer()
    assert np.array_equal(c, rc) and np.array_equal(s, rs)
    assert grid.stats() == rr.stats()
    cells, rcells = grid.export(), rr.export()
    assert cells.keys() == rcells.keys()
    for k, v in rcells.items():
        for f in v:
            assert np.array_equal(cells[k][f], v[f]), (k, f)
    assert [(s_, k) for s_, _, k, _ in grid.slots()] == rr.slots()


def test_c2_four_frames(ref):
    """c2 (4 x 4 occluding boxes, 16,384 emitters, 4 spp per frame) at
    320 x 180, 4 frames."""
    scene, st = scenes.config_scene("c2")
    scene = scene.with_resolution(320, 180)
    cfg = rlcuts.RenderConfig(spp=4 * 4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    n, grid = run_sampled(scene, cfg, ref=ref)
    assert n > 4 * 150000 and grid.fallback_hits() == 0
