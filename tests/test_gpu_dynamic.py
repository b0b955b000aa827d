"""GPU: dynamic emitters (rlc_context_update_scene).

The reference has no API for moving emitters; the semantics are defined as
    ctx' = build_context(scene', cfg); ctx'.tree = ctx.tree
(a fresh scene BVH and emitter records, the creation light tree, the learned
hash grid and framebuffer carried over).  The oracle is the reference library
driven exactly that way (oracle/ref_capi.cpp ref_run_update_scene); every
frame must match it bit for bit."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes
from test_gpu_parity import RL, assert_same_state

pytestmark = pytest.mark.gpu


def run_frames(ref, scene0, cfg, frames, move_camera_at=None):
    ctx = rlcuts.build_context(scene0, cfg)
    grid = rlcuts.HashGrid(ctx, cfg) if cfg.sampler == RL else None
    fb = rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene0, cfg)
    for f in range(frames):
        if f > 0:
            s = scenes.displace_emitters(scene0, f, amplitude=0.05)
            if f == move_camera_at:
                c = s.camera
                s.camera = scenes.Camera((c.origin[0] + 0.3, c.origin[1], c.origin[2] - 0.2),
                                         c.look_at, c.up, c.vfov_degrees, c.width, c.height)
            ctx.update_scene(s)
            rr.update_scene(s)
        rlcuts.render_pass(ctx, cfg, f, grid, fb)
        ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut) if grid else 0
        rch, _ = rr.run_pass(f)
        assert ch == rch, f"frame {f}: split-collapse changes {ch} vs reference {rch}"
    return ctx, grid, fb, rr


def test_moving_emitters_maze_bit_exact(ref):
    scene0 = scenes.maze(4096, seed=7, width=64, height=48)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=0.05))
    _, grid, fb, rr = run_frames(ref, scene0, cfg, 4, move_camera_at=2)
    assert_same_state(grid, fb, rr)
    assert grid.occupied_count() > 50


@pytest.mark.parametrize("sampler", [RL, rlcuts.SamplerKind.energy])
def test_moving_emitters_cornell_multibounce(ref, sampler):
    scene0 = scenes.cornell_grid(2, 1, dome_triangles=64, width=40, height=32)
    cfg = rlcuts.RenderConfig(spp=3, passes=3, sampler=sampler, max_depth=2)
    _, grid, fb, rr = run_frames(ref, scene0, cfg, 3)
    assert_same_state(grid, fb, rr)


def test_update_scene_rejects_topology_changes(ref):
    scene0 = scenes.cornell_grid(1, 1, dome_triangles=8, width=8, height=8)
    ctx = rlcuts.build_context(scene0, rlcuts.RenderConfig())
    other = scenes.cornell_grid(2, 1, dome_triangles=8, width=8, height=8)
    assert other.num_triangles != scene0.num_triangles
    with pytest.raises(ValueError, match="must not change"):
        ctx.update_scene(other)
    mats = scene0.materials.copy()
    mats[0, 0] = 0.123
    with pytest.raises(ValueError, match="must not change"):
        ctx.update_scene(scenes.Scene(scene0.vertices, scene0.material_ids, mats, scene0.camera))


def test_c4_scene_many_updates_bit_exact(ref):
    """The c4 bench scene (65,536 emitters) over 8 moving frames at a reduced
    raster: the in-place shadow-tree refit, the reused host buffers and the
    frozen light tree chained across updates, against the reference."""
    scene0, st = scenes.config_scene("c4")
    scene0 = scene0.with_resolution(96, 54)
    cfg = rlcuts.RenderConfig(spp=8, passes=8, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    ctx = rlcuts.build_context(scene0, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene0, cfg)
    for f in range(cfg.passes):
        if f > 0:
            s = scenes.displace_emitters(scene0, f)
            ctx.update_scene(s)
            rr.update_scene(s)
        rlcuts.render_pass(ctx, cfg, f, grid, fb)
        assert rlcuts.end_of_pass_update(grid, ctx, cfg.cut) == rr.run_pass(f)[0]
    assert_same_state(grid, fb, rr)


@pytest.mark.parametrize("ahead", [1, 3])
def test_prepared_scenes_match_reference(ref, ahead):
    """rlc_context_prepare_scene / _commit_scene: the host builds of the next
    `ahead` frames run concurrently with each other and the GPU; every frame
    must still equal the reference driven through update_scene."""
    scene0 = scenes.maze(4096, seed=11, width=64, height=48)
    cfg = rlcuts.RenderConfig(spp=6, passes=6, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=0.05))
    ctx = rlcuts.build_context(scene0, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    rr = ref.RefRun(scene0, cfg)
    frames = [scene0] + [scenes.displace_emitters(scene0, f, amplitude=0.05) for f in range(1, 6)]
    tokens = {}
    for f in range(6):
        if f > 0:
            for q in range(f, min(6, f + ahead + 1)):
                if q not in tokens:
                    tokens[q] = ctx.prepare_scene(frames[q])
            ctx.commit_scene(tokens.pop(f), frames[f])
            rr.update_scene(frames[f])
        rlcuts.render_pass(ctx, cfg, f, grid, fb)
        ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
        rch, _ = rr.run_pass(f)
        assert ch == rch, f
    assert_same_state(grid, fb, rr)
    with pytest.raises(ValueError, match="token"):
        ctx.commit_scene(123456)
