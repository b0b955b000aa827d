"""GPU: handle lifetimes.  A garbage collector may finalise a context before
the grids and framebuffers that refer to it; the C-ABI keeps the context
alive until its last child is destroyed (rlc_capi.cpp context_release)."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu


def test_children_outlive_their_context():
    scene = scenes.cornell_grid(1, 1, dome_triangles=16, width=16, height=12)
    cfg = rlcuts.RenderConfig(spp=1, passes=1, sampler=rlcuts.SamplerKind.rl_lightcuts,
                              cut=rlcuts.CutConfig(cut_size=8))
    ctx = rlcuts.build_context(scene, cfg)
    grid = rlcuts.HashGrid(ctx, cfg)
    fb = rlcuts.Framebuffer(ctx)
    rlcuts.render_pass(ctx, cfg, 0, grid, fb)
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    ctx.close()  # the caller's reference goes first
    cells = grid.export()
    s, c = fb.download()
    assert len(cells) == grid.occupied_count() > 0
    assert int(c.sum()) == 16 * 12 and np.isfinite(s).all()
    grid.close()
    fb.close()  # the last child tears the context down
