"""GPU: CUDA-graph replays of whole passes (rlc_render_passes_async)
must equal the pass-by-pass path and the reference bit for bit, including when
graph passes and ordinary passes alternate on one grid."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu
RL = rlcuts.SamplerKind.rl_lightcuts


@pytest.fixture(autouse=True)
def graphs_on(monkeypatch):
    monkeypatch.setenv("RLC_GRAPHS", "1")  # opt-in (rlc_capi.cpp run_passes)


def _state(grid, fb):
    s, c = fb.download()
    return s, c, (grid.export() if grid is not None else None)


def _same(a, b):
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    if a[2] is not None:
        assert a[2].keys() == b[2].keys()
        for k, v in a[2].items():
            for f in v:
                assert np.array_equal(v[f], b[2][k][f]), (k, f)


def test_render_frame_graph_change_counts(ref):
    """render_frame replays 8-pass graphs; its per-pass split-collapse counts
    (filed on the device by the graph) equal the reference's."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=64, width=32, height=24)
    cfg = rlcuts.RenderConfig(spp=18, passes=18, sampler=RL,
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=1.5))
    ctx = rlcuts.build_context(scene, cfg)
    res = rlcuts.render_frame(ctx, cfg)
    rr = ref.RefRun(scene, cfg)
    want = [rr.run_pass(p)[0] for p in range(cfg.passes)]
    assert list(res.sc_changes) == want and sum(want) > 0


@pytest.mark.parametrize("sampler,depth", [(RL, 1), (RL, 2), (rlcuts.SamplerKind.energy, 1)])
def test_graph_passes_match_pass_by_pass(ref, sampler, depth):
    scene = scenes.cornell_grid(2, 1, dome_triangles=64, width=40, height=30)
    cfg = rlcuts.RenderConfig(spp=20, passes=20, sampler=sampler, max_depth=depth,
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    runs = []
    for mode in ("single", "graph", "mixed"):
        ctx = rlcuts.build_context(scene, cfg)
        grid = rlcuts.HashGrid(ctx, cfg) if sampler == RL else None
        fb = rlcuts.Framebuffer(ctx)
        if mode == "single":
            for p in range(cfg.passes):
                rlcuts.render_pass(ctx, cfg, p, grid, fb)
                if grid is not None:
                    rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
        elif mode == "graph":
            l0 = rlcuts.kernel_launches()
            rlcuts.render_passes(ctx, cfg, 0, cfg.passes, grid, fb)
            ctx.synchronize()
            assert rlcuts.kernel_launches() - l0 >= 4 * cfg.passes  # replays are counted
        else:  # graph replays, single passes and graph replays again on one grid
            rlcuts.render_passes(ctx, cfg, 0, 9, grid, fb)  # one 8-pass replay + 1 pass
            rlcuts.render_pass(ctx, cfg, 9, grid, fb)
            if grid is not None:
                rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
            rlcuts.render_passes(ctx, cfg, 10, 10, grid, fb)
            ctx.synchronize()
        runs.append(_state(grid, fb))
    _same(runs[0], runs[1])
    _same(runs[0], runs[2])
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        rr.run_pass(p)
    rs, rc = rr.framebuffer()
    assert np.array_equal(runs[1][0], rs) and np.array_equal(runs[1][1], rc)
