"""A small workload for compute-sanitizer (one tool per run): learned-sampler
passes on a Cornell scene (hash insertion, cut sampling, shadow rays, sort,
fold, split-collapse, accumulation), a hash table small enough to overflow,
multi-bounce paths, and render_frame with its overlapped streams."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1911_10217_b200 import rlcuts, scenes  # noqa: E402

RL = rlcuts.SamplerKind.rl_lightcuts


def run(scene, cfg):
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    s, c = fb.download()
    assert np.isfinite(s).all()
    res = rlcuts.render_frame(ctx, cfg)
    assert np.isfinite(res.image).all()
    return grid.stats()


scene = scenes.cornell_grid(2, 1, dome_triangles=64, width=48, height=32)
print(run(scene, rlcuts.RenderConfig(spp=4, passes=2, sampler=RL, cut=rlcuts.CutConfig(cut_size=32))))
print(run(scene, rlcuts.RenderConfig(spp=4, passes=2, sampler=RL,
                                     hash=rlcuts.HashConfig(capacity=128, probe_limit=8),
                                     cut=rlcuts.CutConfig(cut_size=16))))
print(run(scene, rlcuts.RenderConfig(spp=2, passes=2, sampler=RL, max_depth=3,
                                     cut=rlcuts.CutConfig(cut_size=16))))
print("sanitize case ok")
