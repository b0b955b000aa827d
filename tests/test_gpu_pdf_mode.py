"""pdf_mode frozen_cdf (rlc_context_set_pdf_mode; SURVEY section 8 notes, 0
fact 2): a non-parity mode weighting each learned sample's radiance by the
probability its selection used -- the cluster's share of the pass-frozen
cdf -- instead of the live q the reference reads.  Selection and learning
must stay bit-identical to the reference mode; the image must stay an
unbiased estimate (its mean agrees with the uniform sampler's)."""
import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu
RL = rlcuts.SamplerKind.rl_lightcuts


def run(scene, cfg, frozen: bool):
    ctx = rlcuts.build_context(scene, cfg)
    if frozen:
        rlcuts.set_pdf_mode(ctx, rlcuts.PDF_FROZEN_CDF)
    rlcuts.enable_sample_export(ctx)
    grid = rlcuts.HashGrid(ctx, cfg) if cfg.sampler == RL else None
    fb = rlcuts.Framebuffer(ctx)
    samples = []
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        samples.append(rlcuts.pass_samples(ctx, cfg))
        if grid is not None:
            rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    return fb.download(), (grid.export() if grid is not None else None), samples


def test_frozen_cdf_keeps_selection_and_learning():
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=40)
    cfg = rlcuts.RenderConfig(spp=8, passes=4, sampler=RL, cut=rlcuts.CutConfig(cut_size=32))
    (s0, c0), cells0, smp0 = run(scene, cfg, False)
    (s1, c1), cells1, smp1 = run(scene, cfg, True)
    assert np.array_equal(c0, c1)
    assert cells0.keys() == cells1.keys()
    for k, v in cells0.items():
        for f in v:
            assert np.array_equal(cells1[k][f], v[f]), (k, f)
    for a, b in zip(smp0, smp1):
        for f in ("cluster", "emitter", "q_before", "v", "total"):
            assert np.array_equal(a[f], b[f]), f
    for a, b in zip(smp0, smp1):  # the frozen weight marks learned samples, in its mode only
        assert not a["frozen"].any()
        assert not (b["frozen"] & ~b["learned"]).any()
        assert not (b["learned"] & b["nonzero"] & ~b["frozen"]).any()
    assert not np.array_equal(s0, s1)  # the weights differ where q moved within a pass


def test_frozen_cdf_image_mean_unbiased():
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=32, height=24)
    n = 96
    cfg = rlcuts.RenderConfig(spp=n, passes=n, sampler=RL, cut=rlcuts.CutConfig(cut_size=32))
    (s1, c1), _, _ = run(scene, cfg, True)
    ucfg = rlcuts.RenderConfig(spp=n, passes=n, sampler=rlcuts.SamplerKind.uniform)
    (su, cu), _, _ = run(scene, ucfg, False)
    m1 = (s1.sum(axis=-1) / c1).mean()
    mu = (su.sum(axis=-1) / cu).mean()
    assert abs(m1 - mu) / mu < 0.03, (m1, mu)
