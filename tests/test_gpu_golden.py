"""GPU path against the committed golden runs of the reference
(tests/golden/runs.npz): needs neither /root/reference nor oracle/_ref."""
import pytest

from paper_1911_10217_b200 import rlcuts
from test_oracle import RL, RUN_CASES, check_run_against_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(RUN_CASES))
def test_gpu_runs_golden(name):
    scene, cfg = RUN_CASES[name]()
    ctx = rlcuts.build_context(scene, cfg)
    grid = rlcuts.HashGrid(ctx, cfg) if cfg.sampler == RL else None
    fb = rlcuts.Framebuffer(ctx)
    changes = []
    for p in range(cfg.passes):
        rlcuts.render_pass(ctx, cfg, p, grid, fb)
        changes.append(rlcuts.end_of_pass_update(grid, ctx, cfg.cut) if grid else 0)
    stats = grid.stats() if grid else {"occupied": 0, "lookups": 0, "fallback_hits": 0}
    check_run_against_golden(name, fb.download(), changes, stats,
                             grid.export() if grid else {})
