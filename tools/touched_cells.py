"""Cells touched per frame (folded this pass, so split-collapsed at its end)
and split-collapse changes per frame on a config: the row-exchange volume of
an owner-partitioned split-collapse.
usage: python tools/touched_cells.py [config] [frames]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 12
scene, cfg = bench.make_config(name)
ctx = rlcuts.build_context(scene, cfg)
grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
M = cfg.cut.cut_size
for p in range(frames):
    rlcuts.render_pass(ctx, cfg, p, grid, fb)
    sl = grid.slots()
    touched = sum(1 for s in sl if s[3])
    ch = rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    print(f"frame {p:3d}: cells {len(sl):6d} touched {touched:6d} "
          f"({touched * 28 * M / 1e6:.1f} MB of cut rows) split-collapse changes {ch}")
