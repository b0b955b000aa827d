"""The first frame of a fresh grid on a config (every lookup new): one
render_pass + end_of_pass_update, for profiling the cold path.
usage: python tools/cold_frame.py [config]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scene, cfg = bench.make_config(name)
ctx = rlcuts.build_context(scene, cfg)
grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
rlcuts.render_pass(ctx, cfg, 0, grid, fb)
print("cold frame changes", rlcuts.end_of_pass_update(grid, ctx, cfg.cut), grid.insertion_stats())
