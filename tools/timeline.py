"""Per-stage timeline of a few steady-state c3 frames (CUDA events on each
stream, rlc_context_stage_marks): where the overlapped streams leave the
critical path.  usage: python tools/timeline.py [config] [frames] [warm-up frames]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 20
scene, cfg = bench.make_config(name)
ctx = rlcuts.build_context(scene, cfg)
grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
for p in range(warm):
    rlcuts.render_pass(ctx, cfg, p, grid, fb, sync=False)
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut, sync=False)
ctx.synchronize()
ctx.stage_times()
ctx.enable_timing(True)
for p in range(warm, warm + frames):
    rlcuts.render_pass(ctx, cfg, p, grid, fb, sync=False)
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut, sync=False)
ctx.synchronize()
marks = ctx.stage_marks()
for st, a, b in marks:
    print(f"{st:15s} {a * 1e3:9.1f} {b * 1e3:9.1f}  {(b - a) * 1e3:7.1f} us")
print(f"{frames} frames in {(max(b for _, _, b in marks) - marks[0][1]) * 1e3:.1f} us")
