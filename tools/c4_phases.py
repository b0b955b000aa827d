"""Host phases of rlc_context_update_scene on c4 (RLC_BUILD_TIMING /
RLC_UPDATE_TIMING print them on stderr) for a few frames."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import rlcuts, scenes  # noqa: E402

scene, cfg = bench.make_config("c4")
ctx = rlcuts.build_context(scene, cfg)
grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
frames = [scenes.displace_emitters(scene, p) for p in range(1, 8)]
for p, f in enumerate(frames, 1):
    t = time.perf_counter()
    ctx.update_scene(f)
    u = time.perf_counter()
    rlcuts.render_pass(ctx, cfg, p, grid, fb)
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    print(f"frame {p}: update {1e3 * (u - t):.2f} ms, render {1e3 * (time.perf_counter() - u):.2f} ms",
          file=sys.stderr, flush=True)
