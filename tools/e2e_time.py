"""Host wall time of rlc_render_frame on a config (bench.py's e2e call):
`frames` passes, and 1 pass (grid creation, the cold frame, the image
download), a few repetitions.  usage: python tools/e2e_time.py [config] [frames] [reps]"""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
scene, cfg = bench.make_config(name)
ctx = rlcuts.build_context(scene, cfg)
for n in (frames, 1):
    ecfg = rlcuts.RenderConfig(spp=n * (cfg.spp // cfg.passes), passes=n, sampler=cfg.sampler,
                               cut=cfg.cut, hash=cfg.hash, seed=cfg.seed + 1)
    rlcuts.render_frame(ctx, ecfg)  # warm
    for r in range(reps):
        t0 = time.perf_counter()
        res = rlcuts.render_frame(ctx, ecfg)
        wall = time.perf_counter() - t0
        print(f"{name} render_frame {n} passes: {wall * 1e3:.2f} ms wall, "
              f"{res.lookups / wall / 1e9:.3f} e9 light samples/s")
