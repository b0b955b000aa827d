"""Per-ray traversal counters of a -DRLC_TRAV_STATS build:
    make -C paper_1911_10217_b200/csrc OUT=$PWD/variants/trav/lib.so OBJ=$PWD/build/obj_trav EXTRA=-DRLC_TRAV_STATS
    RLC_LIB_PATH=variants/trav/lib.so python tools/trav_counts.py c3 [max_depth]"""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, bench
from paper_1911_10217_b200 import rlcuts
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
scene, cfg = bench.make_config(name, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ctx = rlcuts.build_context(scene, cfg)
grid = rlcuts.HashGrid(ctx, cfg)
fb = rlcuts.Framebuffer(ctx)
for p in range(4):
    rlcuts.render_pass(ctx, cfg, p, grid, fb)
    rlcuts.end_of_pass_update(grid, ctx, cfg.cut)
    s = rlcuts.trav_stats()
    print(p, s, "shadow nodes/ray %.2f tris/ray %.2f | closest nodes/ray %.2f tris/ray %.2f" % (
        s["shadow_nodes"] / max(s["shadow_rays"], 1), s["shadow_tris"] / max(s["shadow_rays"], 1),
        s["closest_nodes"] / max(s["closest_rays"], 1), s["closest_tris"] / max(s["closest_rays"], 1)))
