"""Host reference-BVH build time (rlc_debug_host_bvh, no GPU needed):
python tools/host_bvh_time.py [config] [reps]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
scene, cfg = bench.make_config(name)
desc = scene.desc()
ms, nodes = C.c_double(), C.c_uint32()
st = _lib.load().rlc_debug_host_bvh(C.byref(desc), reps, C.byref(ms), C.byref(nodes))
assert st == 0, _lib.load().rlc_last_error()
print(f"{name}: {scene.num_triangles} triangles, {nodes.value} nodes, {ms.value:.2f} ms per build")
