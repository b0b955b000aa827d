"""Sharded c3 frames at one rank over a real NCCL communicator: host time to
enqueue a frame and device time per frame, enqueued frame by frame
(rlc_shard_frame) or replayed from a captured CUDA graph (rlc_shard_frames).
usage: python tools/shard_graph_time.py [config] [frames]"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import dist as rdist  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("gloo", rank=0, world_size=1)
scene, cfg = bench.make_config(name)
dev = torch.device("cuda", 0)
for graph in (False, True, False, True):
    ctx = rlcuts.build_context(scene, cfg)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    eng = rdist.GpuEngine(ctx, grid, fb, cfg, dev)
    fr = rdist.NcclFrame(eng, scene.camera.height, 0, 1, 0, owner=True)
    fr.run(0, 8, graph)  # warm-up (and the capture)
    rlcuts.shard_sync(ctx, grid)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    t0 = time.perf_counter()
    fr.run(8, frames, graph)
    host = (time.perf_counter() - t0) / frames * 1e3
    b.record(stream)
    b.synchronize()
    devms = a.elapsed_time(b) / frames
    print(f"{name} one rank, {'graph replay' if graph else 'frame by frame'}: "
          f"host enqueue {host:.3f} ms/frame, device {devms:.3f} ms/frame")
    ctx.set_stream(None)
dist.destroy_process_group()
