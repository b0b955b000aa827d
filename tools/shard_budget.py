"""Per-rank time budget of a sharded c3 frame, measured on one B200 with N
ranks emulated as N contexts (local_exchange: each rank's kernels run alone,
the collectives are done by the host between the steps).  Prints, per mode,
each rank's device time per frame by stage (CUDA events) and the exchange
volumes; the NCCL transfer time is estimated from the measured NVLink
bandwidths of B200_PROFILING.md (all-gather bus 725 GB/s).
usage: python tools/shard_budget.py [N] [frames] [config] [owner|replicated|both]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10217_b200 import dist as rdist  # noqa: E402
from paper_1911_10217_b200 import rlcuts  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 8
name = sys.argv[3] if len(sys.argv) > 3 else "c3"
which = sys.argv[4] if len(sys.argv) > 4 else "both"
modes = {"owner": (True,), "replicated": (False,), "both": (True, False)}[which]
scene, cfg = bench.make_config(name)
H, W = scene.camera.height, scene.camera.width
dev = torch.device("cuda", 0)
for owner in modes:
    engines = []
    for r in range(N):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev, world=N))
    rows = [rdist.band(H, r, N) for r in range(N)]
    warm = 4
    for p in range(warm):
        rdist.local_exchange(engines, rows, p, owner)
    for e in engines:
        e.ctx.synchronize()
        e.ctx.stage_times()
        e.ctx.enable_timing(True)
    t0 = time.perf_counter()
    for p in range(warm, warm + frames):
        rdist.local_exchange(engines, rows, p, owner, serial=True)
    wall = time.perf_counter() - t0
    per_rank = []
    for e in engines:
        st = e.ctx.stage_times()
        e.ctx.enable_timing(False)
        per_rank.append({k: v[0] / frames for k, v in st.items() if v[1]})
    mode = "owner-folded" if owner else "replicated fold"
    print(f"== {name}, N={N}, {mode}: per-rank device ms per frame, each rank's steps run alone "
          f"(stage sums; a rank's own streams overlap, so its frame is below the sum)")
    keys = sorted({k for d in per_rank for k in d})
    print("rank " + " ".join(f"{k:>14s}" for k in keys))
    for r, d in enumerate(per_rank):
        print(f"{r:4d} " + " ".join(f"{d.get(k, 0.0):14.4f}" for k in keys))
    e0 = engines[0]
    block = 32 * (e0.cap + 1)
    slots = N * (e0.cap + 1)
    # the records that exist this frame (block headers): what the peer exchange moves
    heads = [e.trace(warm + frames, rr) for e, rr in zip(engines, rows)]
    for e in engines:
        e.ctx.synchronize()
    counts = [int(h[:8].view(torch.int64).item()) for h in heads]
    peer_out = max(counts) * 32 * (N - 1)
    entries = rlcuts.shard_entry_arrays(e0.ctx)[2]
    if not owner:
        comm = ""
    elif entries:  # entry exchange: q_before reduce-scattered, per-entry finals all-reduced
        rs, ar = (N - 1) / N * slots * 8, 2 * (N - 1) / N * entries * 12
        comm = (f" entry exchange: q_before reduce-scatter {slots * 8 / 1e6:.1f} MB (~{rs / 725e9 * 1e6:.0f} us)"
                f" + per-entry all-reduce {entries * 12 / 1e6:.1f} MB (~{ar / 725e9 * 1e6:.0f} us)")
    else:
        ar = 2 * (N - 1) / N * slots * 12
        comm = (f" q_before + entry-count all-reduce {slots * 12 / 1e6:.1f} MB "
                f"(~{ar / 725e9 * 1e6:.0f} us)")
    print(f"record block {block / 1e6:.2f} MB per rank; all-gather receives "
          f"{(N - 1) * block / 1e6:.1f} MB per rank (~{(N - 1) * block / 725e9 * 1e6:.0f} us at 725 GB/s);"
          + comm)
    print(f"records per rank {min(counts)}..{max(counts)} of {e0.cap} slots: the peer exchange "
          f"stores {peer_out / 1e6:.1f} MB from the busiest rank (~{peer_out / 725e9 * 1e6:.0f} us)")
    print(f"emulation wall time {wall / frames * 1e3:.1f} ms per frame (all {N} ranks, serial)")
    del engines
    torch.cuda.empty_cache()
