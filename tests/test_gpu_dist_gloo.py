"""Two processes sharing the device, world size 2 over gloo: each rank drives
its GpuEngine through ShardedFrame.step -- rlc_shard_trace, the block
all-gather, rlc_shard_fold, the q_before all-reduce (owner mode),
rlc_shard_finish, end_of_pass_update -- with host-staged collectives (no
kernel waits on the other process).  The bands stitch into the reference's
image and both ranks end with the reference's learned state."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _case():
    from paper_1911_10217_b200 import rlcuts, scenes
    scene = scenes.cornell_grid(2, 1, dome_triangles=64, width=40, height=30)
    cfg = rlcuts.RenderConfig(spp=4, passes=4, sampler=rlcuts.SamplerKind.rl_lightcuts,
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    return scene, cfg


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, outdir: str, owner: bool):
    from paper_1911_10217_b200 import dist as rdist
    from paper_1911_10217_b200 import rlcuts
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    scene, cfg = _case()
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    eng = rdist.GpuEngine(ctx, grid, fb, cfg, torch.device("cuda", 0), world=world)
    frame = rdist.ShardedFrame(eng, scene.camera.height, rank, world, host_staging=True,
                               owner=owner)
    changes = [frame.step(p) for p in range(cfg.passes)]
    s, c = fb.download()
    with open(os.path.join(outdir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump({"rows": frame.rows, "sum": s, "count": c, "changes": changes,
                     "cells": grid.export(), "stats": grid.stats()}, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("owner", [False, True])
def test_two_processes_gloo_match_reference(ref, tmp_path, owner):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), owner), nprocs=world, join=True)
    scene, cfg = _case()
    rr = ref.RefRun(scene, cfg)
    rch = [rr.run_pass(p)[0] for p in range(cfg.passes)]
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    lookups = 0
    for r in range(world):
        out = pickle.load(open(tmp_path / f"rank{r}.pkl", "rb"))
        r0, r1 = out["rows"]
        assert out["changes"] == rch
        assert np.array_equal(out["sum"][r0:r1], rs[r0:r1])
        assert np.array_equal(out["count"][r0:r1], rc[r0:r1])
        assert out["cells"].keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(out["cells"][k][f], v[f])
        lookups += out["stats"]["lookups"]
    assert lookups == rr.stats()["lookups"]
