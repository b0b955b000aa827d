"""CPU, world_size 2 over gloo: the screen-band sharded pass with the exact
record exchange (paper_1911_10217_b200/dist.py), driven over the oracle
engine, must reproduce the single-process pass bit for bit: every rank ends
with the same cut table, the bands stitch into the same framebuffer, and the
split-collapse counts agree."""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.restate import OracleRun
from paper_1911_10217_b200 import dist as rdist
from paper_1911_10217_b200 import rlcuts, scenes

RL = rlcuts.SamplerKind.rl_lightcuts


def _case(depth=1):
    scene = scenes.cornell_grid(2, 1, dome_triangles=32, width=36, height=27)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, max_depth=depth,
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    return scene, cfg


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, outdir: str, depth: int):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    scene, cfg = _case(depth)
    run = OracleRun(scene, cfg)
    frame = rdist.OracleFrame(rdist.OracleEngine(run), scene.camera.height, rank, world)
    changes = [frame.step(p) for p in range(cfg.passes)]
    s, c = run.framebuffer()
    with open(os.path.join(outdir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump({"rows": frame.rows, "sum": s, "count": c, "changes": changes,
                     "cells": run.export(), "stats": run.stats()}, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,depth", [(2, 1), (3, 1), (2, 3)])
def test_sharded_oracle_matches_single_process(tmp_path, world, depth):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), depth), nprocs=world, join=True)
    scene, cfg = _case(depth)
    single = OracleRun(scene, cfg)
    ref_changes = [single.run_pass(p) for p in range(cfg.passes)]
    ref_sum, ref_count = single.framebuffer()
    ref_cells = single.export()
    lookups = 0
    for r in range(world):
        out = pickle.load(open(tmp_path / f"rank{r}.pkl", "rb"))
        r0, r1 = out["rows"]
        assert np.array_equal(out["sum"][r0:r1], ref_sum[r0:r1])
        assert np.array_equal(out["count"][r0:r1], ref_count[r0:r1])
        assert out["count"][:r0].sum() == 0 and out["count"][r1:].sum() == 0
        assert out["changes"] == ref_changes
        assert out["cells"].keys() == ref_cells.keys()
        for k, v in ref_cells.items():
            for f in v:
                assert np.array_equal(out["cells"][k][f], v[f]), (r, k, f)
        lookups += out["stats"]["lookups"]
    assert lookups == single.stats()["lookups"]


def test_band_partition_covers_rows():
    for h in (1, 7, 1080):
        for w in (1, 2, 3, 8):
            bands = [rdist.band(h, r, w) for r in range(w)]
            assert bands[0][0] == 0 and bands[-1][1] == h
            assert all(bands[i][1] == bands[i + 1][0] for i in range(w - 1))
