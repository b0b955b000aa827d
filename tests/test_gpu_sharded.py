"""GPU: the sharded pass (rlc_shard_trace / _fold / _finish) with N ranks
emulated as N contexts on one device and a host-driven exchange (no kernel
waits on another rank) must reproduce the single-context pass and the
reference bit for bit, with the fold replicated on every rank or done by the
owner of each cell (also on c3 over 8 ranks); the NCCL data plane
(rlc_shard_frame, and its CUDA-graph replay) at one rank."""
import numpy as np
import pytest
import torch

from paper_1911_10217_b200 import dist as rdist
from paper_1911_10217_b200 import rlcuts, scenes

pytestmark = pytest.mark.gpu
RL = rlcuts.SamplerKind.rl_lightcuts


@pytest.mark.parametrize("owner", [False, True])
@pytest.mark.parametrize("world,depth", [(1, 1), (2, 1), (3, 1), (2, 3), (4, 1)])
def test_sharded_gpu_matches_single(ref, world, depth, owner):
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, max_depth=depth,
                              cut=rlcuts.CutConfig(cut_size=64, split_threshold=2.0))
    dev = torch.device("cuda", 0)
    engines = []
    for r in range(world):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev))
    rows = [rdist.band(scene.camera.height, r, world) for r in range(world)]
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        changes = rdist.local_exchange(engines, rows, p, owner)
        rch, _ = rr.run_pass(p)
        assert changes == [rch] * world
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    lookups = 0
    for e, (r0, r1) in zip(engines, rows):
        s, c = e.fb.download()
        assert np.array_equal(s[r0:r1], rs[r0:r1]) and np.array_equal(c[r0:r1], rc[r0:r1])
        cells = e.grid.export()
        assert cells.keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(cells[k][f], v[f])
        lookups += e.grid.lookup_count()
    assert lookups == rr.stats()["lookups"]


@pytest.mark.parametrize("world,owner,capacity,depth", [(2, True, 1 << 16, 1),
                                                        (3, False, 1 << 16, 1),
                                                        (3, True, 200, 1), (2, True, 1 << 16, 3)])
def test_sharded_peer_exchange(ref, world, owner, capacity, depth):
    """The peer exchange's data path: every rank stores its band's records
    straight into every rank's receive buffer (rlc_shard_trace_to; buffers
    kept across passes, so stale records past a block's count must be
    ignored) and folds its own -- equal to the reference."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, max_depth=depth,
                              hash=rlcuts.HashConfig(capacity=capacity, probe_limit=16),
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    dev = torch.device("cuda", 0)
    engines = []
    for r in range(world):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev, world=world))
    rows = [rdist.band(scene.camera.height, r, world) for r in range(world)]
    nbytes = world * 32 * (engines[0].cap + 1)
    bufs = [torch.full((nbytes,), 0x5A, dtype=torch.uint8, device=dev) for _ in range(world)]
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        changes = rdist.local_exchange(engines, rows, p, owner, peer_buffers=bufs)
        rch, _ = rr.run_pass(p)
        assert changes == [rch] * world
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    for e, (r0, r1) in zip(engines, rows):
        s, c = e.fb.download()
        assert np.array_equal(s[r0:r1], rs[r0:r1]) and np.array_equal(c[r0:r1], rc[r0:r1])
        cells = e.grid.export()
        assert cells.keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(cells[k][f], v[f])
        assert [(s_, k) for s_, _, k, _ in e.grid.slots()] == rr.slots()


@pytest.mark.parametrize("world,capacity,depth", [(2, 1 << 16, 1), (3, 1 << 16, 1), (3, 200, 1),
                                                  (2, 1 << 16, 3)])
def test_sharded_entry_exchange(ref, monkeypatch, world, capacity, depth):
    """Owner mode's entry exchange (each entry's final q and record count
    summed over the ranks, q_before per band) -- chosen for passes whose
    records far outnumber the cut entries, forced here -- equals the
    reference, also with an overflowing table."""
    monkeypatch.setenv("RLC_SHARD_ENTRY", "1")
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, max_depth=depth,
                              hash=rlcuts.HashConfig(capacity=capacity, probe_limit=16),
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    dev = torch.device("cuda", 0)
    engines = []
    for r in range(world):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev))
    rows = [rdist.band(scene.camera.height, r, world) for r in range(world)]
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        changes = rdist.local_exchange(engines, rows, p, owner=True)
        assert rlcuts.shard_entry_arrays(engines[0].ctx)[2] == capacity * 32
        rch, _ = rr.run_pass(p)
        assert changes == [rch] * world
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    for e, (r0, r1) in zip(engines, rows):
        s, c = e.fb.download()
        assert np.array_equal(s[r0:r1], rs[r0:r1]) and np.array_equal(c[r0:r1], rc[r0:r1])
        cells = e.grid.export()
        assert cells.keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(cells[k][f], v[f])
        assert [(s_, k) for s_, _, k, _ in e.grid.slots()] == rr.slots()


@pytest.mark.parametrize("entry", ["0", "1"])
def test_sharded_c3_eight_ranks_owner(ref, monkeypatch, entry):
    """The headline scene (1M emitters) at 320 x 180 over 8 emulated ranks,
    owner-partitioned, per-slot and per-entry exchange: 6 frames of bands,
    exchange, insertion and fold equal the reference's single-process
    frames."""
    monkeypatch.setenv("RLC_SHARD_ENTRY", entry)
    scene, st = scenes.config_scene("c3")
    scene = scene.with_resolution(320, 180)
    cfg = rlcuts.RenderConfig(spp=6, passes=6, sampler=RL,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    world = 8
    dev = torch.device("cuda", 0)
    engines = []
    for r in range(world):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev, world=world))
    rows = [rdist.band(scene.camera.height, r, world) for r in range(world)]
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        changes = rdist.local_exchange(engines, rows, p, owner=True)
        rch, _ = rr.run_pass(p)
        assert changes == [rch] * world
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    for e, (r0, r1) in zip(engines, rows):
        s, c = e.fb.download()
        assert np.array_equal(s[r0:r1], rs[r0:r1]) and np.array_equal(c[r0:r1], rc[r0:r1])
    for e in (engines[0], engines[-1]):
        cells = e.grid.export()
        assert cells.keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(cells[k][f], v[f])
        assert [(s_, k) for s_, _, k, _ in e.grid.slots()] == rr.slots()


@pytest.mark.parametrize("owner", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_overflow_matches_reference(ref, world, owner):
    """A hash table too small for the scene: every rank inserts the new keys
    of all ranks' records in canonical order, so the refused keys, the slot
    layout and the learned state equal the single-GPU reference's."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL,
                              hash=rlcuts.HashConfig(capacity=200, probe_limit=16),
                              cut=rlcuts.CutConfig(cut_size=32, split_threshold=2.0))
    dev = torch.device("cuda", 0)
    engines = []
    for r in range(world):
        ctx = rlcuts.build_context(scene, cfg)
        engines.append(rdist.GpuEngine(ctx, rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx),
                                       cfg, dev))
    rows = [rdist.band(scene.camera.height, r, world) for r in range(world)]
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        changes = rdist.local_exchange(engines, rows, p, owner)
        rch, _ = rr.run_pass(p)
        assert changes == [rch] * world
    rs, rc = rr.framebuffer()
    rcells = rr.export()
    fallback = 0
    for e, (r0, r1) in zip(engines, rows):
        s, c = e.fb.download()
        assert np.array_equal(s[r0:r1], rs[r0:r1]) and np.array_equal(c[r0:r1], rc[r0:r1])
        cells = e.grid.export()
        assert cells.keys() == rcells.keys()
        for k, v in rcells.items():
            for f in v:
                assert np.array_equal(cells[k][f], v[f])
        assert [(s_, k) for s_, _, k, _ in e.grid.slots()] == rr.slots()
        fallback += e.grid.fallback_hits()
    assert fallback == rr.stats()["fallback_hits"] > 100


@pytest.mark.parametrize("owner", [False, True])
def test_nccl_frame_one_rank_matches_render_pass(ref, owner):
    """rlc_shard_frame through a real one-rank NCCL communicator (all-gather
    and all-reduce on the context stream) equals render_pass + end_of_pass."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=RL,
                              cut=rlcuts.CutConfig(cut_size=64, split_threshold=2.0))
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    eng = rdist.GpuEngine(ctx, grid, fb, cfg, torch.device("cuda", 0))
    frame = rdist.NcclFrame(eng, scene.camera.height, 0, 1, 0, owner)
    rr = ref.RefRun(scene, cfg)
    for p in range(cfg.passes):
        frame.step(p)
        rr.run_pass(p)
    rlcuts.shard_sync(ctx, grid)
    s, c = fb.download()
    rs, rc = rr.framebuffer()
    assert np.array_equal(s, rs) and np.array_equal(c, rc)
    cells, rcells = grid.export(), rr.export()
    assert cells.keys() == rcells.keys()
    for k, v in rcells.items():
        for f in v:
            assert np.array_equal(cells[k][f], v[f])
    assert grid.stats() == rr.stats()


@pytest.mark.parametrize("peer", [False, True])
def test_nccl_peer_exchange_one_rank(ref, peer):
    """rlc_shard_frame over a one-rank communicator with the peer exchange
    (records stored into the IPC-exported receive buffer, two halves by pass
    parity) equals the reference, frame by frame and from a CUDA graph."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=7, passes=7, sampler=RL,
                              cut=rlcuts.CutConfig(cut_size=64, split_threshold=2.0))
    ctx = rlcuts.build_context(scene, cfg)
    grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
    eng = rdist.GpuEngine(ctx, grid, fb, cfg, torch.device("cuda", 0))
    frame = rdist.NcclFrame(eng, scene.camera.height, 0, 1, 0, True, peer=True)
    rr = ref.RefRun(scene, cfg)
    frame.step(0)
    frame.run(1, cfg.passes - 1, graph=peer)
    for p in range(cfg.passes):
        rr.run_pass(p)
    rlcuts.shard_sync(ctx, grid)
    s, c = fb.download()
    rs, rc = rr.framebuffer()
    assert np.array_equal(s, rs) and np.array_equal(c, rc)
    cells, rcells = grid.export(), rr.export()
    assert cells.keys() == rcells.keys()
    for k, v in rcells.items():
        for f in v:
            assert np.array_equal(cells[k][f], v[f])


@pytest.mark.parametrize("owner,entry", [(True, "0"), (False, "0"), (True, "1")])
def test_nccl_frames_graph_replay_bit_exact(monkeypatch, owner, entry):
    """rlc_shard_frames replaying a captured CUDA graph of two sharded frames
    (NCCL collectives inside) equals the same frames enqueued one by one
    (owner mode also with the entry exchange)."""
    monkeypatch.setenv("RLC_SHARD_ENTRY", entry)
    scene = scenes.cornell_grid(2, 1, dome_triangles=128, width=48, height=36)
    cfg = rlcuts.RenderConfig(spp=9, passes=9, sampler=RL,
                              cut=rlcuts.CutConfig(cut_size=64, split_threshold=2.0))
    out = []
    for graph in (False, True):
        ctx = rlcuts.build_context(scene, cfg)
        grid, fb = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
        eng = rdist.GpuEngine(ctx, grid, fb, cfg, torch.device("cuda", 0))
        frame = rdist.NcclFrame(eng, scene.camera.height, 0, 1, 0, owner)
        frame.run(0, 4, graph)
        frame.run(4, cfg.passes - 4, graph)  # a second replay run of the cached graph
        rlcuts.shard_sync(ctx, grid)
        out.append((fb.download(), grid.export(), grid.stats()))
    (s0, c0), cells0, st0 = out[0]
    (s1, c1), cells1, st1 = out[1]
    assert np.array_equal(s0, s1) and np.array_equal(c0, c1) and st0 == st1
    assert cells0.keys() == cells1.keys()
    for k, v in cells0.items():
        for f in v:
            assert np.array_equal(cells1[k][f], v[f])
