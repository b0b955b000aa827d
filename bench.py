#!/usr/bin/env python
"""Benchmark of the RL-lightcuts direct-lighting path (arXiv 1911.10217).

Metric (BASELINE.json): learnt light samples per second -- each one a cut
sample, a shadow ray and an RL update -- counted exactly like the
reference's RenderResult::lookups (proj/src/hash_grid.cpp:114).

A step is one frame of the configured workload: render_pass (primary ray,
cell hash, cut sample, shadow ray, deferred RL fold, radiance) followed by
end_of_pass_update (split-collapse + cdf rebuild), the real-time temporal
learning loop of config c3 (1 spp per frame).  Inputs (scene, BVH, light
tree, cut tables) are resident in HBM before the timed region; the working
set (~0.5 GB for c3) is larger than L2, so no explicit flush is done.

  python bench.py                       # our B200 path, N=1, config c3
  python bench.py --impl reference      # the reference CPU library arm
  torchrun --nproc-per-node N bench.py --gpus N   # N ranks, screen-band sharded

One JSON line is printed by rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "light samples/sec (sample+shadow ray+RL update)"
UNIT = "light samples/s"
WORKLOADS = {
    "c1": "c1: 1 Cornell box, light tessellated into 1,024 emissive tris, 256x256, "
          "1 spp/frame, base_tile 1/16, M=128",
    "c2": "c2: 4x4 mutually occluding Cornell boxes, 16,384 emissive tris, 1280x720, "
          "4 spp/frame (64 spp over 16 frames), M=128",
    "c3": "c3: procedural maze, 1,000,000 emissive tris, 1920x1080, 1 spp/frame "
          "(64 frames), M=128, hash capacity 65,536",
    "c4": "c4: maze, 65,536 emissive tris displaced every frame (seeded x/z jitter, "
          "scenes.displace_emitters) via rlc_context_update_scene (fresh scene BVH and "
          "emitter records, frozen light tree), 1920x1080, 1 spp/frame, M=128",
}
WORKLOADS["c5"] = ("c5: maze, 4,000,000 emissive tris, 3840x2160, 64 spp in 16 passes "
                   "(4 spp per pass), M=128 (BASELINE's 8-GPU offline case, here on one GPU)")
DYNAMIC = {"c4"}  # workloads whose emitters move every frame


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def make_config(name: str, max_depth: int = 1):
    from paper_1911_10217_b200 import rlcuts, scenes
    scene, st = scenes.config_scene(name)
    cfg = rlcuts.RenderConfig(spp=st["spp"], passes=st["passes"], max_depth=max_depth,
                              sampler=rlcuts.SamplerKind.rl_lightcuts,
                              hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
    return scene, cfg


def workload(args) -> str:
    w = WORKLOADS[args.config]
    return w if args.max_depth == 1 else w + f", max_depth {args.max_depth} (multi-bounce paths)"


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# roofline bookkeeping
# ---------------------------------------------------------------------------
NODE_B, TRI_B = 64, 72  # reference BVH node / Moller-Trumbore triangle bytes
RAY_B, WIDE_NODE_B, TRIACCEL_B = 64, 64, 80  # ShadowRay, quantized 4-wide node, TriAccel


def traversal_stats(name: str) -> dict | None:
    p = os.path.join(ROOT, "profiles", "traversal_stats.json")
    try:
        return json.load(open(p))[name]
    except Exception:
        return None


def measured_peaks() -> tuple[float, str]:
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def frame_hbm(config: str, value: float, peak: float) -> dict | None:
    """Whole-frame HBM traffic (BASELINE's "HBM GB/s"): the DRAM bytes of
    every launch of one steady-state frame per light sample, measured once
    with ncu (profiles/r01_frame_dram_c3.txt), times the live sample rate."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        b = float(json.load(open(p))[config]["frame_bytes_per_sample"])
    except Exception:
        return None
    gbs = value * b / 1e9
    return {"bytes_per_sample": b, "achieved_gbs": gbs, "frac": gbs / peak,
            "source": "ncu DRAM read+write of one frame's launches / its light samples "
                      "(profiles/r01_frame_dram_c3.txt) x this run's light samples/s"}


def ncu_traffic(config: str, kernel: str) -> float | None:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return float(json.load(open(p))[config][kernel])
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference library)
# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_run(scene, cfg, workers: int, min_frames: int, min_seconds: float,
                      max_seconds: float = 1e9, warmup: int = 1, dynamic: bool = False):
    """Times the stock reference render_pass + end_of_pass_update
    (render.cpp:159-200, the loop body of render_frame) on the SAME scene,
    raster and per-frame schedule as our arm, `workers` host threads
    (render.cpp:23-38); frames until both min_frames and min_seconds are
    met (or max_seconds passed).  Dynamic workloads add the per-frame
    context rebuild (build_context with the frozen light tree, the semantics
    of rlc_context_update_scene)."""
    import oracle
    from paper_1911_10217_b200 import rlcuts, scenes
    rcfg = rlcuts.RenderConfig(spp=cfg.spp, passes=cfg.passes, sampler=cfg.sampler, cut=cfg.cut,
                               hash=cfg.hash, seed=cfg.seed, workers=workers,
                               max_depth=cfg.max_depth)
    run = oracle.RefRun(scene, rcfg)

    def update(p):
        if not dynamic or p == 0:
            return 0.0
        s = scenes.displace_emitters(scene, p)
        t0 = time.perf_counter()
        run.update_scene(s)
        return (time.perf_counter() - t0) * 1e3

    for p in range(warmup):
        update(p)
        run.run_pass(p)
    l0 = run.stats()["lookups"]
    total_ms, done = 0.0, 0
    p = warmup
    while True:
        ums = update(p)
        _, ms = run.run_pass(p)
        total_ms += ms + ums
        done += 1
        p += 1
        if done >= min_frames and total_ms / 1e3 >= min_seconds:
            break
        if done >= 1 and total_ms / 1e3 >= max_seconds:
            break
    lookups = run.stats()["lookups"] - l0
    cam = scene.camera
    sample = (f"frames {warmup}..{warmup + done - 1} of the {scene.name} scene at "
              f"{cam.width}x{cam.height} (the same raster and schedule as our arm), "
              f"{lookups} light samples, reference render_pass + end_of_pass_update, "
              f"workers={workers}")
    return lookups / (total_ms / 1e3), sample, total_ms / done, done


def run_reference_arm(args, rank: int, world: int):
    """The reference's own CPU implementation of the path (oracle/_ref: the
    unmodified library, compiled in place) on all host cores, on our arm's
    workload: the same scene, raster and frame schedule.  The timed frames are
    bounded to about a minute of host time."""
    if rank != 0:
        return
    scene, cfg = make_config(args.config, args.max_depth)
    cores = os.cpu_count() or 1
    value, sample, ms_step, done = cpu_reference_run(
        scene, cfg, workers=cores, min_frames=args.steps, min_seconds=0.0,
        max_seconds=args.ref_seconds, warmup=args.warmup, dynamic=args.config in DYNAMIC)
    if done < args.steps:
        sample += f" (the first {done} of the {args.steps} requested frames: time bound)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": done, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload(args)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch

    from paper_1911_10217_b200 import rlcuts

    dist = None
    # one process per GPU; with fewer GPUs than ranks (--dist-backend gloo
    # functional runs only) ranks share devices round-robin
    local_rank = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")

    scene, cfg = make_config(args.config, args.max_depth)
    t0 = time.perf_counter()
    ctx = rlcuts.build_context(scene, cfg, device=local_rank)
    build_s = time.perf_counter() - t0
    grid = rlcuts.HashGrid(ctx, cfg)
    fb = rlcuts.Framebuffer(ctx)
    H = scene.camera.height
    # dynamic workloads: the per-frame scenes are inputs, built before timing
    dynamic = args.config in DYNAMIC
    from paper_1911_10217_b200 import scenes as scn
    frames = ([scn.displace_emitters(scene, p) for p in range(args.warmup + args.steps)]
              if dynamic else None)
    update_ms = [0.0]

    # the scenes of the next frames are prepared ahead (their host builds run
    # beside this frame's GPU work and each other: rlc_context_prepare_scene)
    ahead, tokens = max(0, args.scene_ahead), {}

    def update(p):
        if dynamic and p > 0:
            t = time.perf_counter()
            for q in range(p, p + ahead + 1):
                if q not in tokens:
                    tokens[q] = ctx.prepare_scene(frames[q % len(frames)])
            ctx.commit_scene(tokens.pop(p))
            update_ms[0] += (time.perf_counter() - t) * 1e3

    if world == 1:
        r0, r1 = 0, H
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)

        def step(p):
            update(p)
            rlcuts.render_pass(ctx, cfg, p, grid, fb, sync=False)
            rlcuts.end_of_pass_update(grid, ctx, cfg.cut, sync=False)
    else:
        # screen bands with the exact record exchange: over the
        # C++ NCCL data plane (one rlc_shard_frame call per frame, owner-folded
        # cells, no host synchronization), or over gloo with host staging
        from paper_1911_10217_b200 import dist as rdist
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)
        eng = rdist.GpuEngine(ctx, grid, fb, cfg, torch.device("cuda", local_rank), world=world)
        if args.dist_backend == "nccl":
            frame = rdist.NcclFrame(eng, H, rank, world, local_rank, owner=not args.replicated_fold,
                                    peer=args.peer_exchange)
        else:
            frame = rdist.ShardedFrame(eng, H, rank, world, host_staging=True,
                                       owner=not args.replicated_fold)
        r0, r1 = frame.rows

        def step(p):
            update(p)
            frame.step(p)

    # multi-GPU over NCCL, static scene: the frames replay a captured CUDA
    # graph of two sharded frames (kernels and collectives; rlc_shard_frames)
    graphed = world > 1 and args.dist_backend == "nccl" and not dynamic
    if graphed:
        frame.run(0, args.warmup, graph=True)
    else:
        for p in range(args.warmup):
            step(p)
    update_ms[0] = 0.0
    ctx.synchronize()
    ctx.stage_times()
    # single GPU, static scene: the timed frames are one render_passes call
    # (render_frame's pass loop; CUDA-graph replays for launch-bound frames),
    # the per-kernel CUDA-event times come from a separate untimed run below
    batch = world == 1 and not dynamic
    ctx.enable_timing(False)
    l0 = grid.lookup_count()
    ins0 = grid.insertion_stats()
    launches0 = rlcuts.kernel_launches()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if batch:
        rlcuts.render_passes(ctx, cfg, args.warmup, args.steps, grid, fb)
    elif graphed:
        frame.run(args.warmup, args.steps, graph=True)
    else:
        for p in range(args.warmup, args.warmup + args.steps):
            step(p)
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    update_timed_ms = update_ms[0]
    launches = rlcuts.kernel_launches() - launches0
    ms = e0.elapsed_time(e1)
    lookups = grid.lookup_count() - l0
    ins1 = grid.insertion_stats()
    grid_insert_stats = {f"{k}_per_frame": (ins1[k] - ins0[k]) / args.steps for k in ins1}
    # per-kernel times and work counts: a few more frames with CUDA events
    # around every stage and k_shadow counting its work
    stage_frames = min(args.steps, 20)
    ctx.stage_times()
    ctx.enable_timing(True)
    ctx.count_work(True)
    l_st = grid.lookup_count()
    rlcuts.work_counters(reset=True)
    for p in range(args.warmup + args.steps, args.warmup + args.steps + stage_frames):
        step(p)
    ctx.synchronize()
    work = rlcuts.work_counters(reset=True)
    stage_lookups = grid.lookup_count() - l_st
    ctx.count_work(False)
    stages = ctx.stage_times()
    ctx.enable_timing(False)
    if dist is not None:
        t = torch.tensor([ms, float(lookups)], dtype=torch.float64,
                         device="cuda" if args.dist_backend == "nccl" else "cpu")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, lookups = float(mx[0]), int(sm[1])
    value = lookups / (ms / 1e3)
    st = grid.stats()

    # roofline of the dominant kernel (k_shadow): its own work this run --
    # rays, node steps, triangle tests from the always-on work counters over
    # the timed frames -- in bytes, over its CUDA-event launch time, against
    # the measured HBM copy bandwidth and the measured L2 read bandwidth
    peak, peak_src = measured_peaks()
    l2_gbs = rlcuts.measure_l2_bandwidth(local_rank)
    k_ms, k_n = stages["shadow"]
    roof = None
    if k_n > 0 and work["shadow_rays"] > 0:
        t_launch = k_ms / k_n / 1e3
        rays = work["shadow_rays_queued"] / stage_frames
        nodes = work["shadow_nodes"] / stage_frames
        tris = work["shadow_tris"] / stage_frames
        own = rays * (RAY_B + 4) + nodes * WIDE_NODE_B + tris * TRIACCEL_B
        achieved = own / t_launch / 1e9
        tr = ncu_traffic(args.config, "shadow")
        roof = {"bound": "hbm", "kernel": "k_shadow", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                "traffic": tr, "unit_of_work": "shadow ray",
                "bytes_per_unit": own / rays, "units_per_launch": rays,
                "avg_launch_ms": k_ms / k_n,
                "own_work": {"node_steps_per_ray": nodes / rays, "tri_tests_per_ray": tris / rays,
                             "rays_past_root_per_ray": work["shadow_rays"] / stage_frames / rays,
                             "rays_per_light_sample": rays / (stage_lookups / stage_frames),
                             "bytes": f"{RAY_B + 4} per ray (record + order) + {WIDE_NODE_B} per "
                                      f"node step + {TRIACCEL_B} per triangle test",
                             "source": "rlc_work_counters over the stage-timing frames "
                                       "(k_shadow's counting instance, the launches timed)"},
                "l2": {"peak": l2_gbs, "frac": achieved / l2_gbs if l2_gbs else None,
                       "peak_source": "measured here (rlc_measure_l2_bandwidth: 16-byte .cg "
                                      "loads over a 48 MB L2-resident buffer)"},
                "limiter": "latency of dependent node loads (L1/L2-served): ncu issue-active "
                           "~32%, ~18 of 32 lanes active per instruction "
                           "(profiles/r01_ncu_summary.md); HBM and L2 fractions are both low"}
        if tr:
            roof["dram_achieved"] = tr / t_launch / 1e9
            roof["dram_frac"] = roof["dram_achieved"] / peak
        trav = traversal_stats(args.config)
        if trav is not None:  # the reference BVH's traversal work, per ray
            ref_b = 64 + NODE_B * trav["shadow_nodes"] + TRI_B * trav["shadow_tris"] + 12
            roof["reference_equivalent"] = {
                "bytes_per_ray": ref_b, "gbs": ref_b * rays / t_launch / 1e9,
                "note": "work-normalised speed: the reference BVH's node and triangle "
                        "bytes per ray (SURVEY 8(d)) / our launch time; not a roofline "
                        "fraction (our tree does far less work per ray)"}
        fh = frame_hbm(args.config, value, peak) if args.max_depth == 1 else None
        if fh:
            roof["frame_hbm"] = fh

    # end to end through the C-ABI render_frame: host image out, grid created
    # inside the call (the reference's render_frame, render.cpp:202-240)
    e2e = None
    if not args.no_e2e and world == 1 and dynamic:
        # the public API per frame: update_scene (the frame's scene, host ->
        # device), render_pass, end_of_pass_update, the frame's light-sample
        # count read back (device -> host)
        g2, f2 = rlcuts.HashGrid(ctx, cfg), rlcuts.Framebuffer(ctx)
        ctx.set_stream(None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for q in sorted(tokens):  # scenes still prepared ahead by the loops above
            ctx.commit_scene(tokens.pop(q))
        toks = {}
        for p in range(args.steps):
            for q in range(p, p + ahead + 1):
                if q not in toks:
                    toks[q] = ctx.prepare_scene(frames[q % len(frames)])
            ctx.commit_scene(toks.pop(p))
            rlcuts.render_pass(ctx, cfg, p, g2, f2, sync=False)
            rlcuts.end_of_pass_update(g2, ctx, cfg.cut, sync=False)
            n_done = g2.lookup_count()
        wall = time.perf_counter() - t0
        ntri = scene.num_triangles
        e2e = {"value": n_done / wall, "unit": UNIT,
               "h2d_bytes_per_step": 76 * ntri + 48 * scene.materials.shape[0] + 128,
               "d2h_bytes_per_step": 8, "wall_ms": wall * 1e3,
               "call": "rlc_context_prepare_scene (frames ahead) + rlc_context_commit_scene + "
                    "rlc_render_pass + rlc_end_of_pass_update"}
    elif not args.no_e2e and world == 1:
        ecfg = rlcuts.RenderConfig(spp=args.steps * (cfg.spp // cfg.passes), passes=args.steps,
                                   sampler=cfg.sampler, cut=cfg.cut, hash=cfg.hash,
                                   seed=cfg.seed + 1, max_depth=cfg.max_depth)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = rlcuts.render_frame(ctx, ecfg)
        wall = time.perf_counter() - t0
        npix = scene.camera.width * scene.camera.height
        e2e = {"value": res.lookups / wall, "unit": UNIT,
               "h2d_bytes_per_step": (176 + 28 * st["cut_size"]) / args.steps,
               "d2h_bytes_per_step": (24 * npix + 4 * args.steps + 32) / args.steps,
               "wall_ms": wall * 1e3, "call": "rlc_render_frame"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        try:
            v, sample, _, _ = cpu_reference_run(
                scene, cfg, workers=cores, min_frames=2, min_seconds=args.cpu_seconds,
                dynamic=dynamic)
            v1, sample1, _, _ = cpu_reference_run(
                scene, cfg, workers=1, min_frames=1, min_seconds=0.0, dynamic=dynamic)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": sample, "cpu_model": cpu_model(), "same_config": True,
                   "workers_1": {"value": v1, "cores": 1, "sample": sample1}}
        except Exception as ex:  # the reference library is test infrastructure
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args),
                       "frames_timed": args.steps,
                       "l2": "no flush: resident scene+cut+pass buffers exceed the 126 MB L2",
                       "parallelism": (f"screen bands x{world}, exact update-record all-gather "
                                       f"over {args.dist_backend}, "
                                       f"{'replicated' if args.replicated_fold else 'owner'}-folded"
                                       + (", peer-memory record exchange" if args.peer_exchange else "")
                                       + (", CUDA-graph replay" if graphed else "")
                                       if world > 1 else "single GPU"),
                       "cells": st["occupied"], "fallback_hits": st["fallback_hits"],
                       **grid_insert_stats},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
            "stage_ms_per_step": {k: v[0] / stage_frames for k, v in stages.items()},
            "stage_source": "CUDA events around every stage in %d further frames" % stage_frames,
            "scene_update_ms_per_step": update_timed_ms / args.steps if dynamic else None,
            "context_build_s": build_s,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--max-depth", type=int, default=1,
                    help="path vertices per sample (render.hpp:20); 1 = the headline direct lighting")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: bound on the timed host time")
    ap.add_argument("--peer-exchange", action="store_true",
                    help="N > 1 over NCCL: records stored straight into every rank's receive "
                         "buffer over NVLink (CUDA IPC) instead of ncclAllGather")
    ap.add_argument("--scene-ahead", type=int, default=3,
                    help="dynamic workloads: frames whose scenes are prepared ahead")
    ap.add_argument("--replicated-fold", action="store_true",
                    help="N > 1: every rank folds every record (default: the cell's owner folds)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo stages the record exchange through host memory (functional "
                         "multi-rank runs with fewer GPUs than ranks)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 warm-up steps
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
