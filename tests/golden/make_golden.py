"""Generates tests/golden/*.npz from the compiled reference (oracle/_ref), in
this container where /root/reference is mounted:

    make -C oracle ref && python tests/golden/make_golden.py

Every vector comes from the reference's own functions called through
oracle/ref_capi.cpp; the fixtures travel with the repo so the GPU box (which
has no /root/reference) can check against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import RefRun, ref_lib  # noqa: E402
from oracle.restate import unit_api  # noqa: E402
from paper_1911_10217_b200 import rlcuts, scenes  # noqa: E402

RL = rlcuts.SamplerKind.rl_lightcuts


def line_tree(n, energy=None):
    c = np.stack([np.arange(n, dtype=float), np.zeros(n), np.zeros(n)], 1)
    e = np.ones(n) if energy is None else np.asarray(energy, float)
    return c, e


def units(ref):
    out = {}
    rng = np.random.default_rng(1234)
    # light trees on random emitters (test_light_tree.cpp:114-153 style)
    for k, n in enumerate([1, 2, 5, 17, 100, 257]):
        c = rng.uniform(-3, 3, (n, 3))
        e = rng.uniform(0.1, 2.0, n)
        order, nodes, en = ref["light_tree"](c, e)
        out[f"lt{k}_c"], out[f"lt{k}_e"] = c, e
        out[f"lt{k}_order"], out[f"lt{k}_nodes"], out[f"lt{k}_energy"] = order, nodes, en
    # split-collapse fuzz (test_cut.cpp:337-358 style)
    for k in range(40):
        n = int(4 + rng.integers(0, 124))
        c, e = line_tree(n, rng.uniform(0.5, 2.0, n))
        m = int(2 + rng.integers(0, 31))
        cut = ref["init_cut"](c, e, m)
        q = cut["eps_q"] + rng.uniform(0, 3, len(cut["q"]))
        thr = 0.5 + rng.uniform(0, 4)
        it = int(1 + rng.integers(0, 7))
        ch, res = ref["split_collapse"](c, e, m, q, thr, it)
        out[f"sc{k}_c"], out[f"sc{k}_e"], out[f"sc{k}_q_in"] = c, e, q
        out[f"sc{k}_args"] = np.array([m, thr, it, ch], float)
        for f in ("node_ids", "ends", "q", "cdf", "visits"):
            out[f"sc{k}_{f}"] = res[f]
    # update_q sequences (cut.cpp:76-86), fixed and harmonic
    for k, sched in enumerate([0, 1, 0, 1]):
        m = 8
        q0 = rng.uniform(0.01, 1.0, m)
        v0 = np.ones(m, np.uint32)
        s = rng.integers(0, m, 500).astype(np.uint32)
        v = np.where(rng.random(500) < 0.3, 0.0, rng.exponential(2.0, 500))
        q, vis, qb = ref["update_q_seq"](q0, v0, 1e-4 / m, 0.2 if k < 2 else 0.7, sched, s, v)
        out[f"uq{k}_in"] = np.concatenate([q0, [sched, 0.2 if k < 2 else 0.7]])
        out[f"uq{k}_s"], out[f"uq{k}_v"] = s, v
        out[f"uq{k}_q"], out[f"uq{k}_visits"], out[f"uq{k}_qb"] = q, vis, qb
    # sample_cluster with boundary targets (cut.cpp:97-106)
    q = rng.uniform(0.1, 1.0, 64)
    cdf = np.cumsum(q)
    u = np.concatenate([rng.random(2000), cdf[:-1] / cdf[-1], [0.0, 1.0 - 2 ** -53]])
    s, p = ref["sample_cluster"](q, cdf, u)
    out["cl_q"], out["cl_cdf"], out["cl_u"], out["cl_s"], out["cl_p"] = q, cdf, u, s, p
    # level_for_footprint (hash_grid.cpp:34-44), incl. values near the
    # rounding thresholds r = 2^(k+1/2)
    bt = 0.1
    r = np.concatenate([np.exp(rng.uniform(-5, 14, 3000)),
                        bt * 2.0 ** (np.arange(-2, 18) + 0.5)])
    pdf = 1.0 / (r * bt) ** 2
    out["lv_pdf"], out["lv_out"] = pdf, ref["level_for_footprint"](pdf, bt)
    # make_key + hash_key (hash_grid.cpp:27-100)
    n = 3000
    pos = rng.uniform(-4, 4, (n, 3))
    pos[:500] = np.round(pos[:500] * 4) / 4  # points on cell boundaries
    nrm = rng.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm[:300] = np.eye(3)[rng.integers(0, 3, 300)] * rng.choice([-1.0, 1.0], (300, 1))
    lvl = rng.integers(0, 6, n).astype(np.uint32)
    j1, j2 = rng.random(n), rng.random(n)
    for k, (bits, js) in enumerate([(4, 0.0), (4, 1.0), (6, 0.5)]):
        keys, h = ref["make_key"](pos, nrm, lvl, j1, j2, 0.25, bits, js)
        out[f"mk{k}_keys"], out[f"mk{k}_hash"] = np.array(keys, np.int64), h
    out["mk_pos"], out["mk_nrm"], out["mk_lvl"], out["mk_j1"], out["mk_j2"] = pos, nrm, lvl, j1, j2
    # counter RNG (rng.hpp:26-43)
    out["rng"] = np.stack([ref["rng_draws"](s, a, b, 0, 8) for s, a, b in
                           [(1, 0, 0), (7, 123456, 9), (2**63, 2**40, 3)]])
    return out


def runs():
    """Whole-path reference runs: framebuffer and per-cell cut state."""
    out = {}
    cases = {
        "cornell2": (scenes.cornell_grid(2, 1, dome_triangles=32, width=40, height=30),
                     rlcuts.RenderConfig(spp=4, passes=4, sampler=RL)),
        "c1small": (scenes.config_scene("c1")[0].with_resolution(48, 48),
                    rlcuts.RenderConfig(spp=4, passes=4, sampler=RL,
                                        hash=rlcuts.HashConfig(base_tile=1 / 16))),
        "harmonic": (scenes.cornell_grid(1, 3, dome_triangles=128, width=32, height=32),
                     rlcuts.RenderConfig(spp=6, passes=3, sampler=RL, seed=5,
                                         cut=rlcuts.CutConfig(
                                             cut_size=24, split_threshold=2.0, iterations=2,
                                             alpha_schedule=rlcuts.AlphaSchedule.harmonic))),
        "energy": (scenes.cornell_grid(2, 1, dome_triangles=32, width=32, height=24),
                   rlcuts.RenderConfig(spp=2, passes=1, sampler=rlcuts.SamplerKind.energy)),
        "bounce3": (scenes.cornell_grid(2, 1, dome_triangles=32, width=32, height=24),
                    rlcuts.RenderConfig(spp=4, passes=2, sampler=RL, max_depth=3)),
        "bounce2u": (scenes.cornell_grid(1, 2, dome_triangles=32, width=24, height=24),
                     rlcuts.RenderConfig(spp=2, passes=1, max_depth=2,
                                         sampler=rlcuts.SamplerKind.uniform)),
    }
    for name, (scene, cfg) in cases.items():
        r = RefRun(scene, cfg)
        ch = [r.run_pass(p)[0] for p in range(cfg.passes)]
        s, c = r.framebuffer()
        out[f"{name}_sum"], out[f"{name}_count"] = s, c
        out[f"{name}_changes"] = np.array(ch, np.int64)
        st = r.stats()
        out[f"{name}_stats"] = np.array([st["occupied"], st["lookups"], st["fallback_hits"]])
        if cfg.sampler == RL:
            cells = r.export()
            keys = sorted(cells)
            out[f"{name}_keys"] = np.array(keys, np.int64)
            for f in ("node_ids", "ends", "q", "cdf", "visits"):
                out[f"{name}_{f}"] = np.stack([cells[k][f] for k in keys])
    return out


def main():
    ref = unit_api(ref_lib(), "ref")
    np.savez_compressed(os.path.join(HERE, "units.npz"), **units(ref))
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **runs())
    for f in ("units.npz", "runs.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
