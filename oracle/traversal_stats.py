"""TEST INFRASTRUCTURE: measures, with the CPU restatement (reference BVH,
reference traversal order), the mean traversal work per ray of each bench
configuration and writes profiles/traversal_stats.json.  bench.py turns
these into the algorithmic bytes of the visibility kernels.

    python -m oracle.traversal_stats [--passes 4]
"""
import argparse
import json
import os

from paper_1911_10217_b200 import rlcuts, scenes
from oracle.restate import OracleRun

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOWNSCALE = {"c1": 1, "c2": 2, "c3": 4, "c4": 4, "c5": 8}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--passes", type=int, default=4)
    ap.add_argument("--only", nargs="*", default=None, help="configurations to (re)measure")
    args = ap.parse_args()
    path = os.path.join(ROOT, "profiles", "traversal_stats.json")
    out = json.load(open(path)) if args.only and os.path.exists(path) else {}
    for name, ds in DOWNSCALE.items():
        if args.only and name not in args.only:
            continue
        scene, st = scenes.config_scene(name)
        scene = scene.with_resolution(scene.camera.width // ds, scene.camera.height // ds)
        spp_pp = st["spp"] // st["passes"]
        cfg = rlcuts.RenderConfig(spp=spp_pp * args.passes, passes=args.passes,
                                  sampler=rlcuts.SamplerKind.rl_lightcuts,
                                  hash=rlcuts.HashConfig(base_tile=st["base_tile"]))
        run = OracleRun(scene, cfg)
        for p in range(args.passes):
            run.run_pass(p)
        t = run.trav_stats()
        s = run.stats()
        t["lookups"] = s["lookups"]
        t["shadow_rays_per_sample"] = t["shadow_rays"] / max(s["lookups"], 1)
        t["samples_per_path"] = s["lookups"] / max(t["primary_rays"], 1)
        t["measured_at"] = f"{scene.camera.width}x{scene.camera.height}, {args.passes} passes"
        out[name] = t
        print(name, t)
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
