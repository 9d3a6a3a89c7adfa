"""LiDAR throughput on the GPU box (§8(f) row 4, reading R32): rays/s and sensor scans/s of
gsb_render_lidar on the C3 scene (520 k Gaussians) for several ray patterns, CUDA events on the
render stream, fresh poses per step.  One JSON line per pattern.

   python scripts/lidar_bench.py [envs] [steps] [pattern ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.CONFIGS["C3"]
g = gsb.Scene.from_synth(synth.make_scene(cfg))
poses = [torch.from_numpy(synth.make_poses(cfg, np.arange(B), s)).cuda() for s in range(steps + 2)]
mount = torch.from_numpy(synth.lidar_body_mount()[None].copy()).cuda()
world = torch.from_numpy(synth.lidar_world_sensor(cfg, np.arange(B))[:, None].copy()).cuda()
patterns = {
    "rotating_32x1024_body": (synth.lidar_pattern("rotating", 32, 1024), mount, [0]),
    "rotating_32x1024_world": (synth.lidar_pattern("rotating", 32, 1024), world, None),
    "solid_state_64x256_world": (synth.lidar_pattern("solid_state", 64, 256), world, None),
    "non_repetitive_20000_body": (synth.lidar_pattern("non_repetitive", n_points=20000), mount, [0]),
    "height_scan_11x17_body": (synth.lidar_pattern("height_scan", 11, 17), mount, [0]),
}
only = sys.argv[3:]
for name, (dirs, sx, sb) in patterns.items():
    if only and name not in only:
        continue
    grid = os.environ.get("GSB_LIDAR_GRID")   # "n_az,n_el" override (sweeps)
    lid = gsb.Lidar(g, dirs, *(int(v) for v in grid.split(","))) if grid else gsb.Lidar(g, dirs)
    R = lid.n_rays
    rng = torch.empty((B, 1, R), device="cuda")
    alp = torch.empty((B, 1, R), device="cuda")
    lid.render(poses[0], sx, rng, alp, sensor_body=sb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for s in range(steps):
        lid.render(poses[s + 1], sx, rng, alp, sensor_body=sb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    info = lid.info()
    print(json.dumps({"pattern": name, "envs": B, "rays_per_scan": R, "ms_per_step": ms,
                      "scans_per_s": B / (ms / 1e3), "rays_per_s": B * R / (ms / 1e3),
                      "keys_per_scan": info["keys"] / B, "grid": [info["n_az"], info["n_el"]],
                      "items": info["n_items"], "hit_frac_alpha_gt_0.5": float((alp > 0.5).float().mean())}),
          flush=True)
    lid.close()
