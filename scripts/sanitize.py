"""Small renders for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402

for name in ("T1", "T6", "T3"):
    cfg = synth.CONFIGS[name]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(cfg.n_envs, cfg.n_cams, cfg.width, cfg.height)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    rgb = torch.zeros((B, C, 3, H, W), device="cuda")
    dep = torch.zeros((B, C, H, W), device="cuda")
    alp = torch.zeros((B, C, H, W), device="cuda")
    nev = torch.zeros((B, C, H, W), dtype=torch.int32, device="cuda")
    g.render(torch.from_numpy(b.poses).cuda(), torch.from_numpy(b.intrinsics).cuda(), torch.from_numpy(b.w2c).cuda(),
             gsb.RenderParams(W, H, stats=True), rgb, dep, alp, nev)
    torch.cuda.synchronize()
    print(name, "ok", g.stats(), float(rgb.mean()))

# LiDAR (reading R32) and the standalone encoder with motion blur (reading R33)
cfg = synth.CONFIGS["T1"]
sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
g = gsb.Scene.from_synth(sc)
for pat in (synth.lidar_pattern("rotating", 8, 64), synth.lidar_pattern("solid_state", 8, 32)):
    lid = gsb.Lidar(g, pat)
    B = cfg.n_envs
    rr = torch.zeros((B, 2, lid.n_rays), device="cuda")
    ra = torch.zeros((B, 2, lid.n_rays), device="cuda")
    sx = np.stack([synth.lidar_world_sensor(cfg, np.arange(B)),
                   np.broadcast_to(synth.lidar_body_mount(), (B, 3, 4))], 1).astype(np.float32).copy()
    lid.render(torch.from_numpy(b.poses).cuda(), torch.from_numpy(sx).cuda(), rr, ra, sensor_body=[-1, 0])
    torch.cuda.synchronize()
    print("lidar ok", lid.info(), float(ra.mean()))
    lid.close()
rgb = torch.rand((2, 2, 3, 33, 47), device="cuda")
dep = torch.rand((2, 2, 33, 47), device="cuda")
out8 = torch.zeros((2, 2, 3, 33, 47), dtype=torch.uint8, device="cuda")
od = torch.zeros((2, 2, 33, 47), dtype=torch.float16, device="cuda")
blur = torch.tensor([[[5, -3], [0, 0]], [[-9, 2], [70, 1]]], dtype=torch.int32, device="cuda")
gsb.obs_encode(rgb, out8, depth=dep, out_depth=od, blur=blur)
torch.cuda.synchronize()
print("encode ok", int(out8.float().mean()))

# static-camera merge with per-env pre-binned cameras (GSB_FLAG_STATIC_PER_ENV)
cfg = synth.CONFIGS["T2"]
sc = synth.make_scene(cfg)
B = cfg.n_envs
K, Wc = synth.make_cameras(cfg, np.arange(B))
g = gsb.Scene.from_synth(sc)
g.prebin_static(K[:, 0].copy(), Wc[:, 0].copy(), gsb.RenderParams(cfg.width, cfg.height))
g.reserve(B, 1, cfg.width, cfg.height)
rgb = torch.zeros((B, 1, 3, cfg.height, cfg.width), device="cuda")
g.render_static(torch.from_numpy(synth.make_poses(cfg, np.arange(B), 1)).cuda(),
                gsb.RenderParams(cfg.width, cfg.height, static_per_env=True), rgb)
torch.cuda.synchronize()
print("static per-env ok", float(rgb.mean()))
