"""Small renders for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402

for name in ("T1", "T6", "T3", "T1-masked"):
    # T1-masked: K4b block masks forced on (they serve long-list passes only by default)
    os.environ["GSB_MASK_MIN_AVG"] = "0" if name.endswith("masked") else "512"
    cfg = synth.CONFIGS[name.split("-")[0]]
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

# keys carrying record slots with equal-depth runs (in-place run sort and the re-keyed fallback),
# on the split (K4a) and the fused (K4) path, incl. > 1024 tied keys in a tile (HBM sort)
import os  # noqa: E402
sys.path.insert(0, "tests")
from helpers import identity_cam, scene_from  # noqa: E402
for n, spread, layers, size in ((600, 0.25, 1, 128), (400, 0.3, 40, 128), (2500, 0.05, 1, 128), (3000, 0.3, 25, 32)):
    rng = np.random.default_rng(n + layers)
    z = 2.0 + 0.05 * rng.integers(0, layers, n)
    means = np.stack([rng.uniform(-spread, spread, n), rng.uniform(-spread, spread, n), z], 1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = scene_from(means, np.exp(rng.uniform(np.log(0.01), np.log(0.04), (n, 3))), q, rng.uniform(0.05, 0.6, n),
                    rng.uniform(0, 1, (n, 3)))
    Wd, Hd = size, (size * 3 // 4 if size > 32 else size)
    K, W = identity_cam(fx=100.0, fy=100.0, cx=Wd / 2 + 0.5, cy=Hd / 2 + 0.5)
    g = gsb.Scene.from_synth(sc)
    g.reserve(1, 1, Wd, Hd)
    for split_min in ("0", "1000000000"):
        os.environ["GSB_K4_SPLIT_MIN"] = split_min
        rgb = torch.zeros((1, 1, 3, Hd, Wd), device="cuda")
        g.render(None, torch.from_numpy(K[None, None].copy()).cuda(), torch.from_numpy(W[None, None].copy()).cuda(),
                 gsb.RenderParams(Wd, Hd), rgb)
        torch.cuda.synchronize()
    os.environ.pop("GSB_K4_SPLIT_MIN")
    print("ties ok", n, layers, float(rgb.mean()))

# round 2: fixed-plan render (device-side long-list count, overflow flag) and the K4a index sort
# on 513..4096-key lists with equal-depth runs (64x64 view of a 3000-Gaussian layered plane)
cfg = synth.CONFIGS["T2"]
sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
g = gsb.Scene.from_synth(sc)
g.reserve(cfg.n_envs, 1, cfg.width, cfg.height)
rgb = torch.zeros((cfg.n_envs, 1, 3, cfg.height, cfg.width), device="cuda")
g.render(torch.from_numpy(b.poses).cuda(), torch.from_numpy(b.intrinsics).cuda(), torch.from_numpy(b.w2c).cuda(),
         gsb.RenderParams(cfg.width, cfg.height, fixed_plan=True), rgb)
torch.cuda.synchronize()
print("fixed plan ok", g.overflow(), float(rgb.mean()))
g.reserve(cfg.n_envs, 1, cfg.width, cfg.height, 0, 1000)
g.render(torch.from_numpy(b.poses).cuda(), torch.from_numpy(b.intrinsics).cuda(), torch.from_numpy(b.w2c).cuda(),
         gsb.RenderParams(cfg.width, cfg.height, fixed_plan=True), rgb)
torch.cuda.synchronize()
print("fixed plan overflow ok", g.overflow())
n, layers = 3000, 25
rng = np.random.default_rng(64)
z = 2.0 + 0.05 * rng.integers(0, layers, n)
means = np.stack([rng.uniform(-0.3, 0.3, n), rng.uniform(-0.3, 0.3, n), z], 1)
q = rng.normal(size=(n, 4))
q /= np.linalg.norm(q, axis=1, keepdims=True)
sc = scene_from(means, np.exp(rng.uniform(np.log(0.01), np.log(0.04), (n, 3))), q, rng.uniform(0.05, 0.6, n),
                rng.uniform(0, 1, (n, 3)))
K, W = identity_cam(fx=100.0, fy=100.0, cx=32.5, cy=32.5)
g = gsb.Scene.from_synth(sc)
g.reserve(1, 1, 64, 64)
os.environ["GSB_K4_SPLIT_MIN"] = "0"
rgb = torch.zeros((1, 1, 3, 64, 64), device="cuda")
g.render(None, torch.from_numpy(K[None, None].copy()).cuda(), torch.from_numpy(W[None, None].copy()).cuda(),
         gsb.RenderParams(64, 64, stats=True), rgb)
torch.cuda.synchronize()
os.environ.pop("GSB_K4_SPLIT_MIN")
print("index sort ties ok", g.stats(), float(rgb.mean()))
