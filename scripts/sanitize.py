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
