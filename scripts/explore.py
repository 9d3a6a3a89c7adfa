"""Exploration on the GPU box: pinned-copy bandwidth and device frames/s on every config."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402

res = {}
# pinned copy bandwidth (the e2e ceiling)
n = 1 << 28  # 1 GiB of fp32
h = torch.empty(n, pin_memory=True)
d = torch.empty(n, device="cuda")
for name, (dst, src) in {"d2h": (h, d), "h2d": (d, h)}.items():
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    res[name + "_GBps"] = 3 * 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
del h, d
torch.cuda.empty_cache()
print(json.dumps(res), flush=True)

envs = {"C2": 64, "C3": 1024, "C4": 4096, "C5": 1024, "C6": 4096, "C7": 256, "T1": 3}
MODES = ("rig", "static", "scores", "obs", "static_env")
_named = [n for n in sys.argv[1:] if n in synth.CONFIGS]
_modes_only = bool(sys.argv[1:]) and all(a in MODES for a in sys.argv[1:])
for name in ([] if _modes_only or ("static" in sys.argv[1:]) else (_named or ["C2", "C4", "C5", "C3"])):
    cfg = synth.CONFIGS[name]
    B = envs.get(name, cfg.n_envs)
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, cfg.n_cams, cfg.width, cfg.height)
    K, W = synth.make_cameras(cfg, np.arange(B))
    poses = [torch.from_numpy(synth.make_poses(cfg, np.arange(B), s)).cuda() for s in range(4)]
    K, W = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    rgb = torch.empty((B, cfg.n_cams, 3, cfg.height, cfg.width), device="cuda")
    dep = torch.empty((B, cfg.n_cams, cfg.height, cfg.width), device="cuda")
    g.render(poses[0], K, W, gsb.RenderParams(cfg.width, cfg.height, stats=True), rgb, dep)
    st = g.stats()
    prm = gsb.RenderParams(cfg.width, cfg.height, timing=True)
    for s in range(2):
        g.render(poses[s], K, W, prm, rgb, dep)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for s in range(3):
        g.render(poses[(s + 1) % 4], K, W, prm, rgb, dep)
    e1.record()
    torch.cuda.synchronize()
    tm = g.timings()
    F = B * cfg.n_cams
    out = {"config": name, "frames": F, "W": cfg.width, "H": cfg.height, "N": sc.n,
           "fps": 3 * F / (e0.elapsed_time(e1) / 1e3), "V/f": st["V"] / F, "K/f": st["K"] / F, "P/f": st["P"] / F,
           "stage_ms": {k: round(v, 2) for k, v in tm.items() if k.endswith("_ms")},
           "long_lists": tm["long_lists"], "max_list": tm["max_list"]}
    print(json.dumps(out), flush=True)
    del g, rgb, dep
    torch.cuda.empty_cache()

# §8(f) row 1 measurement: C4 with camera 1 wrist-mounted on body 9, poses from a 13-float
# physics-state buffer, through gsb_render_rig
if "rig" in sys.argv[1:] or not sys.argv[1:]:
    cfg = synth.CONFIGS["C4"]
    B = 4096
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, cfg.n_cams, cfg.width, cfg.height)
    K, W = synth.make_cameras(cfg, np.arange(B))
    c2b = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
    W[:, 1, :, :3] = c2b.T
    W[:, 1, :, 3] = -c2b.T @ np.array([0.33, 0.0, 0.06])
    nb = cfg.n_bodies
    states = []
    for s in range(4):
        st = np.zeros((B, nb, 13), np.float32)
        st[..., :7] = synth.make_poses(cfg, np.arange(B), s)
        states.append(torch.from_numpy(st).cuda())
    K, W = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    rgb = torch.empty((B, cfg.n_cams, 3, cfg.height, cfg.width), device="cuda")
    dep = torch.empty((B, cfg.n_cams, cfg.height, cfg.width), device="cuda")
    cam_body = np.array([-1, 9], np.int32)
    prm = gsb.RenderParams(cfg.width, cfg.height)
    for s in range(2):
        g.render_rig(states[s], K, W, prm, rgb, dep, cam_body=cam_body, pose_env_stride=nb * 13, pose_body_stride=13)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for s in range(3):
        g.render_rig(states[(s + 1) % 4], K, W, prm, rgb, dep, cam_body=cam_body, pose_env_stride=nb * 13,
                     pose_body_stride=13)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"config": "C4-rig (cam 1 on body 9, strided 13-float states)", "frames": B * 2,
                      "fps": 3 * B * 2 / (e0.elapsed_time(e1) / 1e3)}), flush=True)

# §8(f) row 2 measurement: C3 with cameras fixed in the world (env 0's camera for every env):
# gsb_render with the camera broadcast vs gsb_prebin_static + gsb_render_static (bit-identical)
if "static" in sys.argv[1:] or not sys.argv[1:]:
    for name in [n for n in sys.argv[1:] if n in synth.CONFIGS] or ["C3"]:
        cfg = synth.CONFIGS[name]
        B = envs.get(name, cfg.n_envs)
        sc = synth.make_scene(cfg)
        g = gsb.Scene.from_synth(sc)
        Ks, Ws = synth.static_cameras(cfg)
        prm0 = gsb.RenderParams(cfg.width, cfg.height)
        torch.cuda.synchronize()
        t0 = time.time()
        g.prebin_static(Ks, Ws, prm0)
        t_prebin = time.time() - t0
        g.reserve(B, cfg.n_cams, cfg.width, cfg.height)
        K = torch.from_numpy(np.broadcast_to(Ks, (B,) + Ks.shape).copy()).cuda()
        W = torch.from_numpy(np.broadcast_to(Ws, (B,) + Ws.shape).copy()).cuda()
        poses = [torch.from_numpy(synth.make_poses(cfg, np.arange(B), s)).cuda() for s in range(4)]
        rgb = torch.empty((B, cfg.n_cams, 3, cfg.height, cfg.width), device="cuda")
        dep = torch.empty((B, cfg.n_cams, cfg.height, cfg.width), device="cuda")
        res = {}
        for mode in ("render", "render_static"):
            def call(s, prm):
                if mode == "render":
                    g.render(poses[s], K, W, prm, rgb, dep)
                else:
                    g.render_static(poses[s], prm, rgb, dep)
            prm = gsb.RenderParams(cfg.width, cfg.height, timing=True)
            call(0, gsb.RenderParams(cfg.width, cfg.height, stats=True))
            st = g.stats()
            for s in range(2):
                call(s, prm)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for s in range(3):
                call((s + 1) % 4, prm)
            e1.record()
            torch.cuda.synchronize()
            tm = g.timings()
            F = B * cfg.n_cams
            res[mode] = {"fps": 3 * F / (e0.elapsed_time(e1) / 1e3), "P/f": st["P"] / F, "K/f": st["K"] / F,
                         "stage_ms": {k: round(v, 2) for k, v in tm.items() if k.endswith("_ms")}}
        print(json.dumps({"config": name + "-static (env 0 cameras for all envs)", "frames": B * cfg.n_cams,
                          "prebin_s": round(t_prebin, 3), **res}), flush=True)
        del g, rgb, dep
        torch.cuda.empty_cache()

# §8(f) row 2 with per-env cameras (GSB_FLAG_STATIC_PER_ENV): the bench's C3 workload exactly
# (each env's domain-randomised camera, fixed over the episode), background pre-binned per env
if "static_env" in sys.argv[1:]:
    cfg = synth.CONFIGS["C3"]
    B = 1024
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    K, W = synth.make_cameras(cfg, np.arange(B))
    torch.cuda.synchronize()
    t0 = time.time()
    g.prebin_static(K[:, 0].copy(), W[:, 0].copy(), gsb.RenderParams(cfg.width, cfg.height))
    t_prebin = time.time() - t0
    g.reserve(B, 1, cfg.width, cfg.height)
    Kd, Wd = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    poses = [torch.from_numpy(synth.make_poses(cfg, np.arange(B), s)).cuda() for s in range(4)]
    rgb = torch.empty((B, 1, 3, cfg.height, cfg.width), device="cuda")
    dep = torch.empty((B, 1, cfg.height, cfg.width), device="cuda")
    res = {}
    for mode in ("render", "render_static_per_env"):
        prm = gsb.RenderParams(cfg.width, cfg.height, static_per_env=(mode != "render"))

        def call(s):
            if mode == "render":
                g.render(poses[s], Kd, Wd, prm, rgb, dep)
            else:
                g.render_static(poses[s], prm, rgb, dep)
        for s in range(2):
            call(s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for s in range(5):
            call((s + 1) % 4)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = {"fps": 5 * B / (e0.elapsed_time(e1) / 1e3)}
    print(json.dumps({"config": "C3 per-env static cameras (GSB_FLAG_STATIC_PER_ENV)", "frames": B,
                      "prebin_s": round(t_prebin, 3), "prebin_GB": round(torch.cuda.memory_allocated() / 1e9, 1),
                      **res}), flush=True)
    del g, rgb, dep
    torch.cuda.empty_cache()

# §8(f) row 3 measurement: C3 render with GSB_FLAG_SCORES (pruning-score accumulation) vs plain
if "scores" in sys.argv[1:] or not sys.argv[1:]:
    cfg = synth.CONFIGS["C3"]
    B = 1024
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, cfg.n_cams, cfg.width, cfg.height)
    K, W = synth.make_cameras(cfg, np.arange(B))
    K, W = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    poses = [torch.from_numpy(synth.make_poses(cfg, np.arange(B), s)).cuda() for s in range(4)]
    rgb = torch.empty((B, cfg.n_cams, 3, cfg.height, cfg.width), device="cuda")
    dep = torch.empty((B, cfg.n_cams, cfg.height, cfg.width), device="cuda")
    res = {}
    for mode in ("plain", "scores"):
        prm = gsb.RenderParams(cfg.width, cfg.height, timing=True, scores=(mode == "scores"))
        for s in range(2):
            g.render(poses[s], K, W, prm, rgb, dep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for s in range(3):
            g.render(poses[(s + 1) % 4], K, W, prm, rgb, dep)
        e1.record()
        torch.cuda.synchronize()
        tm = g.timings()
        res[mode] = {"fps": 3 * B / (e0.elapsed_time(e1) / 1e3), "composite_ms": round(tm["composite_ms"], 2)}
    ws, wm = g.scores()
    res["scored_gaussians"] = int((ws > 0).sum().item())
    print(json.dumps({"config": "C3 with GSB_FLAG_SCORES", **res}), flush=True)

# §8(f) row 4 measurement: C3 observations (uint8 RGB + fp16 depth, image DR with noise), device
# and host (e2e: pinned host inputs/outputs) vs the fp32 outputs
if "obs" in sys.argv[1:] or not sys.argv[1:]:
    cfg = synth.CONFIGS["C3"]
    B = 1024
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, cfg.n_cams, cfg.width, cfg.height, host_io=True)
    K, W = synth.make_cameras(cfg, np.arange(B))
    Kd, Wd = torch.from_numpy(K).cuda(), torch.from_numpy(W).cuda()
    P = [synth.make_poses(cfg, np.arange(B), s) for s in range(4)]
    Pd = [torch.from_numpy(p).cuda() for p in P]
    rng = np.random.default_rng(0)
    dr = np.stack([rng.uniform(0.7, 1.4, (B, 1)), rng.uniform(0.7, 1.3, (B, 1)), rng.uniform(-0.05, 0.05, (B, 1)),
                   np.full((B, 1), 0.02)], -1).astype(np.float32)
    drd = torch.from_numpy(dr).cuda()
    H_, W_ = cfg.height, cfg.width
    q = torch.empty((B, 1, 3, H_, W_), dtype=torch.uint8, device="cuda")
    d16 = torch.empty((B, 1, H_, W_), dtype=torch.float16, device="cuda")
    hq = torch.empty((B, 1, 3, H_, W_), dtype=torch.uint8).pin_memory()
    hd = torch.empty((B, 1, H_, W_), dtype=torch.float16).pin_memory()
    hP = [torch.from_numpy(p).pin_memory() for p in P]
    hK, hW, hdr = torch.from_numpy(K).pin_memory(), torch.from_numpy(W).pin_memory(), torch.from_numpy(dr).pin_memory()
    prm = gsb.RenderParams(W_, H_, timing=True)
    res = {}

    def dev(s):
        g.render_obs(Pd[s], Kd, Wd, prm, q, d16, image_dr=drd, seed=1, step=s)

    def host(s):
        g.render_obs_host(hP[s], hK, hW, prm, hq, hd, image_dr=hdr, seed=1, step=s)

    for mode, fn in (("device", dev), ("host_e2e", host)):
        for s in range(2):
            fn(s)
        torch.cuda.synchronize()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for s in range(3):
            fn((s + 1) % 4)
        e1.record()
        torch.cuda.synchronize()
        wall = time.time() - t0
        res[mode] = {"fps": 3 * B / (e0.elapsed_time(e1) / 1e3), "wall_fps": 3 * B / wall,
                     "composite_ms": round(g.timings()["composite_ms"], 2)}
    res["d2h_bytes_per_step"] = int(hq.numel() + 2 * hd.numel())
    print(json.dumps({"config": "C3 observations (uint8 RGB + fp16 depth, image DR)", **res}), flush=True)
