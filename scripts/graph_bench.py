#!/usr/bin/env python
"""Small-batch latency: regular gsb_render vs a CUDA-graph replay of a GSB_FLAG_FIXED_PLAN render
(verdict r1 #7; Alg. 1's per-step S_t transfer then render).  One JSON line per config:
ms per step (CUDA events, median of 50 after 10 warm-up), both ways, and the speed-up.
  python scripts/graph_bench.py [C1 C2 T1 ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402


def timed(fn, n=50, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for name in sys.argv[1:] or ["C1", "C2"]:
    cfg = synth.CONFIGS[name]
    envs = min(cfg.n_envs, 64)
    b = synth.make_batch(cfg, list(range(envs)))
    sc = synth.make_scene(cfg)
    g = gsb.Scene.from_synth(sc)
    B, C, H, W = envs, cfg.n_cams, cfg.height, cfg.width
    g.reserve(B, C, W, H)
    poses = torch.from_numpy(b.poses).cuda()
    intr, w2c = torch.from_numpy(b.intrinsics).cuda(), torch.from_numpy(b.w2c).cuda()
    rgb = torch.empty((B, C, 3, H, W), device="cuda")
    dep = torch.empty((B, C, H, W), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        reg = timed(lambda: g.render(poses, intr, w2c, gsb.RenderParams(W, H), rgb, dep))
        fp = gsb.RenderParams(W, H, fixed_plan=True)
        fixed = timed(lambda: g.render(poses, intr, w2c, fp, rgb, dep))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.render(poses, intr, w2c, fp, rgb, dep)
        rep = timed(graph.replay)
    print(json.dumps({"config": name, "envs": B, "frames": B * C, "regular_ms": reg, "fixed_plan_ms": fixed,
                      "graph_replay_ms": rep, "speedup_graph_vs_regular": reg / rep,
                      "graph_frames_per_s": B * C / rep * 1e3}), flush=True)
