"""Probe the host-buffer (e2e) path: render vs render_host vs raw chunked D2H."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["C3"]
B, C, W, H = 1024, 1, cfg.width, cfg.height
sc = synth.make_scene(cfg)
g = gsb.Scene.from_synth(sc)
g.reserve(B, C, W, H, host_io=True)
K, Wc = synth.make_cameras(cfg, np.arange(B))
P = synth.make_poses(cfg, np.arange(B), 0)
dK, dW, dP = (torch.from_numpy(x).cuda() for x in (K, Wc, P))
hK, hW, hP = (torch.from_numpy(x).pin_memory() for x in (K, Wc, P))
rgb = torch.empty((B, C, 3, H, W), device="cuda")
dep = torch.empty((B, C, H, W), device="cuda")
hrgb = torch.empty((B, C, 3, H, W), pin_memory=True)
hdep = torch.empty((B, C, H, W), pin_memory=True)
prm = gsb.RenderParams(W, H)


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


res = {}
res["render_ms"] = timed(lambda: g.render(dP, dK, dW, prm, rgb, dep))
res["render_host_rgb_ms"] = timed(lambda: g.render_host(hP, hK, hW, prm, hrgb))
res["render_host_rgb_depth_ms"] = timed(lambda: g.render_host(hP, hK, hW, prm, hrgb, hdep))


def raw():
    for c in range(16):
        sl = slice(c * 64, (c + 1) * 64)
        hrgb[sl].copy_(rgb[sl], non_blocking=True)
        hdep[sl].copy_(dep[sl], non_blocking=True)


res["raw_d2h_5GB_ms"] = timed(raw)
s2 = torch.cuda.Stream()


def overlap():
    ev = torch.cuda.Event()
    g.render(dP, dK, dW, prm, rgb, dep)
    ev.record()
    with torch.cuda.stream(s2):
        s2.wait_event(ev)
        raw()
    torch.cuda.current_stream().wait_stream(s2)


res["render_then_d2h_ms"] = timed(overlap)
print(json.dumps(res))

# independent concurrency test: render on the current stream, unrelated D2H on s2 at the same time
rgb2 = torch.empty_like(rgb)
dep2 = torch.empty_like(dep)


def concurrent():
    with torch.cuda.stream(s2):
        for c in range(16):
            sl = slice(c * 64, (c + 1) * 64)
            hrgb[sl].copy_(rgb2[sl], non_blocking=True)
            hdep[sl].copy_(dep2[sl], non_blocking=True)
    g.render(dP, dK, dW, prm, rgb, dep)
    torch.cuda.current_stream().wait_stream(s2)


res2 = {"concurrent_render_and_unrelated_d2h_ms": timed(concurrent)}
import time
t0 = time.perf_counter()
g.render_host(hP, hK, hW, prm, hrgb, hdep)
res2["render_host_wall_ms"] = (time.perf_counter() - t0) * 1e3
st_ = torch.cuda.Stream()
with torch.cuda.stream(st_):
    res2["render_host_on_side_stream_ms"] = timed(lambda: g.render_host(hP, hK, hW, prm, hrgb, hdep, stream=st_))
print(json.dumps(res2))
