"""K6 (gsb_obs_encode: reading R33 motion blur + R31 DR/noise/uint8/fp16) throughput on C3-sized
batches (1024 frames of 640x480 fp32 RGB + depth, resident in HBM): device time per call by CUDA
events and achieved HBM bandwidth against MEASURED_PEAKS.json (algorithmic bytes: 12 B RGB +
4 B depth read, 3 B + 2 B written per pixel; blur taps re-read neighbours from L1/L2)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_25459_b200 as gsb  # noqa: E402

B, H, W = 1024, 480, 640
rgb = torch.rand((B, 1, 3, H, W), device="cuda")
dep = torch.rand((B, 1, H, W), device="cuda") * 5
out8 = torch.empty((B, 1, 3, H, W), dtype=torch.uint8, device="cuda")
od = torch.empty((B, 1, H, W), dtype=torch.float16, device="cuda")
dr = torch.tensor([1.1, 0.9, 0.02, 0.02], device="cuda").repeat(B, 1, 1).contiguous()
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs")
except Exception:
    pass
for name, bx, by in (("no_blur", 0, 0), ("blur_5_2", 5, 2), ("blur_12_0", 12, 0)):
    blur = torch.tensor([bx, by], dtype=torch.int32, device="cuda").repeat(B, 1, 1).contiguous()
    gsb.obs_encode(rgb, out8, depth=dep, out_depth=od, blur=blur, image_dr=dr, seed=1, step=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        gsb.obs_encode(rgb, out8, depth=dep, out_depth=od, blur=blur, image_dr=dr, seed=1, step=2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gbs = B * H * W * 21 / (ms / 1e3) / 1e9
    print(json.dumps({"case": name, "frames": B, "ms": ms, "frames_per_s": B / (ms / 1e3), "GBps": gbs,
                      "peak_GBps": peak, "frac": gbs / peak if peak else None}), flush=True)
