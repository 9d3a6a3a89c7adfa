"""Does a device->host copy overlap with SM compute on this box? (pure torch)"""
import json
import torch

h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
s2 = torch.cuda.Stream()


def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def mm():
    for _ in range(40):
        a @ a


def cp():
    with torch.cuda.stream(s2):
        for _ in range(4):
            h.copy_(d, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s2):
        for _ in range(4):
            h.copy_(d, non_blocking=True)
    mm()
    torch.cuda.current_stream().wait_stream(s2)


def hbm_kernel():
    for _ in range(40):
        d.add_(1)


def both_hbm():
    with torch.cuda.stream(s2):
        for _ in range(4):
            h.copy_(d, non_blocking=True)
    hbm_kernel()
    torch.cuda.current_stream().wait_stream(s2)


print(json.dumps({"matmul_ms": t(mm), "d2h_4GB_ms": t(cp), "both_ms": t(both),
                  "hbm_ms": t(hbm_kernel), "d2h_and_hbm_ms": t(both_hbm)}))
