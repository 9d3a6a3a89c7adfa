#!/usr/bin/env python
"""Measure the GPU's alpha error against the fp64 oracle (reading R28's margins).

For every (pixel, Gaussian) pair whose oracle alpha lies near the 1/255 skip threshold, compare
  arg_oracle = log2(o) + power * log2(e)                      (fp64, oracle.project)
  arg_gpu    = K4's fp32 evaluation on the GPU's own K1 record (gsb_debug_project fields 0,1,12-15)
             dx = u - pxc; t1 = p dx; mm = fma(-t1, t1, log2o); ta = fma(r, v - pyc, q dx);
             arg = fma(-ta, ta, mm)                            (emulated here in binary32)
and write per-pair features to gpurun_out/alpha_error_<cfg>.npz for fitting the error model.
Also records the per-pixel T error of full renders (alpha output vs oracle alpha)."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from tests import gpu_util as gu  # noqa: E402

LOG2E = 1.4426950408889634
THR = np.log2(1.0 / 255.0)
f32 = np.float32


def fma32(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def pairs_near_threshold(proj, ids, W, H, win):
    """(gaussian index, px, py) of pixel centres inside the R8 box of each id (vectorised)."""
    u, v = proj[ids, oracle.F_U], proj[ids, oracle.F_V]
    rx = np.sqrt(proj[ids, oracle.F_KAPPA] * proj[ids, oracle.F_SXX])
    ry = np.sqrt(proj[ids, oracle.F_KAPPA] * proj[ids, oracle.F_SYY])
    x0 = np.clip(np.ceil(u - rx - 0.5), 0, W - 1).astype(np.int64)
    x1 = np.clip(np.floor(u + rx - 0.5), 0, W - 1).astype(np.int64)
    y0 = np.clip(np.ceil(v - ry - 0.5), 0, H - 1).astype(np.int64)
    y1 = np.clip(np.floor(v + ry - 0.5), 0, H - 1).astype(np.int64)
    nx, ny = np.maximum(x1 - x0 + 1, 0), np.maximum(y1 - y0 + 1, 0)
    out_g, out_x, out_y = [], [], []
    cnt = nx * ny
    sel = cnt > 0
    ids, x0, y0, nx, cnt = ids[sel], x0[sel], y0[sel], nx[sel], cnt[sel]
    for lo in range(0, ids.size, 20000):
        sl = slice(lo, lo + 20000)
        c = cnt[sl]
        g = np.repeat(ids[sl], c)
        k = np.arange(c.sum()) - np.repeat(np.cumsum(c) - c, c)
        px = np.repeat(x0[sl], c) + k % np.repeat(nx[sl], c)
        py = np.repeat(y0[sl], c) + k // np.repeat(nx[sl], c)
        dx = proj[g, oracle.F_U] - (px + 0.5)
        dy = proj[g, oracle.F_V] - (py + 0.5)
        power = -0.5 * (proj[g, oracle.F_A] * dx * dx + proj[g, oracle.F_C] * dy * dy) - proj[g, oracle.F_B] * dx * dy
        arg = np.log2(proj[g, oracle.F_O]) + power * LOG2E
        keep = np.abs(arg - THR) < win
        out_g.append(g[keep]); out_x.append(px[keep]); out_y.append(py[keep])
    return np.concatenate(out_g), np.concatenate(out_x), np.concatenate(out_y)


def measure(name, max_frames=4, win=0.05):
    cfg = synth.CONFIGS[name]
    sc = synth.make_scene(cfg)
    envs = list(range(min(cfg.n_envs, max_frames)))
    b = synth.make_batch(cfg, envs)
    W, H = cfg.width, cfg.height
    import paper_2604_25459_b200 as gsb
    g = gsb.Scene.from_synth(sc)
    g.reserve(len(envs), cfg.n_cams, W, H)
    rec, zb, va = gu.gpu_project(g, b, W, H)
    prm = oracle.RenderParams(W, H)
    cols = {k: [] for k in ("d_arg", "d_arg_rec", "arg", "gx", "gy", "u", "v", "du", "dv", "Q", "sxx", "syy",
                            "det_rel", "o", "z", "gid", "env", "cam", "px", "py", "rec")}
    for e in range(len(envs)):
        for c in range(cfg.n_cams):
            f = e * cfg.n_cams + c
            proj, ozb, ovalid = oracle.project(sc, b.poses[e], b.intrinsics[e, c], b.w2c[e, c], prm)
            ids = np.nonzero(ovalid & va[f])[0]
            gi, px, py = pairs_near_threshold(proj, ids, W, H, win)
            r = rec[f][gi]
            dx64 = proj[gi, oracle.F_U] - (px + 0.5)
            dy64 = proj[gi, oracle.F_V] - (py + 0.5)
            A, B, C = proj[gi, oracle.F_A], proj[gi, oracle.F_B], proj[gi, oracle.F_C]
            power = -0.5 * (A * dx64 * dx64 + C * dy64 * dy64) - B * dx64 * dy64
            arg_o = np.log2(proj[gi, oracle.F_O]) + power * LOG2E
            # GPU arithmetic in binary32 on the GPU's record
            u, v, p, q, rr, l2o = (r[:, k].astype(f32) for k in (0, 1, 12, 13, 14, 15))
            pxc, pyc = (px + 0.5).astype(f32), (py + 0.5).astype(f32)
            dx = (u - pxc).astype(f32)
            t1 = (p * dx).astype(f32)
            mm = fma32(-t1, t1, l2o)
            qdx = (q * dx).astype(f32)
            ta = fma32(rr, (v - pyc).astype(f32), qdx)
            arg_g = fma32(-ta, ta, mm)
            # the same on the record in fp64 (record error only)
            dxr = u.astype(np.float64) - (px + 0.5)
            dyr = v.astype(np.float64) - (py + 0.5)
            arg_r = l2o.astype(np.float64) - (p * dxr) ** 2 - (q.astype(np.float64) * dxr + rr * dyr) ** 2
            cols["d_arg"].append(arg_g.astype(np.float64) - arg_o)
            cols["d_arg_rec"].append(arg_r - arg_o)
            cols["arg"].append(arg_o)
            cols["gx"].append(-(A * dx64 + B * dy64) * LOG2E)    # d arg / d u
            cols["gy"].append(-(B * dx64 + C * dy64) * LOG2E)
            cols["u"].append(proj[gi, oracle.F_U]); cols["v"].append(proj[gi, oracle.F_V])
            cols["du"].append(r[:, 0] - proj[gi, oracle.F_U]); cols["dv"].append(r[:, 1] - proj[gi, oracle.F_V])
            cols["Q"].append(-power * LOG2E)
            cols["sxx"].append(proj[gi, oracle.F_SXX]); cols["syy"].append(proj[gi, oracle.F_SYY])
            det = proj[gi, oracle.F_SXX] * proj[gi, oracle.F_SYY] - proj[gi, oracle.F_SXY] ** 2
            cols["det_rel"].append(det / (proj[gi, oracle.F_SXX] * proj[gi, oracle.F_SYY]))
            cols["o"].append(proj[gi, oracle.F_O]); cols["z"].append(proj[gi, oracle.F_Z64])
            cols["gid"].append(gi); cols["env"].append(np.full(gi.size, envs[e])); cols["cam"].append(np.full(gi.size, c))
            cols["px"].append(px); cols["py"].append(py); cols["rec"].append(r)
    out = {k: np.concatenate(v) for k, v in cols.items()}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"alpha_error_{name}.npz"), **out)
    d = np.abs(out["d_arg"])
    print(name, "pairs", d.size, "max |d arg| (log2)", float(d.max()), "p99.9", float(np.quantile(d, 0.999)),
          "median", float(np.median(d)), "max |du|", float(np.abs(out["du"]).max()), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["T1", "T2", "T4", "T5", "T6", "C1"]:
        measure(n, max_frames=1 if n.startswith("C") and n != "C1" else 4)
