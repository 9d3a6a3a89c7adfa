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


pairs_near_threshold = gu.pairs_near_threshold


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
            arg_g = gu.k4_arg_f32(r, px, py)
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
