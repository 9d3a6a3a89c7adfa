"""Helpers for the -m gpu parity tests: run libgsb through its C ABI on torch CUDA memory and
compare against the CPU oracle (tests are the only place the two meet)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from oracle import binning


def to_dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def gpu_render(scene: synth.Scene, batch: synth.Batch, W: int, H: int, bg=(0.0, 0.0, 0.0), sh_degree=-1,
               chunk_frames=0, key_capacity=0, stats=False, gscene=None, near=0.01, far=1000.0):
    B, C = batch.intrinsics.shape[:2]
    g = gscene or gsb.Scene.from_synth(scene)
    if gscene is None:
        g.reserve(B, C, W, H, chunk_frames, key_capacity)
    rgb = torch.full((B, C, 3, H, W), float("nan"), device="cuda")
    dep = torch.full((B, C, H, W), float("nan"), device="cuda")
    alp = torch.full((B, C, H, W), float("nan"), device="cuda")
    nev = torch.full((B, C, H, W), -7, dtype=torch.int32, device="cuda")
    prm = gsb.RenderParams(W, H, near=near, far=far, background=bg, sh_degree=sh_degree, stats=stats)
    g.render(to_dev(batch.poses), to_dev(batch.intrinsics), to_dev(batch.w2c), prm, rgb, dep, alp, nev)
    torch.cuda.synchronize()
    out = dict(rgb=rgb.cpu().numpy(), depth=dep.cpu().numpy(), alpha=alp.cpu().numpy(),
               n_eval=nev.cpu().numpy())
    if stats:
        out["stats"] = g.stats()
    out["scene"] = g
    return out


def gpu_project(g: gsb.Scene, batch: synth.Batch, W: int, H: int, sh_degree=-1):
    B, C = batch.intrinsics.shape[:2]
    N = g.n
    rec = torch.zeros((B * C, N, 16), device="cuda")
    zb = torch.zeros((B * C, N), dtype=torch.int32, device="cuda")
    va = torch.zeros((B * C, N), dtype=torch.uint8, device="cuda")
    g.debug_project(to_dev(batch.poses), to_dev(batch.intrinsics), to_dev(batch.w2c),
                    gsb.RenderParams(W, H, sh_degree=sh_degree), rec, zb, va)
    torch.cuda.synchronize()
    return rec.cpu().numpy(), zb.cpu().numpy().view(np.uint32), va.cpu().numpy().astype(bool)


def pairs_near_threshold(proj, ids, W, H, win):
    """(Gaussian row, px, py) of every pixel centre inside the R8 box of each id whose oracle
    arg = log2(o e^power) lies within `win` (log2 units) of log2(1/255)."""
    LOG2E = 1.4426950408889634
    thr = np.log2(1.0 / 255.0)
    u, v = proj[ids, oracle.F_U], proj[ids, oracle.F_V]
    rx = np.sqrt(proj[ids, oracle.F_KAPPA] * proj[ids, oracle.F_SXX])
    ry = np.sqrt(proj[ids, oracle.F_KAPPA] * proj[ids, oracle.F_SYY])
    x0 = np.clip(np.ceil(u - rx - 0.5), 0, W - 1).astype(np.int64)
    x1 = np.clip(np.floor(u + rx - 0.5), 0, W - 1).astype(np.int64)
    y0 = np.clip(np.ceil(v - ry - 0.5), 0, H - 1).astype(np.int64)
    y1 = np.clip(np.floor(v + ry - 0.5), 0, H - 1).astype(np.int64)
    nx, ny = np.maximum(x1 - x0 + 1, 0), np.maximum(y1 - y0 + 1, 0)
    cnt = nx * ny
    sel = cnt > 0
    ids, x0, y0, nx, cnt = ids[sel], x0[sel], y0[sel], nx[sel], cnt[sel]
    out_g, out_x, out_y = [np.zeros(0, np.int64)], [np.zeros(0, np.int64)], [np.zeros(0, np.int64)]
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
        keep = np.abs(arg - thr) < win
        out_g.append(g[keep]); out_x.append(px[keep]); out_y.append(py[keep])
    return np.concatenate(out_g), np.concatenate(out_x), np.concatenate(out_y)


def k4_arg_f32(rec, px, py):
    """K4's binary32 evaluation of arg = log2(o) - (p dx)^2 - (q dx + r dy)^2 on the GPU's own K1
    records (gsb_debug_project fields u, v, p, q, r, log2 o), emulated in numpy (fma = exact
    binary64 product + sum, then rounded to binary32)."""
    f32 = np.float32

    def fma(a, b, c):
        return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(f32)

    u, v, p, q, r, l2o = (rec[:, k].astype(f32) for k in (0, 1, 12, 13, 14, 15))
    dx = (u - (px + 0.5).astype(f32)).astype(f32)
    t1 = (p * dx).astype(f32)
    mm = fma(-t1, t1, l2o)
    ta = fma(r, (v - (py + 0.5).astype(f32)).astype(f32), (q * dx).astype(f32))
    return fma(-ta, ta, mm)


def kappa_f32(scene: synth.Scene) -> np.ndarray:
    return np.float32(2.0 * np.log(255.0 * scene.opacities.astype(np.float64)))


def expected_n_eval(term_id, tile_ids_for_pixel):
    """n_eval implied by the oracle's termination id on the GPU's own tile list."""
    if term_id < 0:
        return len(tile_ids_for_pixel)
    hits = np.nonzero(tile_ids_for_pixel == term_id)[0]
    return int(hits[0]) + 1 if hits.size else -1


def compare_frame(gout, f_env, f_cam, ref: oracle.FrameResult, W, H, pix=None, gpu_rec=None, gpu_zb=None,
                  gpu_valid=None, kap=None):
    """Element-by-element comparison of one frame (all pixels, or the sampled `pix`)."""
    rgb = gout["rgb"][f_env, f_cam].transpose(1, 2, 0)   # [H,W,3]
    dep = gout["depth"][f_env, f_cam]
    alp = gout["alpha"][f_env, f_cam]
    nev = gout["n_eval"][f_env, f_cam]
    if pix is not None:
        px, py = pix
        rgb, dep, alp, nev = rgb[py, px], dep[py, px], alp[py, px], nev[py, px]
        ref_rgb, ref_dep, ref_alp, ref_term = ref.rgb, ref.depth, ref.alpha, ref.term_id
        masked = ref.masked
        tnear = ref.term_near
    else:
        ref_rgb, ref_dep, ref_alp, ref_term, masked = ref.rgb, ref.depth, ref.alpha, ref.term_id, ref.masked
        tnear = ref.term_near
    ok = ~masked
    # reading R28: the GPU's T = 1 - alpha within the oracle's relative bound eT wherever no
    # threshold flip is possible (unmasked, no termination test within the bound)
    eT = ref.eT
    T_ref = 1.0 - ref_alp
    t_ok = ok & ~tnear
    T_excess = np.abs((1.0 - alp.astype(np.float64)) - T_ref) - (eT * T_ref + 2.0 ** -23)
    d_rgb = np.abs(rgb - ref_rgb).max(axis=-1)
    d_dep = np.abs(dep - ref_dep)
    d_alp = np.abs(alp - ref_alp)
    res = dict(
        masked_frac=float(masked.mean()),
        max_rgb=float(d_rgb[ok].max()) if ok.any() else 0.0,
        max_dep_excess=float((d_dep - (oracle.TOL_DEPTH_REL * np.abs(ref_dep) + oracle.TOL_DEPTH_ABS))[ok].max())
        if ok.any() else -1.0,
        max_alpha=float(d_alp[ok].max()) if ok.any() else 0.0,
        rgb_fail=int((d_rgb[ok] > oracle.TOL_RGB).sum()),
        dep_fail=int((d_dep > oracle.TOL_DEPTH_REL * np.abs(ref_dep) + oracle.TOL_DEPTH_ABS)[ok].sum()),
        alp_fail=int((d_alp[ok] > oracle.TOL_RGB).sum()),
        n_pix=int(ok.size),
        T_fail=int((T_excess[t_ok] > 0).sum()),
        T_err_over_bound=float(np.max(np.abs((1.0 - alp.astype(np.float64)) - T_ref)[t_ok]
                                      / (eT * T_ref + 2.0 ** -23)[t_ok])) if t_ok.any() else 0.0,
        term_near_frac=float(np.mean(tnear)),
        # information only: how far apart are the MASKED pixels?
        masked_max_rgb=float(d_rgb[~ok].max()) if (~ok).any() else 0.0,
        masked_over_tol=int((d_rgb[~ok] > oracle.TOL_RGB).sum() + (d_dep > oracle.TOL_DEPTH_REL * np.abs(ref_dep)
                                                                   + oracle.TOL_DEPTH_ABS)[~ok].sum()),
    )
    if gpu_rec is not None:
        # n_eval: oracle termination id located in the GPU's own (bit-exact) tile list
        offs, ids = binning.bin_frame(gpu_rec[:, 0], gpu_rec[:, 1], gpu_rec[:, 10], gpu_rec[:, 11], kap, gpu_zb,
                                      gpu_valid, W, H)
        tw = (W + 15) // 16
        if pix is None:
            py, px = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
            px, py = px.reshape(-1), py.reshape(-1)
            term = ref_term.reshape(-1)
            nv = nev.reshape(-1)
            okf = (ok & ~tnear).reshape(-1)
        else:
            px, py = pix
            term, nv, okf = ref_term, nev, ok & ~tnear
        bad = 0
        for k in np.nonzero(okf)[0]:
            t = (py[k] // 16) * tw + px[k] // 16
            e = expected_n_eval(int(term[k]), ids[offs[t]:offs[t + 1]])
            bad += int(e != nv[k])
        res["n_eval_fail"] = bad
        res["n_eval_unchecked_frac"] = float((~okf).mean())
    return res
