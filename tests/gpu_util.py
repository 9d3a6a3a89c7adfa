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
