"""CPU oracle for the batched 3DGS hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this package.  The product path (paper_2604_25459_b200) never imports it and
shares no code with it (no kernels, headers, helpers, constants or pre/post-processing).

Layout:
  gsb_oracle.c  plain C, fp64 (+ the exact fp32 depth chain, reading R11), pthreads:
                per-pixel brute force over all Gaussians in (z_f32 bits, id) order.
  mini.py       independent NumPy re-implementation (fp64) for small frames (pin 11).
  binning.py    integer-path oracle: fp32 tile rects (R9) and per-tile (zbits, id) lists (R10).
  obs.py        observation epilogue of reading R31 (image DR, uint8 / fp16 encoding), numpy fp32.
  gsb_oracle.c also holds the reading-R32 ray-cast LiDAR (brute force per ray over all
                Gaussians in (rho_f32 bits, id) order; `lidar_frame`).

Each function cites the passage it follows; DESIGN.md §2 lists every reading (R1-R31).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "gsb_oracle.c")

NF = 20
(F_U, F_V, F_SXX, F_SXY, F_SYY, F_A, F_B, F_C, F_R, F_G, F_BL, F_O, F_KAPPA, F_Z32, F_Z64, F_XC, F_YC,
 F_EU, F_EV, F_EQ) = range(NF)

# parity tolerances (BASELINE.json north_star)
TOL_RGB = 2e-3
TOL_DEPTH_REL = 1e-3
TOL_DEPTH_ABS = 1e-6
# The camera path's threshold-margin mask (reading R28) is a forward error bound of the GPU's
# binary32 evaluation computed per entry in gsb_oracle.c (R28_K_POS / R28_K_CONIC / R28_K_EVAL);
# the LiDAR path (reading R32) keeps flat relative margins:
DELTA_ALPHA = 1e-4
DELTA_T = 1e-4
# masked-pixel fraction the parity tests accept per frame: the R28 bound is a worst case of
# binary32 error, so c.3's 1e-4 is out of reach; measured 0-5.4e-3 per frame (C4, C5 the highest)
MASK_CAP = 1e-2


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so: plain C, -O2, no fast-math, no FMA contraction (R11).
    GSB_ORACLE_LIB names a prebuilt variant instead (scripts/host_sanitize.py: ASan/UBSan)."""
    if os.environ.get("GSB_ORACLE_LIB"):
        return os.environ["GSB_ORACLE_LIB"]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_oracle())
        P = ctypes.c_void_p
        L.gsbo_project.restype = ctypes.c_int
        L.gsbo_project.argtypes = [P, P, P, P, P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P,
                                   ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                   ctypes.c_float, P, P, P]
        L.gsbo_composite.restype = ctypes.c_int
        L.gsbo_composite.argtypes = [P, P, ctypes.c_int64, P, P, ctypes.c_int64, P, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     P, P, P, P, P, P, P, P, P, ctypes.c_int,
                                     ctypes.c_int64, P, P, P, P]
        L.gsbo_depth_key.restype = ctypes.c_float
        L.gsbo_depth_key.argtypes = [P, P, P]
        L.gsbo_compose_w2c.restype = None
        L.gsbo_compose_w2c.argtypes = [P, P, P]
        L.gsbo_fmaf.restype = ctypes.c_float
        L.gsbo_fmaf.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
        L.gsbo_lidar_project.restype = ctypes.c_int
        L.gsbo_lidar_project.argtypes = [P, P, P, P, P, ctypes.c_int64, P, ctypes.c_int, P, ctypes.c_float,
                                         ctypes.c_float, P, P, P]
        L.gsbo_lidar_cast.restype = ctypes.c_int
        L.gsbo_lidar_cast.argtypes = [P, P, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, P, P, P, P, P, ctypes.c_int]
        L.gsbo_range_key.restype = ctypes.c_float
        L.gsbo_range_key.argtypes = [P, P, P]
        L.gsbo_lidar_peak.restype = ctypes.c_double
        L.gsbo_lidar_peak.argtypes = [P, P, P]
        L.gsbo_r28_delta.restype = None
        L.gsbo_r28_delta.argtypes = [P, P, P, P, ctypes.c_int64, P]
        L.gsbo_sh_basis.restype = None
        L.gsbo_sh_basis.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, P]
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


@dataclass
class RenderParams:
    width: int
    height: int
    near: float = 0.01      # R4
    far: float = 1000.0
    bg: tuple = (0.0, 0.0, 0.0)   # R15
    sh_degree: Optional[int] = None


def project(scene, pose_env: np.ndarray, intr: np.ndarray, w2c: np.ndarray, prm: RenderParams):
    """Steps 1-5 (pose, depth key, cull, EWA projection, SH colour) for one frame.
    Returns (proj [N,NF] f64, zbits [N] u32, valid [N] bool)."""
    L = lib()
    N = scene.n
    D = scene.sh_degree if prm.sh_degree is None else prm.sh_degree
    out = np.zeros((N, NF), np.float64)
    zb = np.zeros(N, np.uint32)
    valid = np.zeros(N, np.uint8)
    keep = [_c(scene.means, np.float32), _c(scene.scales, np.float32), _c(scene.quats, np.float32),
            _c(scene.opacities, np.float32), _c(scene.sh, np.float32), _c(scene.body_id, np.int32),
            _c(pose_env, np.float32).reshape(-1), _c(intr, np.float32).reshape(-1),
            _c(w2c, np.float32).reshape(-1)]
    rc = L.gsbo_project(_p(keep[0]), _p(keep[1]), _p(keep[2]), _p(keep[3]), _p(keep[4]),
                        scene.sh_degree, D, _p(keep[5]), N, _p(keep[6]), scene.n_bodies,
                        _p(keep[7]), _p(keep[8]), prm.width, prm.height, prm.near, prm.far,
                        _p(out), _p(zb), _p(valid))
    if rc != 0:
        raise ValueError("oracle: body index out of range")
    return out, zb, valid.astype(bool)


def depth_order(zbits: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """Step 6 / reading R10: valid ids sorted by (bits(z_f32) as u32, id) ascending."""
    ids = np.nonzero(valid)[0].astype(np.uint32)
    return ids[np.lexsort((ids, zbits[ids]))].astype(np.uint32)


@dataclass
class FrameResult:
    rgb: np.ndarray        # [npix,3] (or [H,W,3] for full frames)
    depth: np.ndarray
    alpha: np.ndarray
    term_id: np.ndarray    # id of the Gaussian at which the pixel terminated, -1 if none
    n_eval_all: np.ndarray  # entries visited in the all-Gaussian order (diagnostic)
    masked: np.ndarray     # reading R28 threshold-margin mask
    budget_rgb: np.ndarray
    budget_depth: np.ndarray
    proj: np.ndarray
    zbits: np.ndarray
    valid: np.ndarray
    order: np.ndarray
    term_near: np.ndarray  # a termination test within the R28 bound of 1e-4 (n_eval not compared)
    eT: np.ndarray         # R28 relative error bound of the GPU's final T


def composite(proj, order, px, py, prm: RenderParams, mode: str = "box", nthreads: Optional[int] = None,
              margin_scale: float = 1.0, valid=None, scores: Optional[dict] = None):
    """Step 7-9 for the listed pixel coordinates (see gsb_oracle.c).  margin_scale multiplies
    the reading-R28 error bound (1 = the model, 0 = no threshold mask).
    scores: if a dict, also accumulate the reading-R30 pruning scores of these pixels into it:
    w_sum / w_max [N] (f64, by Gaussian id) and, when it holds "mask_in" ([npix] bool), the
    flag "touched" [N] of Gaussians whose exact R8 box holds a masked pixel."""
    L = lib()
    px = _c(px, np.int32).reshape(-1)
    py = _c(py, np.int32).reshape(-1)
    npix = px.size
    order = _c(order, np.uint32)
    bg = _c(prm.bg, np.float32)
    if order.size:
        cmax = float(max(proj[order][:, F_R:F_BL + 1].max(), np.abs(bg).max()))
        zmax = float(proj[order][:, F_Z32].max())
    else:
        cmax, zmax = float(np.abs(bg).max()), 0.0
    rgb = np.zeros((npix, 3)); dep = np.zeros(npix); alp = np.zeros(npix)
    term = np.zeros(npix, np.int64); nev = np.zeros(npix, np.int64)
    brgb = np.zeros(npix); bdep = np.zeros(npix)
    tnear = np.zeros(npix, np.uint8)
    eT = np.zeros(npix)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    proj = _c(proj, np.float64)
    n_gauss = proj.shape[0]
    ws = wm = mk = tch = None
    if scores is not None:
        ws, wm = np.zeros(n_gauss), np.zeros(n_gauss)
        if scores.get("mask_in") is not None:
            mk = _c(np.asarray(scores["mask_in"]).reshape(-1), np.uint8)
            tch = np.zeros(n_gauss, np.uint8)
    rc = L.gsbo_composite(_p(proj), _p(order), order.size, _p(px), _p(py), npix, _p(bg),
                          1 if mode == "box" else 0, float(margin_scale), cmax, zmax,
                          _p(rgb), _p(dep), _p(alp), _p(term), _p(nev), _p(brgb), _p(bdep), _p(tnear),
                          _p(eT), int(nthreads), n_gauss, _p(ws) if ws is not None else None,
                          _p(wm) if wm is not None else None, _p(mk) if mk is not None else None,
                          _p(tch) if tch is not None else None)
    if rc != 0:
        raise MemoryError("oracle composite: allocation failed")
    if scores is not None:
        scores["w_sum"], scores["w_max"] = ws, wm
        scores["touched"] = tch.astype(bool) if tch is not None else None
    masked = (brgb > 0.5 * TOL_RGB) | (bdep > 0.5 * (TOL_DEPTH_REL * dep + TOL_DEPTH_ABS))
    return rgb, dep, alp, term, nev, masked, brgb, bdep, tnear.astype(bool), eT


def render_frame(scene, pose_env, intr, w2c, prm: RenderParams, pixels=None, mode: str = "box",
                 nthreads: Optional[int] = None, **kw) -> FrameResult:
    """One frame end to end.  pixels: None (full frame) or (px, py) int arrays."""
    proj, zb, valid = project(scene, pose_env, intr, w2c, prm)
    order = depth_order(zb, valid)
    full = pixels is None
    if full:
        py, px = np.meshgrid(np.arange(prm.height), np.arange(prm.width), indexing="ij")
        px, py = px.reshape(-1), py.reshape(-1)
    else:
        px, py = pixels
    rgb, dep, alp, term, nev, masked, brgb, bdep, tnear, eT = composite(proj, order, px, py, prm, mode, nthreads, **kw)
    if full:
        H, W = prm.height, prm.width
        rgb, dep, alp = rgb.reshape(H, W, 3), dep.reshape(H, W), alp.reshape(H, W)
        term, nev, masked, tnear = term.reshape(H, W), nev.reshape(H, W), masked.reshape(H, W), tnear.reshape(H, W)
        eT = eT.reshape(H, W)
        brgb, bdep = brgb.reshape(H, W), bdep.reshape(H, W)
    return FrameResult(rgb, dep, alp, term, nev, masked, brgb, bdep, proj, zb, valid, order, tnear, eT)


def frame_scores(scene, pose_env, intr, w2c, prm: RenderParams, nthreads: Optional[int] = None):
    """Reading R30 (§8(f) row 3; pruning by rendering importance): for one full frame,
    per Gaussian id the sum and the max over pixels of the blend weight w = alpha T of every
    blended entry (step 7), plus the R28 "touched" flag (the Gaussian's R8 box holds a pixel in
    the threshold margin, where either side of a flip is correct) and the frame's alpha.
    Returns (w_sum [N], w_max [N], touched [N] bool, alpha [H,W])."""
    fr = render_frame(scene, pose_env, intr, w2c, prm, nthreads=nthreads)
    py, px = np.meshgrid(np.arange(prm.height), np.arange(prm.width), indexing="ij")
    sc = {"mask_in": fr.masked.reshape(-1)}
    composite(fr.proj, fr.order, px.reshape(-1), py.reshape(-1), prm, nthreads=nthreads, scores=sc)
    return sc["w_sum"], sc["w_max"], sc["touched"], fr.alpha


def r28_delta(proj, gid, px, py) -> np.ndarray:
    """Reading R28: the bound on |power_gpu - power| (natural-log units) that the threshold
    mask uses, for pairs (Gaussian row gid of `proj`, pixel (px, py))."""
    proj = _c(proj, np.float64)
    gid, px, py = _c(gid, np.int64).reshape(-1), _c(px, np.int32).reshape(-1), _c(py, np.int32).reshape(-1)
    out = np.zeros(gid.size)
    lib().gsbo_r28_delta(_p(proj), _p(gid), _p(px), _p(py), gid.size, _p(out))
    return out


def compose_w2c(pose, mount) -> np.ndarray:
    """Reading R29: world->camera (3x4 f32) of a camera on a body at `pose` with body->camera
    `mount` (C implementation)."""
    p = _c(pose, np.float32).reshape(-1)
    b = _c(mount, np.float32).reshape(-1)
    out = np.zeros(12, np.float32)
    lib().gsbo_compose_w2c(_p(p), _p(b), _p(out))
    return out.reshape(3, 4)


def depth_key(w2c, pose_or_none, mu) -> np.float32:
    """R11 exact fp32 depth key of a single mean (C implementation)."""
    L = lib()
    w = _c(w2c, np.float32).reshape(-1)
    m = _c(mu, np.float32).reshape(-1)
    p = None if pose_or_none is None else _c(pose_or_none, np.float32).reshape(-1)
    return np.float32(L.gsbo_depth_key(_p(w), _p(p), _p(m)))


def sh_basis(deg: int, x: float, y: float, z: float) -> np.ndarray:
    Y = np.zeros(16)
    lib().gsbo_sh_basis(deg, x, y, z, _p(Y))
    return Y[: (deg + 1) ** 2]


# ------------------------------------------------------------------------------------------
# reading R32: batched ray-cast LiDAR against the Gaussians (§8(f) row 4; P:315, P:837-843,
# tab:lidar P:320-329).  See the R32 block of gsb_oracle.c for the step-by-step definition.
# ------------------------------------------------------------------------------------------
LF = 12
L_X, L_Y, L_Z, L_P00, L_P01, L_P02, L_P11, L_P12, L_P22, L_O, L_RHO32, L_RHO64 = range(LF)
TOL_ALPHA = 2e-3


@dataclass
class LidarResult:
    range: np.ndarray      # [R] sum_w w t^  (metres along the unit ray)
    alpha: np.ndarray      # [R] 1 - T
    masked: np.ndarray     # [R] reading-R28 threshold margin (range or alpha not compared)
    n_blend: np.ndarray    # [R] entries blended
    budget_range: np.ndarray
    budget_alpha: np.ndarray
    proj: np.ndarray       # [N, LF]
    rhobits: np.ndarray    # [N] u32 binary32 range key
    valid: np.ndarray      # [N] bool (R32 step 3)
    order: np.ndarray      # valid ids by (rhobits, id)


def lidar_project(scene, pose_env, w2s, near: float = 0.01, far: float = 1000.0):
    """R32 steps 1-3 for one (env, sensor): (proj [N,LF] f64, rhobits [N] u32, valid [N] bool)."""
    N = scene.n
    out = np.zeros((N, LF), np.float64)
    rb = np.zeros(N, np.uint32)
    valid = np.zeros(N, np.uint8)
    keep = [_c(scene.means, np.float32), _c(scene.scales, np.float32), _c(scene.quats, np.float32),
            _c(scene.opacities, np.float32), _c(scene.body_id, np.int32),
            _c(pose_env, np.float32).reshape(-1), _c(w2s, np.float32).reshape(-1)]
    rc = lib().gsbo_lidar_project(_p(keep[0]), _p(keep[1]), _p(keep[2]), _p(keep[3]), _p(keep[4]), N,
                                  _p(keep[5]), scene.n_bodies, _p(keep[6]), near, far, _p(out), _p(rb), _p(valid))
    if rc != 0:
        raise ValueError("oracle: body index out of range")
    return out, rb, valid.astype(bool)


def lidar_frame(scene, pose_env, w2s, dirs, near: float = 0.01, far: float = 1000.0,
                nthreads: Optional[int] = None, delta_alpha: float = DELTA_ALPHA,
                delta_T: float = DELTA_T) -> LidarResult:
    """R32 steps 1-6 for one (env, sensor) and the rays `dirs` [R,3] (unit, sensor frame)."""
    proj, rb, valid = lidar_project(scene, pose_env, w2s, near, far)
    order = depth_order(rb, valid)     # (bits(rho), id): R10 with rho for z
    dirs = _c(dirs, np.float32).reshape(-1, 3)
    R = dirs.shape[0]
    if order.size:
        kap = 2.0 * np.log(255.0 * scene.opacities[order].astype(np.float64))
        smax = np.abs(scene.scales[order].astype(np.float64)).max(axis=1)
        tmax = float((proj[order, L_RHO64] + np.sqrt(np.maximum(kap, 0.0)) * smax).max())
    else:
        tmax = 0.0
    rg = np.zeros(R); al = np.zeros(R); br = np.zeros(R); ba = np.zeros(R)
    nb = np.zeros(R, np.int64)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    lib().gsbo_lidar_cast(_p(proj), _p(order), order.size, _p(dirs), R, delta_alpha, delta_T, tmax,
                          _p(rg), _p(al), _p(br), _p(ba), _p(nb), int(nthreads))
    masked = (br > 0.5 * (TOL_DEPTH_REL * rg + TOL_DEPTH_ABS)) | (ba > 0.5 * TOL_ALPHA)
    return LidarResult(rg, al, masked, nb, br, ba, proj, rb, valid, order)


def range_key(w2s, pose_or_none, mu) -> np.float32:
    """R32 binary32 range key of a single mean (C implementation)."""
    w = _c(w2s, np.float32).reshape(-1)
    m = _c(mu, np.float32).reshape(-1)
    p = None if pose_or_none is None else _c(pose_or_none, np.float32).reshape(-1)
    return np.float32(lib().gsbo_range_key(_p(w), _p(p), _p(m)))


def lidar_peak(g_row, d):
    """(D2, t^) of one projected Gaussian row (LF fields) on the half-ray along d."""
    g = _c(g_row, np.float64).reshape(-1)
    dv = _c(d, np.float64).reshape(-1)
    th = np.zeros(1)
    D2 = lib().gsbo_lidar_peak(_p(g), _p(dv), _p(th))
    return float(D2), float(th[0])
