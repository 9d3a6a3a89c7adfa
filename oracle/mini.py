"""NumPy mini-oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py header).

An independent re-implementation of the same definition as gsb_oracle.c (pin 11 of
DESIGN.md §5: "two oracles"), written differently on purpose: vectorised over pixels,
looping over Gaussians in depth order; quaternion algebra via Hamilton products
instead of matrix formulas where possible.  fp64, except the R11 depth key, which is
computed with an exactly rounded binary32 FMA emulation (`fma32`).

Citations: PAPER.md App. B.2 Eqs. P:707-708 and Alg. 1 (pose), 3DGS formulation cited
at P:212 (projection, SH, compositing), north_star (alpha clamp 0.99, skip < 1/255,
depth-sorted brute force), readings R2-R19.
"""
from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------------------------------
# exactly rounded binary32 arithmetic used by reading R11
# ------------------------------------------------------------------------------------
def fma32(a, b, c) -> np.ndarray:
    """Correctly rounded float32 fma(a, b, c).

    a*b is exact in binary64 (24+24 bit significands); TwoSum gives the exact error e of
    s = fl64(a*b + c); rounding s to binary32 is then correct unless s sits exactly on a
    binary32 rounding midpoint, where the sign of e decides (no double-rounding)."""
    a64 = np.asarray(a, np.float32).astype(np.float64)
    b64 = np.asarray(b, np.float32).astype(np.float64)
    c64 = np.asarray(c, np.float32).astype(np.float64)
    p = a64 * b64
    s = p + c64
    bp = s - p
    e = (p - (s - bp)) + (c64 - bp)
    r = s.astype(np.float32)
    up = np.nextafter(r, np.float32(np.inf))
    dn = np.nextafter(r, np.float32(-np.inf))
    r64 = r.astype(np.float64)
    mid_up = s == (r64 + up.astype(np.float64)) / 2
    mid_dn = s == (r64 + dn.astype(np.float64)) / 2
    r = np.where(mid_up & (e > 0), up, r)
    r = np.where(mid_dn & (e < 0), dn, r)
    return r.astype(np.float32)


def _f(x):
    return np.float32(x)


def depth_key_f32(w2c, pose, mu) -> np.ndarray:
    """Reading R11 for an array of means (mu [...,3]) under one body pose (or None)."""
    w = np.asarray(w2c, np.float32).reshape(3, 4)
    mu = np.asarray(mu, np.float32)
    W20, W21, W22, t2 = w[2, 0], w[2, 1], w[2, 2], w[2, 3]
    if pose is None:
        M2 = [W20, W21, W22]
        m2 = t2
    else:
        pose = np.asarray(pose, np.float32)
        tx, ty, tz, qw, qx, qy, qz = [pose[..., j] for j in range(7)]
        two, one = _f(2.0), _f(1.0)
        xx, yy, zz = qx * qx, qy * qy, qz * qz
        xy, xz, yz = qx * qy, qx * qz, qy * qz
        wx, wy, wz = qw * qx, qw * qy, qw * qz
        R0 = [one - two * (yy + zz), two * (xy - wz), two * (xz + wy)]
        R1 = [two * (xy + wz), one - two * (xx + zz), two * (yz - wx)]
        R2 = [two * (xz - wy), two * (yz + wx), one - two * (xx + yy)]
        M2 = [fma32(W20, R0[c], fma32(W21, R1[c], W22 * R2[c])) for c in range(3)]
        m2 = fma32(W20, tx, fma32(W21, ty, fma32(W22, tz, t2)))
    return fma32(M2[0], mu[..., 0], fma32(M2[1], mu[..., 1], fma32(M2[2], mu[..., 2], m2)))


def compose_w2c_f32(pose, mount) -> np.ndarray:
    """Reading R29 in NumPy (independent of the C version): W = [B_R R^T | B_t - W t]."""
    pose = np.asarray(pose, np.float32).reshape(7)
    B = np.asarray(mount, np.float32).reshape(3, 4)
    tx, ty, tz, qw, qx, qy, qz = [pose[j] for j in range(7)]
    two, one = _f(2.0), _f(1.0)
    xx, yy, zz = qx * qx, qy * qy, qz * qz
    xy, xz, yz = qx * qy, qx * qz, qy * qz
    wx, wy, wz = qw * qx, qw * qy, qw * qz
    R = [[one - two * (yy + zz), two * (xy - wz), two * (xz + wy)],
         [two * (xy + wz), one - two * (xx + zz), two * (yz - wx)],
         [two * (xz - wy), two * (yz + wx), one - two * (xx + yy)]]
    W = np.zeros((3, 4), np.float32)
    for r in range(3):
        for c in range(3):
            W[r, c] = fma32(B[r, 0], R[c][0], fma32(B[r, 1], R[c][1], B[r, 2] * R[c][2]))
        W[r, 3] = fma32(-W[r, 0], tx, fma32(-W[r, 1], ty, fma32(-W[r, 2], tz, B[r, 3])))
    return W


# ------------------------------------------------------------------------------------
# fp64 geometry
# ------------------------------------------------------------------------------------
def _qmul(a, b):
    aw, av = a[..., :1], a[..., 1:]
    bw, bv = b[..., :1], b[..., 1:]
    w = aw * bw - np.sum(av * bv, -1, keepdims=True)
    v = aw * bv + bw * av + np.cross(av, bv)
    return np.concatenate([w, v], -1)


def _qrot(q, v):
    """Rotate vectors v by quaternion q via the Hamilton sandwich q (0,v) q*.
    (For the fp32-rounded, not exactly unit, per-frame quaternions this differs from the
    matrix formula of reading R22 by O(|q|^2 - 1) ~ 1e-7 relative; pin 11 accounts for it.)"""
    qc = q * np.array([1.0, -1.0, -1.0, -1.0])
    vq = np.concatenate([np.zeros(np.broadcast_shapes(v.shape[:-1], q.shape[:-1]) + (1,)),
                         np.broadcast_to(v, np.broadcast_shapes(v.shape[:-1], q.shape[:-1]) + (3,))], -1)
    return _qmul(_qmul(q, vq), qc)[..., 1:]


def _rotmat(q):
    """3x3 matrix of the linear map v -> q v q*, for unit q; built column by column."""
    e = np.eye(3)
    cols = [_qrot(q, e[j]) for j in range(3)]
    return np.stack(cols, -1)


SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def sh_eval(deg, coeffs, d):
    """R18: sum_j Y_j(d) c_j for d [N,3] unit, coeffs [N,(D+1)^2,3]."""
    x, y, z = d[:, 0:1], d[:, 1:2], d[:, 2:3]
    out = SH_C0 * coeffs[:, 0]
    if deg >= 1:
        out = out - SH_C1 * y * coeffs[:, 1] + SH_C1 * z * coeffs[:, 2] - SH_C1 * x * coeffs[:, 3]
    if deg >= 2:
        xx, yy, zz = x * x, y * y, z * z
        out = (out + SH_C2[0] * x * y * coeffs[:, 4] + SH_C2[1] * y * z * coeffs[:, 5]
               + SH_C2[2] * (2 * zz - xx - yy) * coeffs[:, 6] + SH_C2[3] * x * z * coeffs[:, 7]
               + SH_C2[4] * (xx - yy) * coeffs[:, 8])
    if deg >= 3:
        out = (out + SH_C3[0] * y * (3 * xx - yy) * coeffs[:, 9] + SH_C3[1] * x * y * z * coeffs[:, 10]
               + SH_C3[2] * y * (4 * zz - xx - yy) * coeffs[:, 11]
               + SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy) * coeffs[:, 12]
               + SH_C3[4] * x * (4 * zz - xx - yy) * coeffs[:, 13] + SH_C3[5] * z * (xx - yy) * coeffs[:, 14]
               + SH_C3[6] * x * (xx - 3 * yy) * coeffs[:, 15])
    return out


def project(scene, pose_env, intr, w2c, width, height, near=0.01, far=1000.0, sh_degree=None):
    """Per-Gaussian projected quantities for one frame (dict of arrays)."""
    D = scene.sh_degree if sh_degree is None else sh_degree
    N = scene.n
    mu = scene.means.astype(np.float64)
    body = scene.body_id.astype(np.int64)
    pose_env = np.asarray(pose_env, np.float32).reshape(-1, 7)
    qk = np.tile([1.0, 0.0, 0.0, 0.0], (N, 1))
    tk = np.zeros((N, 3))
    att = body >= 0
    if att.any():
        qk[att] = pose_env[body[att], 3:].astype(np.float64)
        tk[att] = pose_env[body[att], :3].astype(np.float64)
    # RLGK: p_world = R(q_k) p_local + t_k ; q_world = q_k (x) q_local
    muw = _qrot(qk, mu) + tk
    ql = scene.quats.astype(np.float64)
    ql = ql / np.linalg.norm(ql, axis=1, keepdims=True)
    qw = _qmul(qk, ql)
    Rw = _rotmat(qw)                                   # [N,3,3]
    S = scene.scales.astype(np.float64)
    Sigma_w = np.einsum("nij,nj,nkj->nik", Rw, S * S, Rw)
    w = np.asarray(w2c, np.float64).reshape(3, 4)
    Wr, tc = w[:, :3], w[:, 3]
    xc = muw @ Wr.T + tc
    z = xc[:, 2]
    fx, fy, cx, cy = [float(v) for v in np.asarray(intr, np.float64).reshape(4)]
    u = fx * xc[:, 0] / z + cx
    v = fy * xc[:, 1] / z + cy
    limx, limy = 1.3 * width / (2 * fx), 1.3 * height / (2 * fy)
    txz = np.clip(xc[:, 0] / z, -limx, limx)
    tyz = np.clip(xc[:, 1] / z, -limy, limy)
    J = np.zeros((N, 2, 3))
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = -fx * txz / z
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = -fy * tyz / z
    Sc = np.einsum("ij,njk,lk->nil", Wr, Sigma_w, Wr)
    S2 = np.einsum("nij,njk,nlk->nil", J, Sc, J) + 0.3 * np.eye(2)
    det = S2[:, 0, 0] * S2[:, 1, 1] - S2[:, 0, 1] ** 2
    conic = np.stack([S2[:, 1, 1] / det, -S2[:, 0, 1] / det, S2[:, 0, 0] / det], 1)
    # exact fp32 depth key, per body (R11)
    z32 = np.empty(N, np.float32)
    st = ~att
    if st.any():
        z32[st] = depth_key_f32(w2c, None, scene.means[st])
    for k in np.unique(body[att]):
        sel = body == k
        z32[sel] = depth_key_f32(w2c, pose_env[k], scene.means[sel])
    o = scene.opacities.astype(np.float64)
    valid = (z32 > np.float32(near)) & (z32 <= np.float32(far)) & (o >= 1.0 / 255.0)
    # colour in the body frame (R19): camera centre -> body frame via q_k*
    cw = -Wr.T @ tc
    qinv = qk * np.array([1.0, -1.0, -1.0, -1.0])
    cb = _qrot(qinv, cw[None, :] - tk)
    d = mu - cb
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rgb = np.maximum(sh_eval(D, scene.sh.astype(np.float64), d) + 0.5, 0.0)
    return dict(u=u, v=v, conic=conic, S2=S2, rgb=rgb, o=o, z32=z32, valid=valid,
                kappa=2 * np.log(255 * o))


def render(scene, pose_env, intr, w2c, width, height, near=0.01, far=1000.0, bg=(0, 0, 0), sh_degree=None):
    """Full-frame brute-force composite (vectorised over pixels)."""
    pr = project(scene, pose_env, intr, w2c, width, height, near, far, sh_degree)
    ids = np.nonzero(pr["valid"])[0]
    zb = pr["z32"].view(np.uint32)
    order = ids[np.lexsort((ids, zb[ids]))]
    py, px = np.meshgrid(np.arange(height) + 0.5, np.arange(width) + 0.5, indexing="ij")
    T = np.ones((height, width))
    C = np.zeros((height, width, 3))
    Dp = np.zeros((height, width))
    alive = np.ones((height, width), bool)
    term = -np.ones((height, width), np.int64)
    for i in order:
        dx = pr["u"][i] - px
        dy = pr["v"][i] - py
        a, b, c = pr["conic"][i]
        power = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
        alpha = np.minimum(0.99, pr["o"][i] * np.exp(power))
        use = alive & (power <= 0) & (alpha >= 1.0 / 255.0)
        tT = T * (1 - alpha)
        stop = use & (tT < 1e-4)
        term[stop] = i
        alive &= ~stop
        blend = use & ~stop
        wgt = np.where(blend, alpha * T, 0.0)
        C += wgt[..., None] * pr["rgb"][i]
        Dp += wgt * float(pr["z32"][i])
        T = np.where(blend, tT, T)
        if not alive.any():
            break
    rgb = C + T[..., None] * np.asarray(bg, np.float64)
    return dict(rgb=rgb, depth=Dp, alpha=1 - T, term_id=term, proj=pr, order=order)
