"""Seeded synthetic workloads for the batched 3DGS hot path (shared input module).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle.  It holds none of the method's arithmetic (no projection, no SH, no
binning, no compositing); it only draws inputs: a Gaussian scene template, per-env
rigid body poses S_t in R^{B x N_bodies x 7} (App. B.2) and per-env
camera intrinsics/extrinsics with the paper's camera domain randomisation
(App. D.2: +-0.02 m per axis, rotation about a random axis by <= 5 deg).

Recipe: SURVEY.md §8(d) d.2 (restated in DESIGN.md §3).  RNG streams are keyed by
config id and by the GLOBAL env id, so batch size and sharding never change an
env's inputs.

Conventions (readings R2, R21, R22):
  * quaternions are scalar-first Hamilton (w, x, y, z)
  * pose vector = (tx, ty, tz, qw, qx, qy, qz), world <- body
  * world_to_cam = [R | t] row-major 3x4, OpenCV axes (x right, y down, z fwd)
  * body_id = -1 for static (world) Gaussians, else 0-based body index
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional, Tuple

import numpy as np

SH_C0 = 0.28209479177387814  # only used to turn a target DC colour into a coefficient


# --------------------------------------------------------------------------------------
# small fp64 rotation helpers (input generation only: FK of the synthetic robot and the
# look-at / DR of the synthetic cameras)
# --------------------------------------------------------------------------------------
def _quat_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    aw, ax, ay, az = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    bw, bx, by, bz = b[..., 0], b[..., 1], b[..., 2], b[..., 3]
    return np.stack([
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    ], axis=-1)


def _axis_angle_quat(axis: np.ndarray, angle: np.ndarray) -> np.ndarray:
    axis = np.asarray(axis, np.float64)
    axis = axis / np.linalg.norm(axis, axis=-1, keepdims=True)
    h = 0.5 * np.asarray(angle, np.float64)
    return np.concatenate([np.cos(h)[..., None], np.sin(h)[..., None] * axis], axis=-1)


def _quat_to_mat(q: np.ndarray) -> np.ndarray:
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def _mat_to_quat(R: np.ndarray) -> np.ndarray:
    """Rotation matrix -> unit quaternion (w,x,y,z), w >= 0 (Shepperd's method)."""
    R = np.asarray(R, np.float64)
    out = np.empty(R.shape[:-2] + (4,))
    flat_R = R.reshape(-1, 3, 3)
    flat_q = out.reshape(-1, 4)
    for n in range(flat_R.shape[0]):
        m = flat_R[n]
        tr = m[0, 0] + m[1, 1] + m[2, 2]
        if tr > 0:
            s = math.sqrt(tr + 1.0) * 2
            q = [0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s]
        elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
            s = math.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2
            q = [(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s]
        elif m[1, 1] > m[2, 2]:
            s = math.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2
            q = [(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s]
        else:
            s = math.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2
            q = [(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s]
        q = np.array(q)
        if q[0] < 0:
            q = -q
        flat_q[n] = q / np.linalg.norm(q)
    return out


def _frame_from_normal(normal: np.ndarray, angle: np.ndarray) -> np.ndarray:
    """Quaternions whose local +z maps to `normal`, with a random in-plane angle."""
    n = normal / np.linalg.norm(normal, axis=-1, keepdims=True)
    helper = np.where(np.abs(n[..., 2:3]) < 0.9, np.array([0.0, 0.0, 1.0]), np.array([1.0, 0.0, 0.0]))
    t1 = np.cross(helper, n)
    t1 /= np.linalg.norm(t1, axis=-1, keepdims=True)
    t2 = np.cross(n, t1)
    c, s = np.cos(angle)[..., None], np.sin(angle)[..., None]
    e1 = c * t1 + s * t2
    e2 = np.cross(n, e1)
    R = np.stack([e1, e2, n], axis=-1)  # columns = local axes in world
    return _mat_to_quat_vec(R)


def _mat_to_quat_vec(R: np.ndarray) -> np.ndarray:
    """Vectorised rotation-matrix -> quaternion (w,x,y,z) for proper rotations."""
    m00, m11, m22 = R[..., 0, 0], R[..., 1, 1], R[..., 2, 2]
    qw = np.sqrt(np.maximum(0.0, 1 + m00 + m11 + m22)) / 2
    qx = np.sqrt(np.maximum(0.0, 1 + m00 - m11 - m22)) / 2
    qy = np.sqrt(np.maximum(0.0, 1 - m00 + m11 - m22)) / 2
    qz = np.sqrt(np.maximum(0.0, 1 - m00 - m11 + m22)) / 2
    qx = np.copysign(qx, R[..., 2, 1] - R[..., 1, 2])
    qy = np.copysign(qy, R[..., 0, 2] - R[..., 2, 0])
    qz = np.copysign(qz, R[..., 1, 0] - R[..., 0, 1])
    q = np.stack([qw, qx, qy, qz], axis=-1)
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def _random_rotations(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    return q


# --------------------------------------------------------------------------------------
# workload configurations (BASELINE.json "configs"; SURVEY §8 size table)
# --------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int
    n_envs: int
    n_cams: int
    width: int
    height: int
    n_bg: int
    n_bodies: int
    per_body: int
    sh_degree: int
    kind: str = "room"          # "room" (C2-C5 recipe) or "box" (C1 recipe)
    fov60: bool = False         # C4: 60 deg FOV intrinsics

    @property
    def n_rb(self) -> int:
        return self.n_bodies * self.per_body

    @property
    def n_gaussians(self) -> int:
        return self.n_bg + self.n_rb

    @property
    def n_frames(self) -> int:
        return self.n_envs * self.n_cams


CONFIGS: Dict[str, Config] = {
    # BASELINE.json configs[0..4]
    "C1": Config("C1", 1, 1, 1, 64, 48, 1000, 0, 0, 0, kind="box"),
    "C2": Config("C2", 2, 64, 1, 640, 480, 100_000, 10, 2000, 3),
    "C3": Config("C3", 3, 1024, 1, 640, 480, 500_000, 10, 2000, 3),
    "C4": Config("C4", 4, 4096, 2, 128, 128, 180_000, 10, 2000, 3, fov60=True),
    "C5": Config("C5", 5, 8192, 1, 640, 480, 980_000, 10, 2000, 3),
    # §8(f) row 4 second workloads: 224x224 policy views (ViT input) and a 1280x720 sweep
    # point, both on the C3 scene
    "C6": Config("C6", 6, 4096, 1, 224, 224, 500_000, 10, 2000, 3, fov60=True),
    "C7": Config("C7", 7, 256, 1, 1280, 720, 500_000, 10, 2000, 3),
    # parity-test configs: oracle finishes in seconds, several tiles + ragged tail
    "T1": Config("T1", 11, 3, 2, 100, 75, 6000, 10, 200, 3),
    "T2": Config("T2", 12, 2, 1, 130, 97, 20000, 10, 300, 3),
    "T3": Config("T3", 13, 4, 1, 48, 40, 3000, 0, 0, 0),
    "T4": Config("T4", 14, 2, 2, 64, 64, 8000, 10, 200, 1, fov60=True),
    "T5": Config("T5", 15, 2, 1, 160, 120, 12000, 10, 200, 2),
    # long tile lists (C4-like density at parity size): exercises K4's large-capacity variant
    "T6": Config("T6", 16, 2, 2, 64, 64, 40000, 10, 200, 3, fov60=True),
    # robot-dominated tile lists (thousands of robot Gaussians in a few tiles): the static-camera
    # merge path with robot lists beyond K4's fused-sort capacity
    "T7": Config("T7", 17, 3, 1, 64, 64, 2000, 2, 3000, 1, fov60=True),
}


# --------------------------------------------------------------------------------------
# scene template
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class Scene:
    means: np.ndarray      # [N,3] f32 body-local (body_id>=0) or world (body_id=-1), metres
    scales: np.ndarray     # [N,3] f32 linear sigma > 0
    quats: np.ndarray      # [N,4] f32 (w,x,y,z)
    opacities: np.ndarray  # [N]   f32 in (0,1]
    sh: np.ndarray         # [N,(D+1)^2,3] f32 coefficient-major
    sh_degree: int
    body_id: np.ndarray    # [N] int32, -1 = static
    n_bodies: int

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx: np.ndarray) -> "Scene":
        return Scene(self.means[idx], self.scales[idx], self.quats[idx], self.opacities[idx],
                     self.sh[idx], self.sh_degree, self.body_id[idx], self.n_bodies)


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _room_background(rng: np.random.Generator, n_bg: int, n_coef: int):
    """Floor z=0 over [-3,3]^2 plus four 6 x 2.5 m walls (SURVEY d.2 'Background room')."""
    areas = np.array([36.0, 15.0, 15.0, 15.0, 15.0])
    counts = np.floor(n_bg * areas / areas.sum()).astype(int)
    counts[0] += n_bg - counts.sum()
    pos, nrm = [], []
    # floor
    k = counts[0]
    pos.append(np.stack([rng.uniform(-3, 3, k), rng.uniform(-3, 3, k), np.zeros(k)], 1))
    nrm.append(np.tile([0.0, 0.0, 1.0], (k, 1)))
    # walls: x=+3, x=-3, y=+3, y=-3 (normals point inward)
    for w, (axis, sign) in enumerate([(0, 1.0), (0, -1.0), (1, 1.0), (1, -1.0)]):
        k = counts[1 + w]
        p = np.zeros((k, 3))
        p[:, axis] = 3.0 * sign
        p[:, 1 - axis] = rng.uniform(-3, 3, k)
        p[:, 2] = rng.uniform(0, 2.5, k)
        n = np.zeros((k, 3))
        n[:, axis] = -sign
        pos.append(p)
        nrm.append(n)
    pos = np.concatenate(pos)
    nrm = np.concatenate(nrm)
    pos += nrm * rng.normal(0, 0.005, (n_bg, 1))
    quats = _frame_from_normal(nrm, rng.uniform(0, 2 * np.pi, n_bg))
    s0 = 0.8 * math.sqrt(96.0 / n_bg)
    scales = np.empty((n_bg, 3))
    scales[:, 0] = s0 * np.exp(rng.normal(0, 0.35, n_bg))
    scales[:, 1] = s0 * np.exp(rng.normal(0, 0.35, n_bg))
    scales[:, 2] = 0.15 * s0 * np.exp(rng.normal(0, 0.35, n_bg))
    giants = rng.random(n_bg) < 0.01
    scales[giants] *= 6.0
    opac = np.clip(_sigmoid(rng.normal(2.0, 1.5, n_bg)), 0.004, 0.999)
    kvec = rng.normal(0, 1.0, (3, 3))
    phase = rng.uniform(0, 2 * np.pi, 3)
    col = 0.5 + 0.35 * np.sin(2 * np.pi * pos @ kvec.T + phase)
    sh = np.zeros((n_bg, n_coef, 3))
    sh[:, 0, :] = (col - 0.5) / SH_C0
    if n_coef > 1:
        sh[:, 1:, :] = rng.normal(0, 0.03, (n_bg, n_coef - 1, 3))
    return pos, scales, quats, opac, sh


def _box_background(rng: np.random.Generator, n: int, n_coef: int):
    """C1 recipe: static Gaussians uniform in a box in front of an identity camera."""
    pos = np.stack([rng.uniform(-1, 1, n), rng.uniform(-0.75, 0.75, n), rng.uniform(2, 4, n)], 1)
    sig = np.exp(rng.uniform(math.log(0.03), math.log(0.08), (n, 3)))
    quats = _random_rotations(rng, n)
    opac = rng.uniform(0.05, 0.99, n)
    col = rng.uniform(0.1, 0.9, (n, 3))
    sh = np.zeros((n, n_coef, 3))
    sh[:, 0, :] = (col - 0.5) / SH_C0
    if n_coef > 1:
        sh[:, 1:, :] = rng.normal(0, 0.03, (n, n_coef - 1, 3))
    return pos, sig, quats, opac, sh


def _robot(rng: np.random.Generator, n_bodies: int, per_body: int, n_coef: int):
    """Capsule links along local x (r=4 cm, half-length 12 cm, centre (0.15,0,0))."""
    r, h, cx = 0.04, 0.12, 0.15
    n = n_bodies * per_body
    a_cyl, a_cap = 2 * np.pi * r * 2 * h, 4 * np.pi * r * r
    on_cyl = rng.random(n) < a_cyl / (a_cyl + a_cap)
    pos = np.empty((n, 3))
    nrm = np.empty((n, 3))
    phi = rng.uniform(0, 2 * np.pi, n)
    xs = rng.uniform(-h, h, n)
    nrm_c = np.stack([np.zeros(n), np.cos(phi), np.sin(phi)], 1)
    pos_c = np.stack([cx + xs, r * np.cos(phi), r * np.sin(phi)], 1)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    end = np.where(d[:, 0:1] >= 0, cx + h, cx - h)
    pos_s = np.concatenate([end + r * d[:, 0:1], r * d[:, 1:]], 1)
    pos[:] = np.where(on_cyl[:, None], pos_c, pos_s)
    nrm[:] = np.where(on_cyl[:, None], nrm_c, d)
    quats = _frame_from_normal(nrm, rng.uniform(0, 2 * np.pi, n))
    scales = np.empty((n, 3))
    scales[:, 0] = 0.006 * np.exp(rng.normal(0, 0.25, n))
    scales[:, 1] = 0.006 * np.exp(rng.normal(0, 0.25, n))
    scales[:, 2] = 0.0015
    opac = _sigmoid(rng.normal(3.0, 1.0, n))
    palette = rng.uniform(0.15, 0.85, (n_bodies, 3))
    body = np.repeat(np.arange(n_bodies), per_body)
    col = np.clip(palette[body] + rng.normal(0, 0.03, (n, 3)), 0.0, 1.0)
    sh = np.zeros((n, n_coef, 3))
    sh[:, 0, :] = (col - 0.5) / SH_C0
    if n_coef > 1:
        sh[:, 1:, :] = rng.normal(0, 0.03, (n, n_coef - 1, 3))
    return pos, scales, quats, opac, sh, body


def make_scene(cfg: Config) -> Scene:
    """Scene template for `cfg` (seed 1000 + cfg_id).  Static Gaussians first, then
    robot Gaussians grouped by body (creation index = global Gaussian id)."""
    rng = np.random.default_rng(1000 + cfg.cfg_id)
    n_coef = (cfg.sh_degree + 1) ** 2
    if cfg.kind == "box":
        pos, sc, q, o, sh = _box_background(rng, cfg.n_bg, n_coef)
    else:
        pos, sc, q, o, sh = _room_background(rng, cfg.n_bg, n_coef)
    body = -np.ones(cfg.n_bg, np.int64)
    if cfg.n_bodies > 0:
        rp, rs, rq, ro, rsh, rb = _robot(rng, cfg.n_bodies, cfg.per_body, n_coef)
        pos = np.concatenate([pos, rp])
        sc = np.concatenate([sc, rs])
        q = np.concatenate([q, rq])
        o = np.concatenate([o, ro])
        sh = np.concatenate([sh, rsh])
        body = np.concatenate([body, rb])
    return Scene(
        means=np.ascontiguousarray(pos, np.float32),
        scales=np.ascontiguousarray(sc, np.float32),
        quats=np.ascontiguousarray(q, np.float32),
        opacities=np.ascontiguousarray(o, np.float32),
        sh=np.ascontiguousarray(sh, np.float32),
        sh_degree=cfg.sh_degree,
        body_id=np.ascontiguousarray(body, np.int32),
        n_bodies=cfg.n_bodies,
    )


# --------------------------------------------------------------------------------------
# per-env body poses S_t (synthetic stand-in for the physics engine)
# --------------------------------------------------------------------------------------
JOINT_AXES = np.array([[0, 0, 1], [0, 1, 0], [0, 1, 0], [1, 0, 0], [0, 1, 0],
                       [0, 1, 0], [1, 0, 0], [0, 1, 0], [0, 1, 0], [1, 0, 0]], np.float64)


def env_phases(cfg: Config, env: int) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence(2000 + cfg.cfg_id, spawn_key=(env,)))
    return rng.uniform(0, 2 * np.pi, max(cfg.n_bodies, 1))[: cfg.n_bodies]


def make_poses(cfg: Config, env_ids, step: int) -> np.ndarray:
    """Body poses [len(env_ids), n_bodies, 7] (tx,ty,tz,qw,qx,qy,qz), world <- body.
    Serial chain: base at (0,0,0.05), joint axes z,y,y,x,y,y,x,y,y,x, link offset 0.3 m,
    theta_j = 0.6 sin(0.9 (j+1) 0.02 s + phi_{e,j}); FK in fp64, rounded to fp32."""
    env_ids = np.asarray(env_ids, np.int64).reshape(-1)
    nb = cfg.n_bodies
    out = np.zeros((env_ids.size, nb, 7), np.float64)
    if nb == 0:
        return out.astype(np.float32)
    phases = np.stack([env_phases(cfg, int(e)) for e in env_ids])       # [B, nb]
    j = np.arange(nb)
    theta = 0.6 * np.sin(0.9 * (j + 1) * 0.02 * step + phases)         # [B, nb]
    axes = JOINT_AXES[np.arange(nb) % len(JOINT_AXES)]
    q_joint = _axis_angle_quat(np.broadcast_to(axes, theta.shape + (3,)), theta)
    t = np.broadcast_to(np.array([0.0, 0.0, 0.05]), (env_ids.size, 3)).copy()
    q = q_joint[:, 0]
    out[:, 0, :3], out[:, 0, 3:] = t, q
    for k in range(1, nb):
        R = _quat_to_mat(q)
        t = t + R @ np.array([0.3, 0.0, 0.0])
        q = _quat_mul(q, q_joint[:, k])
        q /= np.linalg.norm(q, axis=-1, keepdims=True)
        out[:, k, :3], out[:, k, 3:] = t, q
    return out.astype(np.float32)


def make_pose_steps(cfg: Config, env_ids, steps: int, first_step: int = 0) -> np.ndarray:
    return np.stack([make_poses(cfg, env_ids, first_step + s) for s in range(steps)])


# --------------------------------------------------------------------------------------
# per-env cameras (App. D.2 P:891 domain randomisation)
# --------------------------------------------------------------------------------------
NOMINAL_CAMS = [((2.0, -1.5, 1.3), (0.0, 0.0, 0.5)), ((-1.2, -1.8, 1.6), (0.0, 0.0, 0.4))]


def intrinsics_for(cfg: Config) -> np.ndarray:
    W, H = cfg.width, cfg.height
    if cfg.fov60:
        f = (W / 2) / math.tan(math.radians(30.0))
    else:
        f = 525.0 * W / 640.0
    return np.array([f, f, W / 2.0, H / 2.0], np.float64)


def _look_at_c2w(eye, target) -> np.ndarray:
    eye, target = np.asarray(eye, float), np.asarray(target, float)
    fwd = target - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, [0.0, 0.0, 1.0])
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], axis=1)  # columns: cam axes in world


def make_cameras(cfg: Config, env_ids) -> Tuple[np.ndarray, np.ndarray]:
    """(intrinsics [B,C,4] f32, world_to_cam [B,C,3,4] f32) for the given global env ids."""
    env_ids = np.asarray(env_ids, np.int64).reshape(-1)
    B, C = env_ids.size, cfg.n_cams
    K = np.broadcast_to(intrinsics_for(cfg), (B, C, 4)).astype(np.float32).copy()
    W2C = np.zeros((B, C, 3, 4), np.float64)
    for bi, e in enumerate(env_ids):
        for c in range(C):
            if cfg.kind == "box":
                Rc2w, eye = np.eye(3), np.zeros(3)
            else:
                eye0, tgt = NOMINAL_CAMS[c % len(NOMINAL_CAMS)]
                Rc2w = _look_at_c2w(eye0, tgt)
                rng = np.random.default_rng(np.random.SeedSequence(3000 + cfg.cfg_id, spawn_key=(int(e), c)))
                eye = np.asarray(eye0) + rng.uniform(-0.02, 0.02, 3)
                axis = rng.normal(size=3)
                ang = math.radians(rng.uniform(0.0, 5.0))
                Rc2w = _quat_to_mat(_axis_angle_quat(axis, ang)) @ Rc2w
            R = Rc2w.T
            W2C[bi, c, :, :3] = R
            W2C[bi, c, :, 3] = -R @ eye
    return K, W2C.astype(np.float32)


def static_cameras(cfg: Config) -> Tuple[np.ndarray, np.ndarray]:
    """Cameras fixed in the world (§8(f) row 2): env 0's cameras, shared by every env.
    (intrinsics [C,4] f32, world_to_cam [C,3,4] f32)."""
    K, W2C = make_cameras(cfg, [0])
    return K[0].copy(), W2C[0].copy()


@dataclasses.dataclass
class Batch:
    poses: np.ndarray       # [B, nb, 7] f32
    intrinsics: np.ndarray  # [B, C, 4] f32
    w2c: np.ndarray         # [B, C, 3, 4] f32


def make_batch(cfg: Config, env_ids=None, step: int = 0) -> Batch:
    if env_ids is None:
        env_ids = np.arange(cfg.n_envs)
    K, W2C = make_cameras(cfg, env_ids)
    return Batch(make_poses(cfg, env_ids, step), K, W2C)


def env_slice(n_envs: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous env slice of rank r: [r*B/G, (r+1)*B/G)."""
    lo = (n_envs * rank) // world
    hi = (n_envs * (rank + 1)) // world
    return lo, hi


def sample_pixels(width: int, height: int, seed: int, grid: int = 64, full_tiles: int = 2):
    """Pixel sample of one frame for the full-size parity checks and the oracle timing
    (SURVEY §8(d) d.6): one uniformly drawn pixel in each cell of a grid x grid partition of
    the image (4096 stratified pixels at grid = 64), plus every pixel of `full_tiles` distinct
    16x16 tiles drawn uniformly (ragged edge tiles included).  Returns (px, py, n_strat) int64;
    the first n_strat entries are the stratified ones."""
    rng = np.random.default_rng(seed)
    gx = min(grid, width)
    gy = min(grid, height)
    cx, cy = np.meshgrid(np.arange(gx), np.arange(gy))
    cx, cy = cx.reshape(-1), cy.reshape(-1)
    x0, x1 = (cx * width) // gx, ((cx + 1) * width) // gx
    y0, y1 = (cy * height) // gy, ((cy + 1) * height) // gy
    px = x0 + (rng.random(cx.size) * (x1 - x0)).astype(np.int64)
    py = y0 + (rng.random(cy.size) * (y1 - y0)).astype(np.int64)
    tw, th = (width + 15) // 16, (height + 15) // 16
    tiles = rng.choice(tw * th, size=min(full_tiles, tw * th), replace=False)
    tx, ty = [px], [py]
    for t in tiles:
        x_lo, y_lo = (t % tw) * 16, (t // tw) * 16
        yy, xx = np.meshgrid(np.arange(y_lo, min(y_lo + 16, height)), np.arange(x_lo, min(x_lo + 16, width)),
                             indexing="ij")
        tx.append(xx.reshape(-1))
        ty.append(yy.reshape(-1))
    return np.concatenate(tx).astype(np.int64), np.concatenate(ty).astype(np.int64), int(px.size)


# --------------------------------------------------------------------------------------
# LiDAR inputs (§8(f) row 4, reading R32; tab:lidar P:320-329): ray patterns in the sensor
# frame (x forward, y left, z up) and sensor extrinsics.  Inputs only: no method arithmetic.
# --------------------------------------------------------------------------------------
def lidar_pattern(kind: str, n_channels: int = 32, n_azimuth: int = 1024, step: int = 0,
                  fov=(-25.0, 15.0), n_points: int = 0, seed: int = 0) -> np.ndarray:
    """Unit ray directions [R,3] f32.
    rotating:        n_channels elevations uniform in fov (deg) x n_azimuth azimuths over 360 deg
    solid_state:     a bounded n_channels x n_azimuth grid, +-35 deg azimuth, elevation fov
    non_repetitive:  a rose-curve (Livox-like) scan of n_points rays over a 70 deg cone whose
                     phase advances with `step`, so successive scans cover different directions
    height_scan:     a downward n_channels x n_azimuth grid (1.6 x 1.0 m at 1 m below the
                     sensor), the Height Scan sensor of P:837
    random:          n_points directions uniform on the sphere (seeded)"""
    if kind == "rotating":
        el = np.radians(np.linspace(fov[0], fov[1], n_channels))
        az = np.linspace(-np.pi, np.pi, n_azimuth, endpoint=False) + np.pi / n_azimuth
        E, A = np.meshgrid(el, az, indexing="ij")
    elif kind == "solid_state":
        el = np.radians(np.linspace(fov[0], fov[1], n_channels))
        az = np.radians(np.linspace(-35.0, 35.0, n_azimuth))
        E, A = np.meshgrid(el, az, indexing="ij")
    elif kind == "non_repetitive":
        n = n_points or n_channels * n_azimuth
        t = np.arange(n) * (2 * np.pi / n) * 17.0 + 0.37 * step
        r = np.radians(35.0) * np.abs(np.sin(2.5 * t + 0.11 * step))
        ang = t * 0.5
        y, z = r * np.cos(ang), r * np.sin(ang)
        d = np.stack([np.ones(n), np.tan(y), np.tan(z)], 1)
        return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    elif kind == "height_scan":
        xs = np.linspace(-0.8, 0.8, n_azimuth)
        ys = np.linspace(-0.5, 0.5, n_channels)
        Y, X = np.meshgrid(ys, xs, indexing="ij")
        d = np.stack([X.ravel(), Y.ravel(), -np.ones(X.size)], 1)
        return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    elif kind == "random":
        rng = np.random.default_rng(seed)
        d = rng.normal(size=(n_points or n_channels * n_azimuth, 3))
        return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    else:
        raise ValueError(kind)
    d = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], -1).reshape(-1, 3)
    return (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)


def lidar_world_sensor(cfg: Config, env_ids) -> np.ndarray:
    """World->sensor [B,3,4] f32 of a LiDAR fixed in the room near the robot (1.2 m above the
    floor at (1.0, -0.8), facing the robot, yawed per env by U(+-10 deg))."""
    env_ids = np.asarray(env_ids, np.int64).reshape(-1)
    out = np.zeros((env_ids.size, 3, 4), np.float64)
    for bi, e in enumerate(env_ids):
        rng = np.random.default_rng(np.random.SeedSequence(4000 + cfg.cfg_id, spawn_key=(int(e),)))
        yaw = math.atan2(0.8, -1.0) + math.radians(rng.uniform(-10.0, 10.0))
        c, s = math.cos(yaw), math.sin(yaw)
        Rs2w = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])  # sensor x forward, z up
        eye = np.array([1.0, -0.8, 1.2]) + rng.uniform(-0.02, 0.02, 3)
        out[bi, :, :3] = Rs2w.T
        out[bi, :, 3] = -Rs2w.T @ eye
    return out.astype(np.float32)


def lidar_body_mount() -> np.ndarray:
    """Body->sensor [3,4] f32 of a LiDAR on body 0 (the robot base): 0.2 m above the body
    origin, axes aligned with the body (reading R29 composes it per env on the device)."""
    m = np.zeros((3, 4), np.float32)
    m[:, :3] = np.eye(3)
    m[:, 3] = [0.0, 0.0, -0.2]
    return m
