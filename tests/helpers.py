"""Small hand-built scenes for closed-form pins (inputs only; no method arithmetic)."""
import numpy as np

import synth

C0 = 0.28209479177387814  # SH DC constant (reading R18), used to encode a target colour


def scene_from(means, scales, quats=None, opac=None, colours=None, body=None, n_bodies=0, sh_degree=0,
               sh_rest=None):
    means = np.asarray(means, np.float32).reshape(-1, 3)
    n = means.shape[0]
    scales = np.broadcast_to(np.asarray(scales, np.float32), (n, 3)).copy()
    quats = np.tile(np.float32([1, 0, 0, 0]), (n, 1)) if quats is None else np.asarray(quats, np.float32).reshape(n, 4)
    opac = np.full(n, 0.5, np.float32) if opac is None else np.broadcast_to(np.asarray(opac, np.float32), (n,)).copy()
    colours = np.full((n, 3), 0.5) if colours is None else np.broadcast_to(np.asarray(colours, np.float64), (n, 3))
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3), np.float32)
    sh[:, 0, :] = (colours - 0.5) / C0
    if sh_rest is not None:
        sh[:, 1:, :] = sh_rest
    body = -np.ones(n, np.int32) if body is None else np.broadcast_to(np.asarray(body, np.int32), (n,)).copy()
    return synth.Scene(means, scales, quats, opac, sh, sh_degree, body, n_bodies)


def identity_cam(fx=100.0, fy=100.0, cx=32.5, cy=24.5):
    K = np.float32([fx, fy, cx, cy])
    W = np.zeros((3, 4), np.float32)
    W[:, :3] = np.eye(3)
    return K, W


def random_tiny_scene(rng, n, n_bodies=0, sh_degree=0):
    means = np.stack([rng.uniform(-0.6, 0.6, n), rng.uniform(-0.6, 0.6, n), rng.uniform(1.5, 3.0, n)], 1)
    scales = np.exp(rng.uniform(np.log(0.02), np.log(0.2), (n, 3)))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    opac = rng.uniform(0.02, 1.0, n)
    col = rng.uniform(0, 1, (n, 3))
    body = rng.integers(-1, n_bodies, n) if n_bodies > 0 else None
    rest = rng.normal(0, 0.2, (n, (sh_degree + 1) ** 2 - 1, 3)) if sh_degree > 0 else None
    return scene_from(means, scales, q, opac, col, body, n_bodies, sh_degree, rest)


def random_pose(rng, n_bodies):
    t = rng.normal(0, 0.1, (n_bodies, 3))
    q = rng.normal(size=(n_bodies, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return np.concatenate([t, q], 1).astype(np.float32)
