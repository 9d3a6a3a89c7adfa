"""Pins of the reading-R32 ray-cast LiDAR oracle (P:315, P:837-843,
tab:lidar P:320-329) against things other than itself: closed forms of a Gaussian on a ray,
brute-force minimisation along the ray, Porter-Duff stacking, the termination rule, rigid
invariance, and an exactly rounded re-computation of the binary32 range key.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import mini
from tests.helpers import random_pose, random_tiny_scene, scene_from

I34 = np.hstack([np.eye(3), np.zeros((3, 1))]).astype(np.float32)


def _cast(scene, dirs, W=I34, pose=None, **kw):
    pose = np.zeros((max(scene.n_bodies, 0), 7), np.float32) if pose is None else pose
    return oracle.lidar_frame(scene, pose, W, np.asarray(dirs, np.float32).reshape(-1, 3), nthreads=2, **kw)


def _unit(v):
    v = np.asarray(v, np.float64)
    return (v / np.linalg.norm(v)).astype(np.float32)


def test_lidar_isotropic_on_ray_closed_form():
    """Isotropic Gaussian at distance r on the ray: t^ = r, D2 = 0, alpha = min(0.99, o),
    range = alpha r (R32 step 5)."""
    r, s, o = 3.0, 0.05, 0.7
    sc = scene_from([r, 0, 0], s, opac=o)
    res = _cast(sc, [[1, 0, 0]])
    o32 = float(np.float32(o))
    assert res.alpha[0] == pytest.approx(o32, rel=1e-12)
    assert res.range[0] == pytest.approx(o32 * r, rel=1e-12)
    assert res.n_blend[0] == 1
    # opacity above the clamp
    res = _cast(scene_from([r, 0, 0], s, opac=1.0), [[1, 0, 0]])
    assert res.alpha[0] == pytest.approx(0.99, rel=1e-15)


@pytest.mark.parametrize("phi_deg", [0.3, 1.0, 2.0])
def test_lidar_isotropic_off_axis_closed_form(phi_deg):
    """A ray at angle phi from an isotropic Gaussian's centre direction: the peak is at
    t* = r cos(phi) with D2 = (r sin(phi) / s)^2 (distance from a point to a line)."""
    r, s, o = 2.0, 0.04, 0.9
    phi = math.radians(phi_deg)
    sc = scene_from([r, 0, 0], s, opac=o)
    d = np.float32([math.cos(phi), math.sin(phi), 0.0])
    res = _cast(sc, d)
    s32, o32 = float(np.float32(s)), float(np.float32(o))
    dd = d.astype(np.float64)
    cosp = dd[0] / np.linalg.norm(dd)
    sinp = math.sqrt(max(0.0, 1 - cosp * cosp))
    D2 = (r * sinp / s32) ** 2
    a = o32 * math.exp(-0.5 * D2)
    if a < 1 / 255:
        assert res.alpha[0] == 0.0 and res.range[0] == 0.0
    else:
        nrm = float(np.linalg.norm(dd))
        assert res.alpha[0] == pytest.approx(a, rel=1e-9)
        assert res.range[0] == pytest.approx(a * r * cosp / nrm, rel=1e-9)


def test_lidar_anisotropic_axis_aligned_closed_form():
    """Axis-aligned Gaussian at (r, h, k) with scales (a, b, c), ray +x: the Mahalanobis
    distance along the ray is (t-r)^2/a^2 + h^2/b^2 + k^2/c^2, minimised at t = r."""
    r, h, k, a, b, c, o = 4.0, 0.03, -0.02, 0.3, 0.05, 0.08, 0.8
    sc = scene_from([r, h, k], [a, b, c], opac=o)
    res = _cast(sc, [[1, 0, 0]])
    f = lambda v: float(np.float32(v))
    D2 = (f(h) / f(b)) ** 2 + (f(k) / f(c)) ** 2
    al = f(o) * math.exp(-0.5 * D2)
    assert res.alpha[0] == pytest.approx(al, rel=1e-10)
    assert res.range[0] == pytest.approx(al * r, rel=1e-10)


def test_lidar_peak_equals_brute_force_minimum_along_the_half_ray():
    """t^ and D2 of the R32 peak equal a brute-force minimisation of the Mahalanobis distance
    over a dense grid of t >= 0 refined by golden-section search (random Gaussians and rays,
    including centres behind the sensor, where the minimum sits at t = 0)."""
    rng = np.random.default_rng(7)
    sc = random_tiny_scene(rng, 40)
    sc.means[:5, 2] *= -1.0   # five behind the sensor along z
    proj, _, _ = oracle.lidar_project(sc, np.zeros((0, 7), np.float32), I34)
    for i in range(sc.n):
        g = proj[i]
        P = np.array([[g[3], g[4], g[5]], [g[4], g[6], g[7]], [g[5], g[7], g[8]]])
        x = g[:3]
        for _ in range(3):
            d = rng.normal(size=3)
            d[2] = abs(d[2]) * 2 + 0.2
            d /= np.linalg.norm(d)
            D2, th = oracle.lidar_peak(g, d)
            q = lambda t: float((x - t * d) @ P @ (x - t * d))
            ts = np.linspace(0.0, 2 * np.linalg.norm(x) + 1.0, 4001)
            vals = np.array([q(t) for t in ts])
            j = int(vals.argmin())
            lo, hi = ts[max(j - 1, 0)], ts[min(j + 1, ts.size - 1)]
            gr = (math.sqrt(5) - 1) / 2
            for _ in range(200):
                m1, m2 = hi - gr * (hi - lo), lo + gr * (hi - lo)
                if q(m1) < q(m2):
                    hi = m2
                else:
                    lo = m1
            tb = 0.5 * (lo + hi)
            assert D2 == pytest.approx(q(tb), rel=1e-9, abs=1e-9)
            assert th == pytest.approx(tb, abs=1e-5 * (1 + tb))


def test_lidar_behind_sensor_and_sensor_inside_gaussian():
    """Centre behind the sensor: the half-ray peak is the origin, D2 = x^T P x.  A large
    Gaussian around the sensor therefore covers every direction at t^ = 0 (alpha > 0,
    range 0); a small one behind it is invisible."""
    s, o = 0.5, 0.6
    sc = scene_from([-0.1, 0, 0], s, opac=o)
    res = _cast(sc, [[1, 0, 0], [0, 0, 1], [-1, 0, 0]], near=0.01)
    o32, s32 = float(np.float32(o)), float(np.float32(s))
    a0 = o32 * math.exp(-0.5 * (float(np.float32(0.1)) / s32) ** 2)
    assert res.alpha[0] == pytest.approx(a0, rel=1e-9) and res.range[0] == 0.0
    assert res.alpha[1] == pytest.approx(a0, rel=1e-9) and res.range[1] == 0.0
    assert res.alpha[2] == pytest.approx(o32, rel=1e-6)      # the ray through the centre
    assert res.range[2] == pytest.approx(o32 * float(np.float32(0.1)), rel=1e-6)
    res = _cast(scene_from([-3.0, 0, 0], 0.05, opac=o), [[1, 0, 0]])
    assert res.alpha[0] == 0.0 and res.n_blend[0] == 0


def test_lidar_two_layers_porter_duff_and_order():
    """Two Gaussians on the ray: range = a1 r1 + (1-a1) a2 r2, alpha = 1-(1-a1)(1-a2), the
    nearer one first whatever the creation order; at equal range keys the lower id first."""
    r1, r2, o1, o2 = 2.0, 3.5, 0.6, 0.8
    sc = scene_from([[r2, 0, 0], [r1, 0, 0]], 0.05, opac=[o2, o1])
    res = _cast(sc, [[1, 0, 0]])
    a1, a2 = float(np.float32(o1)), float(np.float32(o2))
    assert list(res.order) == [1, 0]
    assert res.range[0] == pytest.approx(a1 * r1 + (1 - a1) * a2 * r2, rel=1e-12)
    assert res.alpha[0] == pytest.approx(1 - (1 - a1) * (1 - a2), rel=1e-12)
    # equal keys: id order decides
    sc = scene_from([[r1, 0.001, 0], [r1, -0.001, 0]], 0.05, opac=[o1, o2])
    res = _cast(sc, [[1, 0, 0]])
    assert res.rhobits[0] == res.rhobits[1]
    assert list(res.order) == [0, 1]


def test_lidar_termination_stack():
    """Four o = 0.95 Gaussians on the ray: T = 0.05, 0.0025, 1.25e-4, then T(1-a) = 6.25e-6
    < 1e-4 stops BEFORE the fourth is blended (R13): n_blend = 3, alpha = 1 - 0.05^3."""
    o = 0.95
    sc = scene_from([[2, 0, 0], [2.5, 0, 0], [3, 0, 0], [3.5, 0, 0]], 0.05, opac=o)
    res = _cast(sc, [[1, 0, 0]])
    a = float(np.float32(o))
    assert res.n_blend[0] == 3
    assert res.alpha[0] == pytest.approx(1 - (1 - a) ** 3, rel=1e-12)
    exp_range = a * 2 + (1 - a) * a * 2.5 + (1 - a) ** 2 * a * 3
    assert res.range[0] == pytest.approx(exp_range, rel=1e-12)


def test_lidar_skip_threshold():
    """An entry with alpha < 1/255 is skipped (contributes nothing, T unchanged)."""
    sc = scene_from([[2, 0, 0], [3, 0, 0]], 0.05, opac=[1.0 / 300, 0.5])
    res = _cast(sc, [[1, 0, 0]])
    a = float(np.float32(0.5))
    assert res.n_blend[0] == 1
    assert res.alpha[0] == pytest.approx(a, rel=1e-12)
    assert res.range[0] == pytest.approx(3 * a, rel=1e-12)


def _rigid(R, t):
    G = np.eye(4)
    G[:3, :3], G[:3, 3] = R, t
    return G


def _quat_of(R):
    return synth._mat_to_quat(R)


def test_lidar_rigid_invariance_world_and_body():
    """Moving the whole world and the sensor by the same rigid motion leaves every ray's
    (range, alpha) unchanged; so does moving a body together with its Gaussians' template
    frame (R23: Sigma rotates with q_k)."""
    rng = np.random.default_rng(3)
    sc = random_tiny_scene(rng, 60, n_bodies=2)
    pose = random_pose(rng, 2)
    Ws = I34.copy()
    dirs = synth.lidar_pattern("random", n_points=300, seed=1)
    dirs[:, 2] = np.abs(dirs[:, 2]) + 0.5
    dirs = (dirs / np.linalg.norm(dirs, axis=1, keepdims=True)).astype(np.float32)
    ref = _cast(sc, dirs, Ws, pose)
    # world motion G: static means move, body poses are pre-multiplied, the sensor W -> W G^-1
    ax = rng.normal(size=3)
    R = synth._quat_to_mat(synth._axis_angle_quat(ax, 0.7))
    t = rng.normal(size=3)
    sc2 = scene_from(sc.means, sc.scales, sc.quats, sc.opacities, None, sc.body_id, sc.n_bodies)
    st = sc.body_id < 0
    sc2.means[st] = (sc.means[st].astype(np.float64) @ R.T + t).astype(np.float32)
    qR = _quat_of(R)
    sc2.quats[st] = np.array([synth._quat_mul(qR, q) for q in sc.quats[st].astype(np.float64)], np.float32)
    pose2 = pose.copy().astype(np.float64)
    for k in range(2):
        pose2[k, :3] = R @ pose[k, :3] + t
        pose2[k, 3:] = synth._quat_mul(qR, pose[k, 3:].astype(np.float64))
    W2 = np.linalg.inv(_rigid(R, t))[:3]
    # float32 inputs round the moved scene: compare with a tolerance well above that rounding
    got = _cast(sc2, dirs, W2.astype(np.float32), pose2.astype(np.float32))
    ok = ~(ref.masked | got.masked)
    assert ok.mean() > 0.9
    np.testing.assert_allclose(got.alpha[ok], ref.alpha[ok], atol=2e-4)
    np.testing.assert_allclose(got.range[ok], ref.range[ok], atol=2e-4 * (1 + ref.range[ok].max()))
    assert (ref.alpha > 0.05).sum() > 20


def test_range_key_chain_exact_and_close_to_fp64():
    """R32 step 2: the C binary32 chain equals an exactly rounded re-computation (the mini
    oracle's fma32 emulation + numpy binary32 sqrt, correctly rounded), and is within a few
    ulps of the fp64 range."""
    rng = np.random.default_rng(11)
    for trial in range(300):
        W = np.hstack([synth._quat_to_mat(synth._axis_angle_quat(rng.normal(size=3), rng.uniform(0, 3))),
                       rng.normal(size=(3, 1))]).astype(np.float32)
        mu = rng.normal(size=3).astype(np.float32) * 2
        pose = None
        if trial % 2:
            q = rng.normal(size=4)
            pose = np.concatenate([rng.normal(size=3), q / np.linalg.norm(q)]).astype(np.float32)
        got = oracle.range_key(W, pose, mu)
        # exact re-computation of the same chain
        if pose is None:
            M, m = W[:, :3].astype(np.float32), W[:, 3].astype(np.float32)
        else:
            Rk = mini_rot32(pose[3:])
            M = np.zeros((3, 3), np.float32)
            m = np.zeros(3, np.float32)
            for r in range(3):
                for c in range(3):
                    p = np.float32(W[r, 2] * Rk[2][c])
                    M[r, c] = mini.fma32(W[r, 0], Rk[0][c], mini.fma32(W[r, 1], Rk[1][c], p))
                m[r] = mini.fma32(W[r, 0], pose[0], mini.fma32(W[r, 1], pose[1], mini.fma32(W[r, 2], pose[2], W[r, 3])))
        x = [mini.fma32(M[r, 0], mu[0], mini.fma32(M[r, 1], mu[1], mini.fma32(M[r, 2], mu[2], m[r]))) for r in range(3)]
        zz = np.float32(x[2] * x[2])
        s = mini.fma32(x[0], x[0], mini.fma32(x[1], x[1], zz))
        want = np.sqrt(np.float32(s))
        assert np.float32(got).view(np.uint32) == np.float32(want).view(np.uint32)
        # fp64 reference
        if pose is None:
            xw = mu.astype(np.float64)
        else:
            xw = synth._quat_to_mat(pose[3:].astype(np.float64)) @ mu + pose[:3]
        x64 = W[:, :3].astype(np.float64) @ xw + W[:, 3]
        assert float(got) == pytest.approx(float(np.linalg.norm(x64)), rel=1e-5, abs=1e-5)


def mini_rot32(q):
    """R11 quaternion chain in numpy binary32 (each op rounded)."""
    f = np.float32
    qw, qx, qy, qz = (f(v) for v in q)
    xx, yy, zz = f(qx * qx), f(qy * qy), f(qz * qz)
    xy, xz, yz = f(qx * qy), f(qx * qz), f(qy * qz)
    wx, wy, wz = f(qw * qx), f(qw * qy), f(qw * qz)
    two, one = f(2), f(1)
    return [[f(one - f(two * f(yy + zz))), f(two * f(xy - wz)), f(two * f(xz + wy))],
            [f(two * f(xy + wz)), f(one - f(two * f(xx + zz))), f(two * f(yz - wx))],
            [f(two * f(xz - wy)), f(two * f(yz + wx)), f(one - f(two * f(xx + yy)))]]


def test_lidar_floor_plane_of_surfels_gives_geometric_range():
    """A dense, opaque floor of flat surfels at z = -h: a downward ray at angle beta below the
    horizon hits it at h / sin(beta); the normalised range (range / alpha) matches the ray-plane
    intersection to within the surfels' thickness."""
    rng = np.random.default_rng(5)
    h = 1.0
    g = np.linspace(-3, 3, 121)
    X, Y = np.meshgrid(g, g)
    n = X.size
    means = np.stack([X.ravel(), Y.ravel(), np.full(n, -h)], 1)
    sc = scene_from(means, [0.05, 0.05, 0.002], None, opac=0.98)
    betas = np.radians([20.0, 35.0, 60.0, 90.0])
    az = rng.uniform(-np.pi, np.pi, betas.size)
    dirs = np.stack([np.cos(betas) * np.cos(az), np.cos(betas) * np.sin(az), -np.sin(betas)], 1)
    res = _cast(sc, dirs.astype(np.float32))
    assert (res.alpha > 0.999).all()
    np.testing.assert_allclose(res.range / res.alpha, h / np.sin(betas), rtol=0.01)
