"""Pins of the CPU oracle against things other than itself (pins 1-15).

Each test names the pin it implements and the passage/reading it checks.  None of
these retypes the oracle's formulas: they use closed forms, invariants, special cases,
textbook/library routines, brute force, and an independent second oracle.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from oracle import binning, mini
from tests.helpers import identity_cam, random_pose, random_tiny_scene, scene_from

PRM = oracle.RenderParams(64, 48)


def _frame(scene, K, W, prm=PRM, pose=None, **kw):
    pose = np.zeros((max(scene.n_bodies, 0), 7), np.float32) if pose is None else pose
    return oracle.render_frame(scene, pose, K, W, prm, **kw)


# ---------------------------------------------------------------- pin 1 (closed form)
def test_pin1_isotropic_on_axis_closed_form():
    """Isotropic Gaussian at camera (0,0,z): u=c_x, v=c_y, Sigma2D = diag(s^2 f^2/z^2 + 0.3);
    at the pixel centre that coincides with (u,v) alpha = min(0.99, o), RGB = a c + (1-a) bg,
    depth = a z  (3DGS EWA [P:212]; R3, R7, R12-R16)."""
    z, s, o, c = 3.0, 0.05, 0.8, (0.9, 0.2, 0.4)
    sc = scene_from([0, 0, z], s, opac=o, colours=c)
    K, W = identity_cam(fx=100.0, fy=120.0, cx=32.5, cy=24.5)
    prm = oracle.RenderParams(64, 48, bg=(0.1, 0.3, 0.5))
    r = _frame(sc, K, W, prm)
    p = r.proj[0]
    assert p[oracle.F_U] == pytest.approx(32.5, abs=1e-12)
    assert p[oracle.F_V] == pytest.approx(24.5, abs=1e-12)
    s = float(np.float32(s))  # the template stores float32 scales
    assert p[oracle.F_SXX] == pytest.approx(s * s * 100.0 ** 2 / z ** 2 + 0.3, rel=1e-12)
    assert p[oracle.F_SYY] == pytest.approx(s * s * 120.0 ** 2 / z ** 2 + 0.3, rel=1e-12)
    assert abs(p[oracle.F_SXY]) < 1e-12
    o32 = float(np.float32(o))
    col = np.array(c)
    bg = np.array(prm.bg, np.float32).astype(np.float64)
    np.testing.assert_allclose(r.rgb[24, 32], o32 * col + (1 - o32) * bg, atol=1e-6)
    assert r.depth[24, 32] == pytest.approx(o32 * z, rel=1e-12)
    assert r.alpha[24, 32] == pytest.approx(o32, rel=1e-12)
    # one pixel to the right: alpha = o * exp(-0.5 * 1 / Sxx) exactly (conic a = 1/Sxx)
    a1 = o32 * math.exp(-0.5 / p[oracle.F_SXX])
    assert r.alpha[24, 33] == pytest.approx(a1, rel=1e-12)


# ---------------------------------------------------------------- pin 2 (closed form)
@pytest.mark.parametrize("x0", [0.5, -0.9, 1.5])
def test_pin2_off_axis_jacobian_and_clamp(x0):
    """At (x0,0,z): Sxx = s^2 (f^2/z^2 + f^2 tx^2/z^4) + 0.3 with tx = z*clamp(x0/z, +-1.3 W/(2f)),
    Syy = s^2 f^2/z^2 + 0.3, Sxy = 0 (3DGS EWA Jacobian; reading R6)."""
    z, s, f = 3.0, 0.04, 100.0
    sc = scene_from([x0, 0, z], s)
    K, W = identity_cam(fx=f, fy=f)
    p = _frame(sc, K, W).proj[0]
    lim = 1.3 * 64 / (2 * f)
    x0 = float(np.float32(x0))  # the template stores float32 means and scales
    tx = z * min(max(x0 / z, -lim), lim)
    s32 = float(np.float32(s))
    exp_xx = s32 * s32 * (f * f / z ** 2 + f * f * tx * tx / z ** 4) + 0.3
    assert p[oracle.F_SXX] == pytest.approx(exp_xx, rel=1e-12)
    assert p[oracle.F_SYY] == pytest.approx(s32 * s32 * f * f / z ** 2 + 0.3, rel=1e-12)
    assert abs(p[oracle.F_SXY]) < 1e-12
    assert p[oracle.F_U] == pytest.approx(f * float(np.float32(x0)) / z + 32.5, rel=1e-12)


# ---------------------------------------------------------------- pin 3 (closed form, RLGK)
def test_pin3_anisotropy_body_rotation_swaps_axes():
    """Axis-aligned (sa, sb, sc) Gaussian on body 0 at body-local origin; body at (0,0,3).
    Rotating the BODY by 90 deg about the optical axis (via the pose) swaps the
    Sigma2D diagonals."""
    sa, sb = 0.08, 0.02
    sc = scene_from([0, 0, 0], [sa, sb, 0.01], body=[0], n_bodies=1)
    K, W = identity_cam()
    pose0 = np.float32([[0, 0, 3, 1, 0, 0, 0]])
    h = math.sqrt(0.5)
    pose1 = np.float32([[0, 0, 3, h, 0, 0, h]])
    p0 = _frame(sc, K, W, pose=pose0).proj[0]
    p1 = _frame(sc, K, W, pose=pose1).proj[0]
    sa32, sb32 = float(np.float32(sa)), float(np.float32(sb))
    assert p0[oracle.F_SXX] == pytest.approx(sa32 ** 2 * 100 ** 2 / 9 + 0.3, rel=1e-12)
    assert p0[oracle.F_SYY] == pytest.approx(sb32 ** 2 * 100 ** 2 / 9 + 0.3, rel=1e-12)
    # fp32 pose quaternion is unit only to ~1e-8
    assert p1[oracle.F_SXX] == pytest.approx(p0[oracle.F_SYY], rel=1e-6)
    assert p1[oracle.F_SYY] == pytest.approx(p0[oracle.F_SXX], rel=1e-6)
    assert p1[oracle.F_U] == pytest.approx(32.5, abs=1e-9)


# ---------------------------------------------------------------- pin 4 (closed form + brute force)
def test_pin4_extents_closed_form_and_brute_force():
    """r_x = sigma_x sqrt(2 ln(255 o)) on axis (reading R8), and on random Gaussians every
    pixel whose alpha >= 1/255 (evaluated directly from the definition alpha = o e^power)
    lies inside [u +- r_x] x [v +- r_y]."""
    sc = scene_from([0, 0, 3.0], 0.05, opac=0.7)
    K, W = identity_cam()
    p = _frame(sc, K, W).proj[0]
    sig_px = math.sqrt(p[oracle.F_SXX])
    o32 = float(np.float32(0.7))
    assert math.sqrt(p[oracle.F_KAPPA] * p[oracle.F_SXX]) == pytest.approx(
        sig_px * math.sqrt(2 * math.log(255 * o32)), rel=1e-12)
    rng = np.random.default_rng(4)
    sc = random_tiny_scene(rng, 40)
    prm = oracle.RenderParams(96, 80)
    K, W = identity_cam(cx=48, cy=40)
    proj, zb, valid = oracle.project(sc, np.zeros((0, 7), np.float32), K, W, prm)
    py, px = np.meshgrid(np.arange(80) + 0.5, np.arange(96) + 0.5, indexing="ij")
    for i in np.nonzero(valid)[0]:
        g = proj[i]
        dx, dy = g[oracle.F_U] - px, g[oracle.F_V] - py
        power = -0.5 * (g[oracle.F_A] * dx * dx + g[oracle.F_C] * dy * dy) - g[oracle.F_B] * dx * dy
        alpha = g[oracle.F_O] * np.exp(power)
        rx = math.sqrt(g[oracle.F_KAPPA] * g[oracle.F_SXX])
        ry = math.sqrt(g[oracle.F_KAPPA] * g[oracle.F_SYY])
        inside = (np.abs(dx) <= rx * (1 + 1e-12)) & (np.abs(dy) <= ry * (1 + 1e-12))
        assert not np.any((alpha >= 1 / 255) & ~inside)


# ---------------------------------------------------------------- pin 5 (textbook / library)
def _gauss_sphere(nt=64, nphi=128):
    x, w = np.polynomial.legendre.leggauss(nt)
    phi = (np.arange(nphi) + 0.5) * 2 * np.pi / nphi
    ct, ph = np.meshgrid(x, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    wts = np.outer(w, np.full(nphi, 2 * np.pi / nphi))
    return np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3), wts.reshape(-1)


def test_pin5_sh_orthonormal_gram_matrix():
    """Reading R18: the 16 basis functions are orthonormal on S^2 (Gram = I within 1e-9)
    under Gauss-Legendre x uniform-phi quadrature — pins every constant's magnitude."""
    pts, wts = _gauss_sphere()
    Y = np.array([oracle.sh_basis(3, *p) for p in pts])
    G = (Y * wts[:, None]).T @ Y
    assert np.abs(G - np.eye(16)).max() < 1e-9


def test_pin5_sh_matches_scipy_real_harmonics_up_to_documented_signs():
    """Each basis function equals sign_j * (real spherical harmonic from scipy), with the
    documented 3DGS sign convention (R18)."""
    sp = pytest.importorskip("scipy.special")
    rng = np.random.default_rng(5)
    d = rng.normal(size=(50, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    theta = np.arccos(d[:, 2])          # polar
    phi = np.arctan2(d[:, 1], d[:, 0])  # azimuth

    def real_sh(l, m):
        if hasattr(sp, "sph_harm_y"):
            Y = sp.sph_harm_y(l, abs(m), theta, phi)
        else:  # older scipy signature: sph_harm(m, l, azimuth, polar)
            Y = sp.sph_harm(abs(m), l, phi, theta)
        if m > 0:
            return math.sqrt(2) * (-1) ** m * Y.real
        if m < 0:
            return math.sqrt(2) * (-1) ** m * Y.imag
        return Y.real

    ours = np.array([oracle.sh_basis(3, *p) for p in d])
    signs = []
    for l in range(4):
        for m in range(-l, l + 1):
            ref = real_sh(l, m)
            ratio = ours[:, l * l + l + m] / ref
            assert np.allclose(np.abs(ratio), 1.0, atol=1e-9), (l, m)
            assert np.ptp(np.sign(ratio)) == 0
            signs.append(int(np.sign(ratio[0])))
    # documented sign convention (R18)
    assert signs == SH_SIGNS, signs


# 3DGS basis j = l^2+l+m equals (-1)^j times scipy's real SH (sqrt2 (-1)^m Re/Im Y_l^|m|)
SH_SIGNS = [(-1) ** j for j in range(16)]


# ---------------------------------------------------------------- pin 6 (closed form)
def test_pin6_two_layer_porter_duff_and_id_tiebreak():
    """Two on-axis Gaussians: C = a1 c1 + (1-a1) a2 c2 + (1-a1)(1-a2) bg (front-to-back
    'over', north_star); equal depth => lower id first (reading R10)."""
    c1, c2 = np.array([1.0, 0.0, 0.2]), np.array([0.0, 1.0, 0.6])
    K, W = identity_cam()
    prm = oracle.RenderParams(64, 48, bg=(0.25, 0.5, 0.75))
    bg = np.array(prm.bg)
    sc = scene_from([[0, 0, 2.0], [0, 0, 3.0]], 0.05, opac=[0.6, 0.7], colours=np.stack([c1, c2]))
    r = _frame(sc, K, W, prm)
    a1, a2 = float(np.float32(0.6)), float(np.float32(0.7))
    exp = a1 * c1 + (1 - a1) * a2 * c2 + (1 - a1) * (1 - a2) * bg
    np.testing.assert_allclose(r.rgb[24, 32], exp, atol=1e-6)
    assert r.depth[24, 32] == pytest.approx(a1 * 2 + (1 - a1) * a2 * 3, rel=1e-12)
    # far Gaussian listed first in the array must still composite behind
    sc_rev = scene_from([[0, 0, 3.0], [0, 0, 2.0]], 0.05, opac=[0.7, 0.6], colours=np.stack([c2, c1]))
    np.testing.assert_allclose(_frame(sc_rev, K, W, prm).rgb[24, 32], exp, atol=1e-6)
    # equal depth: id order decides; swapping ids swaps the result
    sc_eq = scene_from([[0, 0, 2.5], [0, 0, 2.5]], 0.05, opac=[0.6, 0.7], colours=np.stack([c1, c2]))
    sc_sw = scene_from([[0, 0, 2.5], [0, 0, 2.5]], 0.05, opac=[0.7, 0.6], colours=np.stack([c2, c1]))
    e1 = a1 * c1 + (1 - a1) * a2 * c2 + (1 - a1) * (1 - a2) * bg
    e2 = a2 * c2 + (1 - a2) * a1 * c1 + (1 - a1) * (1 - a2) * bg
    np.testing.assert_allclose(_frame(sc_eq, K, W, prm).rgb[24, 32], e1, atol=1e-6)
    np.testing.assert_allclose(_frame(sc_sw, K, W, prm).rgb[24, 32], e2, atol=1e-6)


# ---------------------------------------------------------------- pin 7 (closed form)
def test_pin7_termination_stack():
    """Identical on-axis Gaussians with alpha = 0.95 at the centre pixel: T = 0.05, 0.0025,
    1.25e-4, then tT = 6.25e-6 < 1e-4 => stop BEFORE blending the 4th (reading R13):
    3 blended, termination at the 4th entry, final T = 0.05^3."""
    n = 6
    K, W = identity_cam()
    sc = scene_from([[0, 0, 2.0 + 0.1 * i] for i in range(n)], 0.05, opac=0.95, colours=(1, 1, 1))
    r = _frame(sc, K, W)
    a = float(np.float32(0.95))
    assert r.term_id[24, 32] == 3
    assert r.n_eval_all[24, 32] == 4
    assert 1 - r.alpha[24, 32] == pytest.approx((1 - a) ** 3, rel=1e-9)
    # colour 1.0 is stored as a float32 SH DC coefficient: rgb = 1 +- 1e-7
    assert r.rgb[24, 32, 0] == pytest.approx(1 - (1 - a) ** 3, rel=1e-7)


# ---------------------------------------------------------------- pin 8 (special cases)
def test_pin8_clamp_and_cull():
    """o = 1 => alpha = 0.99 at the peak (north_star clamp); o = 0.003 < 1/255 => culled,
    the pixel shows the background (reading R5)."""
    K, W = identity_cam()
    prm = oracle.RenderParams(64, 48, bg=(0.2, 0.2, 0.2))
    r = _frame(scene_from([0, 0, 2.0], 0.05, opac=1.0, colours=(1, 0, 0)), K, W, prm)
    assert r.alpha[24, 32] == pytest.approx(0.99, abs=1e-15)
    np.testing.assert_allclose(r.rgb[24, 32], [0.99 + 0.01 * 0.2, 0.01 * 0.2, 0.01 * 0.2], atol=1e-7)
    r = _frame(scene_from([0, 0, 2.0], 0.05, opac=0.003, colours=(1, 0, 0)), K, W, prm)
    assert not r.valid[0]
    np.testing.assert_allclose(r.rgb, np.float32(0.2), atol=1e-7)
    assert np.all(r.alpha == 0) and np.all(r.depth == 0)


# ---------------------------------------------------------------- pin 9 (invariants)
def test_pin9_partition_of_unity_and_constant_fields():
    """sum w + T = 1; constant colour c with bg = c => RGB = c; constant z => depth = z*alpha."""
    rng = np.random.default_rng(9)
    sc = random_tiny_scene(rng, 60)
    K, W = identity_cam()
    white = scene_from(sc.means, sc.scales, sc.quats, sc.opacities, colours=(1, 1, 1))
    r = _frame(white, K, W)
    np.testing.assert_allclose(r.rgb[..., 0], r.alpha, atol=1e-12)
    assert np.all((r.alpha >= 0) & (r.alpha <= 1))
    const = scene_from(sc.means, sc.scales, sc.quats, sc.opacities, colours=(0.3, 0.6, 0.1))
    prm = oracle.RenderParams(64, 48, bg=(0.3, 0.6, 0.1))
    r = _frame(const, K, W, prm)
    np.testing.assert_allclose(r.rgb, np.broadcast_to(np.float32([0.3, 0.6, 0.1]), r.rgb.shape), atol=1e-6)
    flat = sc.means.copy()
    flat[:, 2] = 2.5
    r = _frame(scene_from(flat, sc.scales, sc.quats, sc.opacities), K, W)
    np.testing.assert_allclose(r.depth, 2.5 * r.alpha, rtol=1e-12, atol=1e-15)


def test_pin9_transmittance_monotone_and_blended_alpha_range():
    """T is non-increasing over the front-to-back sweep and every blended alpha is in
    [1/255, 0.99] — checked on the mini oracle by replaying the per-entry sweep."""
    rng = np.random.default_rng(19)
    sc = random_tiny_scene(rng, 50)
    K, W = identity_cam()
    pr = mini.project(sc, np.zeros((0, 7)), K, W, 64, 48)
    ids = np.nonzero(pr["valid"])[0]
    order = ids[np.lexsort((ids, pr["z32"].view(np.uint32)[ids]))]
    for (px, py) in [(32, 24), (10, 10), (50, 40)]:
        T, Ts = 1.0, [1.0]
        for i in order:
            dx, dy = pr["u"][i] - px - 0.5, pr["v"][i] - py - 0.5
            a, b, c = pr["conic"][i]
            pw = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
            al = min(0.99, pr["o"][i] * math.exp(pw))
            if pw > 0 or al < 1 / 255:
                continue
            assert 1 / 255 <= al <= 0.99
            if T * (1 - al) < 1e-4:
                break
            T *= 1 - al
            Ts.append(T)
        assert all(x >= y for x, y in zip(Ts, Ts[1:]))


# ---------------------------------------------------------------- pin 10 (brute force)
def test_pin10_pure_equals_box_accelerated():
    """Pure all-pairs oracle == box-accelerated oracle, bit-exact (reading R8), on C1 and on
    100 random tiny scenes (<= 64 Gaussians, 32x32)."""
    cfg = synth.CONFIGS["C1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    a = oracle.render_frame(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm, mode="pure")
    c = oracle.render_frame(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm, mode="box")
    assert np.array_equal(a.rgb, c.rgb) and np.array_equal(a.depth, c.depth)
    assert np.array_equal(a.term_id, c.term_id)
    rng = np.random.default_rng(10)
    prm = oracle.RenderParams(32, 32)
    K, W = identity_cam(fx=40, fy=40, cx=16, cy=16)
    for _ in range(100):
        sc = random_tiny_scene(rng, int(rng.integers(1, 65)), n_bodies=2, sh_degree=int(rng.integers(0, 4)))
        pose = random_pose(rng, 2)
        a = oracle.render_frame(sc, pose, K, W, prm, mode="pure", nthreads=1)
        c = oracle.render_frame(sc, pose, K, W, prm, mode="box", nthreads=1)
        assert np.array_equal(a.rgb, c.rgb) and np.array_equal(a.alpha, c.alpha)
        assert np.array_equal(a.depth, c.depth) and np.array_equal(a.term_id, c.term_id)


# ---------------------------------------------------------------- pin 11 (second oracle)
def test_pin11_numpy_mini_oracle_matches_c_oracle_on_c1():
    cfg = synth.CONFIGS["C1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    c = oracle.render_frame(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm)
    m = mini.render(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], cfg.width, cfg.height)
    assert np.abs(c.rgb - m["rgb"]).max() <= 1e-12
    assert np.abs(c.depth - m["depth"]).max() <= 1e-12
    assert np.array_equal(c.term_id, m["term_id"])
    assert np.array_equal(c.zbits, m["proj"]["z32"].view(np.uint32))


def test_pin11_mini_oracle_matches_with_bodies_and_sh3():
    """With body poses and SH-3: agreement up to the O(|q|^2-1) ~ 1e-7 difference between the
    Hamilton sandwich (mini) and the matrix formula (C) for fp32 pose quaternions."""
    cfg = synth.CONFIGS["T1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    for e in range(2):
        c = oracle.render_frame(sc, b.poses[e], b.intrinsics[e, 0], b.w2c[e, 0], prm)
        m = mini.render(sc, b.poses[e], b.intrinsics[e, 0], b.w2c[e, 0], cfg.width, cfg.height)
        assert np.array_equal(c.zbits, m["proj"]["z32"].view(np.uint32))
        np.testing.assert_allclose(c.proj[:, oracle.F_U], m["proj"]["u"], rtol=0, atol=1e-4)
        np.testing.assert_allclose(c.proj[:, oracle.F_R:oracle.F_BL + 1], m["proj"]["rgb"], atol=1e-6)
        ok = ~c.masked
        assert np.abs(c.rgb - m["rgb"])[ok].max() < 1e-3


# ---------------------------------------------------------------- pin 12 (invariant)
def test_pin12_rigid_invariance_pins_body_frame_sh():
    """Moving a body AND the camera by the same rigid transform leaves the image of that
    body's Gaussians unchanged at D=3 (readings R19, R23).  A world-frame SH reading fails
    this test, because the view direction would rotate with the transform."""
    rng = np.random.default_rng(12)
    sc = random_tiny_scene(rng, 40, n_bodies=1, sh_degree=3)
    sc.body_id[:] = 0
    K, W = identity_cam()
    pose = np.float32([[0.05, -0.02, 0.1, 1, 0, 0, 0]])
    r0 = _frame(sc, K, W, pose=pose)
    # rigid G: rotation 30 deg about (1,1,0)/sqrt2 + translation
    ax = np.array([1.0, 1.0, 0.0]) / math.sqrt(2)
    ang = math.radians(30)
    qg = np.concatenate([[math.cos(ang / 2)], math.sin(ang / 2) * ax])
    Rg = synth._quat_to_mat(qg)
    tg = np.array([0.3, -0.2, 0.5])
    q1 = synth._quat_mul(qg, pose[0, 3:].astype(np.float64))
    t1 = Rg @ pose[0, :3].astype(np.float64) + tg
    pose1 = np.float32([np.concatenate([t1, q1])])
    Wr = W[:, :3].astype(np.float64)
    W1 = np.zeros((3, 4))
    W1[:, :3] = Wr @ Rg.T
    W1[:, 3] = W[:, 3] - Wr @ Rg.T @ tg
    r1 = _frame(sc, K, W1.astype(np.float32), pose=pose1)
    ok = ~(r0.masked | r1.masked)
    assert np.abs(r0.rgb - r1.rgb)[ok].max() < 1e-5
    assert ok.mean() > 0.99


def test_spec_rlgk_identity_and_translation():
    """identity pose => world = local; translation-only pose => shifted."""
    rng = np.random.default_rng(13)
    sc = random_tiny_scene(rng, 30, n_bodies=1, sh_degree=2)
    sc.body_id[:] = 0
    K, W = identity_cam()
    static = scene_from(sc.means, sc.scales, sc.quats, sc.opacities, sh_degree=2)
    static.sh[:] = sc.sh
    ident = _frame(sc, K, W, pose=np.float32([[0, 0, 0, 1, 0, 0, 0]]))
    ref = _frame(static, K, W)
    assert np.array_equal(ident.rgb, ref.rgb)
    t = np.float32([0.1, -0.05, 0.25])
    moved = _frame(sc, K, W, pose=np.float32([np.concatenate([t, [1, 0, 0, 0]])]))
    static.means[:] = sc.means + t
    ref2 = _frame(static, K, W)
    # static means + t are rounded to float32 (~1e-7 m): compare at that resolution
    np.testing.assert_allclose(moved.proj[:, oracle.F_U], ref2.proj[:, oracle.F_U], rtol=0, atol=1e-5)
    np.testing.assert_allclose(moved.proj[:, oracle.F_Z64], ref2.proj[:, oracle.F_Z64], rtol=0, atol=1e-6)


def test_spec_quaternion_examples():
    """90 deg + 90 deg about z = 180 deg; R(q) of 90 deg about z maps x -> y."""
    h = math.sqrt(0.5)
    q90 = np.array([h, 0, 0, h])
    q180 = synth._quat_mul(q90, q90)
    np.testing.assert_allclose(q180, [0, 0, 0, 1], atol=1e-15)
    sc = scene_from([1.0, 0, 0], 0.05, body=[0], n_bodies=1)
    K, W = identity_cam()
    pose = np.float32([[0, 0, 3, h, 0, 0, h]])
    p = _frame(sc, K, W, pose=pose).proj[0]
    assert p[oracle.F_XC] == pytest.approx(0.0, abs=1e-7)
    assert p[oracle.F_YC] == pytest.approx(1.0, abs=1e-7)


# ---------------------------------------------------------------- pin 15: R11 chain
def test_fma32_emulation_matches_libm_fmaf_including_midpoints():
    L = oracle.lib()
    rng = np.random.default_rng(15)
    a = rng.normal(size=2000).astype(np.float32)
    b = rng.normal(size=2000).astype(np.float32)
    c = (rng.normal(size=2000) * 10.0 ** rng.integers(-8, 3, 2000)).astype(np.float32)
    ours = mini.fma32(a, b, c)
    ref = np.array([L.gsbo_fmaf(float(x), float(y), float(z)) for x, y, z in zip(a, b, c)], np.float32)
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))
    # exact midpoint: (1+2^-12)^2 = 1 + 2^-11 + 2^-24 is halfway between two binary32 values;
    # a tiny c decides the direction (naive fp64-then-fp32 double rounding gets this wrong)
    x = np.float32(1 + 2 ** -12)
    for cc in [2.0 ** -60, -(2.0 ** -60), 0.0]:
        r = mini.fma32(x, x, np.float32(cc))
        assert r.view(np.uint32) == np.float32(L.gsbo_fmaf(float(x), float(x), float(np.float32(cc)))).view(np.uint32)
    up = mini.fma32(x, x, np.float32(2.0 ** -60))
    assert up > np.float32(1 + 2 ** -11)


def test_r11_depth_chain_c_equals_numpy_and_is_within_ulps_of_fp64():
    rng = np.random.default_rng(16)
    for trial in range(200):
        W = np.zeros((3, 4), np.float32)
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        W[:, :3] = synth._quat_to_mat(q)
        W[:, 3] = rng.normal(0, 2, 3)
        pose = random_pose(rng, 1)[0] if trial % 2 else None
        mu = rng.normal(0, 1, 3).astype(np.float32)
        zc = oracle.depth_key(W, pose, mu)
        zn = mini.depth_key_f32(W, pose, mu[None, :])[0]
        assert zc.view(np.uint32) == zn.view(np.uint32)
        # vs fp64 camera z of the same fp32 inputs
        if pose is None:
            z64 = W[2, :3].astype(np.float64) @ mu + W[2, 3]
        else:
            R = synth._quat_to_mat(pose[3:].astype(np.float64) / np.linalg.norm(pose[3:].astype(np.float64)))
            z64 = W[2, :3].astype(np.float64) @ (R @ mu + pose[:3]) + W[2, 3]
        assert abs(float(zc) - z64) <= 64 * np.finfo(np.float32).eps * (1 + np.abs(W).sum() * (1 + np.abs(mu).sum()))


# ---------------------------------------------------------------- pin 14: binning identities
def test_pin14_binning_identities_and_rect_examples():
    # hand-computed R9 example: u=20.3, Sxx=4, kappa=4 -> rx=4: xl=15.8, xh=23.8 -> px [16,23]
    tx0, tx1, ty0, ty1, ok = binning.rects_f32([20.3], [5.0], [4.0], [1.0], [4.0], [True], 64, 48)
    assert ok[0] and tx0[0] == 1 and tx1[0] == 1 and ty0[0] == 0 and ty1[0] == 0
    tx0, tx1, *_ = binning.rects_f32([15.0], [5.0], [4.0], [1.0], [4.0], [True], 64, 48)
    assert tx0[0] == 0 and tx1[0] == 1         # pixels 11..18 straddle tiles 0 and 1
    # pixel centre exactly on the box edge is inside: u=10, rx=2 -> xl=7.5 ... px 8..11
    _, _, _, _, ok = binning.rects_f32([-5.0], [5.0], [1.0], [1.0], [1.0], [True], 64, 48)
    assert not ok[0]                           # entirely left of the image
    _, _, _, _, ok = binning.rects_f32([np.inf], [5.0], [1.0], [1.0], [1.0], [True], 64, 48)
    assert not ok[0]
    # identities on C1 projected values
    cfg = synth.CONFIGS["C1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    proj, zb, valid = oracle.project(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm)
    f32 = lambda k: proj[:, k].astype(np.float32)
    kap = np.float32(2 * np.log(255 * sc.opacities.astype(np.float64)))
    offs, ids = binning.bin_frame(f32(oracle.F_U), f32(oracle.F_V), f32(oracle.F_SXX), f32(oracle.F_SYY),
                                  kap, zb, valid, cfg.width, cfg.height)
    t = binning.rects_f32(f32(oracle.F_U), f32(oracle.F_V), f32(oracle.F_SXX), f32(oracle.F_SYY),
                          kap, valid, cfg.width, cfg.height)
    tiles_per = np.where(t[4], (t[1] - t[0] + 1) * (t[3] - t[2] + 1), 0)
    assert offs[-1] == ids.size == tiles_per.sum()
    for k in range(offs.size - 1):
        seg = ids[offs[k]:offs[k + 1]]
        assert np.unique(seg).size == seg.size
        key = zb[seg].astype(np.uint64) << np.uint64(32) | seg.astype(np.uint64)
        assert np.all(np.diff(key.astype(np.float64)) > 0) or seg.size < 2


def test_tile_lists_cover_every_contributing_gaussian():
    """Reading R8 end to end: every Gaussian that contributes alpha >= 1/255 at a pixel
    (oracle, fp64) is in that pixel's tile list, except at threshold-margin entries."""
    cfg = synth.CONFIGS["T3"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    proj, zb, valid = oracle.project(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm)
    f32 = lambda k: proj[:, k].astype(np.float32)
    kap = proj[:, oracle.F_KAPPA].astype(np.float32)
    offs, ids = binning.bin_frame(f32(oracle.F_U), f32(oracle.F_V), f32(oracle.F_SXX), f32(oracle.F_SYY),
                                  kap, zb, valid, cfg.width, cfg.height)
    tw = (cfg.width + 15) // 16
    rng = np.random.default_rng(0)
    for _ in range(200):
        px, py = int(rng.integers(cfg.width)), int(rng.integers(cfg.height))
        t = (py // 16) * tw + px // 16
        lst = set(ids[offs[t]:offs[t + 1]].tolist())
        for i in np.nonzero(valid)[0]:
            g = proj[i]
            dx, dy = g[oracle.F_U] - px - 0.5, g[oracle.F_V] - py - 0.5
            pw = -0.5 * (g[oracle.F_A] * dx * dx + g[oracle.F_C] * dy * dy) - g[oracle.F_B] * dx * dy
            araw = g[oracle.F_O] * math.exp(pw)
            if araw >= (1 / 255) * (1 + 1e-6):
                assert i in lst


# ---------------------------------------------------------------- R29: body-attached cameras
def test_r29_compose_c_equals_numpy_and_closed_form():
    """The camera-mount composition chain (reading R29) is bit-identical in the C and NumPy
    oracles; with an identity mount the camera sits at the body origin looking along the body
    axes: W = R(q)^T and W t + w = 0."""
    rng = np.random.default_rng(29)
    for _ in range(200):
        pose = random_pose(rng, 1)[0]
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        B = np.zeros((3, 4), np.float32)
        B[:, :3] = synth._quat_to_mat(q)
        B[:, 3] = rng.normal(0, 0.3, 3)
        wc = oracle.compose_w2c(pose, B)
        wn = mini.compose_w2c_f32(pose, B)
        assert np.array_equal(wc.view(np.uint32), wn.view(np.uint32))
    pose = np.float32([0.4, -0.2, 1.1, *(np.array([0.9, 0.1, -0.3, 0.2]) / np.linalg.norm([0.9, 0.1, -0.3, 0.2]))])
    Bi = np.zeros((3, 4), np.float32)
    Bi[:, :3] = np.eye(3)
    W = oracle.compose_w2c(pose, Bi).astype(np.float64)
    R = synth._quat_to_mat(pose[3:].astype(np.float64))
    np.testing.assert_allclose(W[:, :3], R.T, atol=1e-6)
    np.testing.assert_allclose(W[:, :3] @ pose[:3].astype(np.float64) + W[:, 3], 0, atol=1e-6)


def test_r29_egocentric_view_of_own_body_is_pose_invariant():
    """A camera mounted on body 0 sees body 0's Gaussians identically wherever the body is
    (composition order B o pose^-1; SH in the body frame, R19)."""
    rng = np.random.default_rng(30)
    sc = random_tiny_scene(rng, 40, n_bodies=1, sh_degree=3)
    sc.body_id[:] = 0
    K, _ = identity_cam()
    B = np.zeros((3, 4), np.float32)
    B[:, :3] = np.eye(3)
    B[:, 3] = [0.0, 0.0, 0.3]   # mount 0.3 m behind the body origin, looking along body +z
    imgs = []
    for seed in range(3):
        pose = random_pose(np.random.default_rng(100 + seed), 1)
        pose[0, :3] = np.random.default_rng(seed).normal(0, 1.0, 3)
        W = oracle.compose_w2c(pose[0], B)
        imgs.append(_frame(sc, K, W, pose=pose))
    for r in imgs[1:]:
        ok = ~(r.masked | imgs[0].masked)
        assert np.abs(r.rgb - imgs[0].rgb)[ok].max() < 1e-4
        assert ok.mean() > 0.99


# ---------------------------------------------------------------- pruning scores (R30)
def test_scores_single_gaussian_closed_form():
    """One isotropic on-axis Gaussian (pin 1 geometry): its blend weight at pixel p is its alpha
    there (T = 1), so w_sum = sum over pixels of min(0.99, o exp(-(dx^2/Sxx + dy^2/Syy)/2)) over
    the pixels where that is >= 1/255, and w_max = min(0.99, o) at the pixel centre on (u, v)
    (reading R30 on top of R12-R14)."""
    z, s, o = 3.0, 0.05, 0.8
    sc = scene_from([0, 0, z], s, opac=o)
    K, W = identity_cam(fx=100.0, fy=120.0, cx=32.5, cy=24.5)
    prm = oracle.RenderParams(64, 48)
    ws, wm, touched, alpha = oracle.frame_scores(sc, np.zeros((0, 7), np.float32), K, W, prm)
    s32, o32 = float(np.float32(s)), float(np.float32(o))
    sxx, syy = s32 * s32 * 100.0 ** 2 / z ** 2 + 0.3, s32 * s32 * 120.0 ** 2 / z ** 2 + 0.3
    py, px = np.mgrid[0:48, 0:64]
    a = o32 * np.exp(-0.5 * (((px + 0.5) - 32.5) ** 2 / sxx + ((py + 0.5) - 24.5) ** 2 / syy))
    a = np.minimum(0.99, a)
    exp_sum = a[a >= 1.0 / 255.0].sum()
    assert ws[0] == pytest.approx(exp_sum, rel=1e-12)
    assert wm[0] == pytest.approx(min(0.99, o32), rel=1e-12)
    assert not touched.any()


def test_scores_two_layers_and_partition_identity():
    """Front-to-back 'over': the back Gaussian's weight at the shared centre pixel is
    (1 - a1) a2, and summed over all Gaussians the weights of a pixel are its alpha = 1 - T, so
    sum_i w_sum_i = sum_p alpha_p (pin 9 identity, here per Gaussian) — on a two-layer scene and
    on random tiny scenes with bodies; scores do not depend on the R8 acceleration (pin 10)."""
    K, W = identity_cam()
    prm = oracle.RenderParams(64, 48)
    sc = scene_from([[0, 0, 2.0], [0, 0, 3.0]], [[0.001, 0.001, 0.001], [0.001, 0.001, 0.001]], opac=[0.6, 0.7])
    ws, wm, _, alpha = oracle.frame_scores(sc, np.zeros((0, 7), np.float32), K, W, prm)
    a1, a2 = float(np.float32(0.6)), float(np.float32(0.7))
    # tiny footprint: the centre pixel is the only one above 1/255 for the front Gaussian
    assert wm[0] == pytest.approx(a1, rel=1e-12)
    assert wm[1] == pytest.approx((1 - a1) * a2, rel=1e-12)
    assert ws.sum() == pytest.approx(alpha.sum(), rel=1e-12)
    rng = np.random.default_rng(31)
    for trial in range(4):
        sc = random_tiny_scene(rng, 40, n_bodies=2, sh_degree=1)
        pose = random_pose(rng, 2)
        ws, wm, _, alpha = oracle.frame_scores(sc, pose, K, W, prm)
        assert ws.sum() == pytest.approx(alpha.sum(), rel=1e-12, abs=1e-12)
        assert (wm <= 0.99).all() and (wm >= 0).all()
        assert ((ws > 0) == (wm > 0)).all()
        # pure brute force gives the same scores (the R8 box only skips alpha < 1/255)
        fr = oracle.render_frame(sc, pose, K, W, prm)
        py, px = np.meshgrid(np.arange(48), np.arange(64), indexing="ij")
        sp = {}
        oracle.composite(fr.proj, fr.order, px.reshape(-1), py.reshape(-1), prm, mode="pure", scores=sp)
        np.testing.assert_array_equal(sp["w_sum"], ws)
        np.testing.assert_array_equal(sp["w_max"], wm)


# ---------------------------------------------------------------- observation epilogue (R31)
def test_obs_epilogue_identity_brightness_contrast_and_clamps():
    """Reading R31 with identity DR is the textbook 8-bit encoding rint(clamp(c)*255); an
    additive brightness of m/255 shifts codes by m; contrast pivots about 0.5; gain scales;
    NaN / negative / >1 map to 0 / 0 / 255; depth goes to IEEE half by round-to-nearest-even."""
    from oracle import obs
    codes = np.arange(256)
    c = (codes / 255.0).astype(np.float32).reshape(1, 1, 16, 16).repeat(3, 1)
    q, _ = obs.epilogue(c, None, None)
    np.testing.assert_array_equal(q[0, 0].reshape(-1), codes)
    q, _ = obs.epilogue(c, None, np.float32([[1.0, 1.0, 10 / 255.0, 0.0]]))
    np.testing.assert_array_equal(q[0, 1].reshape(-1), np.minimum(codes + 10, 255))
    half = np.full((1, 3, 2, 2), 0.5, np.float32)
    for k in (0.0, 0.3, 2.0, 7.5):
        q, _ = obs.epilogue(half, None, np.float32([[1.0, k, 0.0, 0.0]]))
        assert (q == 128).all()   # rint(127.5) = 128 (half to even)
    q, _ = obs.epilogue(np.full((1, 3, 1, 1), 0.25, np.float32), None, np.float32([[2.0, 1.0, 0.0, 0.0]]))
    assert (q == 128).all()
    odd = np.float32([np.nan, -0.5, 1.5, 1.0]).reshape(1, 1, 2, 2).repeat(3, 1)
    q, _ = obs.epilogue(odd, None, None)
    np.testing.assert_array_equal(q[0, 0].reshape(-1), [0, 0, 255, 255])
    _, d = obs.epilogue(np.zeros((1, 3, 1, 4), np.float32), np.float32([[[1.0, 2049.0, 3.0e-8, 65520.0]]]), None)
    np.testing.assert_array_equal(d.view(np.uint16).reshape(-1), [0x3C00, 0x6800, 0x0001, 0x7C00])


def test_obs_noise_is_unit_variance_irwin_hall_and_counter_based():
    """The R31 noise: Irwin-Hall(4) of 22-bit hashed uniforms scaled by sqrt(3)/2^22 has mean 0,
    variance 1 and support within 2 sqrt(3) (closed forms); it depends only on (seed, step,
    global frame, pixel, channel) — so env slicing with frame offsets reproduces it — and
    neighbouring channels/pixels are uncorrelated."""
    from oracle import obs
    H, W = 64, 64
    f, ch, y, x = np.meshgrid(np.arange(64), np.arange(3), np.arange(H), np.arange(W), indexing="ij")
    z = obs.noise_z(7, 3, f, y, x, ch, H, W).astype(np.float64) * float(obs.S3)
    assert abs(z.mean()) < 5e-3 and abs(z.std() - 1.0) < 5e-3
    assert np.abs(z).max() <= 2 * np.sqrt(3) + 1e-6
    assert abs(np.corrcoef(z[:, 0].ravel(), z[:, 1].ravel())[0, 1]) < 5e-3
    assert abs(np.corrcoef(z[..., :-1].ravel(), z[..., 1:].ravel())[0, 1]) < 5e-3
    # slicing: frames 10..19 of a batch == frames 0..9 of a slice with offset 10
    rgb = np.random.default_rng(0).uniform(0, 1, (20, 3, 8, 8)).astype(np.float32)
    dr = np.tile(np.float32([1.1, 0.9, 0.02, 0.05]), (20, 1))
    full, _ = obs.epilogue(rgb, None, dr, seed=5, step=9)
    part, _ = obs.epilogue(rgb[10:], None, dr[10:], seed=5, step=9, frame_offset=10)
    np.testing.assert_array_equal(full[10:], part)
    other, _ = obs.epilogue(rgb, None, dr, seed=5, step=10)
    assert (other != full).mean() > 0.3
    assert float(obs.S3) == pytest.approx(np.sqrt(3) / 2 ** 22, rel=1e-7)


# ---------------------------------------------------------------- pin 2b (closed form, rotated)
@pytest.mark.parametrize("theta_deg", [30.0, -65.0, 120.0])
def test_pin2b_rotated_anisotropic_footprint_via_inverse(theta_deg):
    """An anisotropic Gaussian (sa, sb, sc) on the optical axis, rotated by theta about the
    camera z axis through its OWN quaternion: Sigma2D = (f/z)^2 R2 diag(sa^2, sb^2) R2^T + 0.3 I
    with R2 the 2D rotation by theta (J = diag(f/z) there); the conic is np.linalg.inv(Sigma2D),
    so (a, b, c) = inv[0,0], inv[0,1], inv[1,1] including the sign of the off-diagonal b; and
    at off-axis pixels alpha = o exp(-1/2 d^T inv(Sigma2D) d) with d = (u - px, v - py)
    (3DGS EWA [P:212]; readings R7, R12).  A dropped or sign-flipped b term fails here."""
    z, f, sa, sb, sz, o = 3.0, 100.0, 0.08, 0.02, 0.01, 0.9
    h = math.radians(theta_deg) / 2
    q = np.float32([math.cos(h), 0.0, 0.0, math.sin(h)])
    sc = scene_from([0, 0, z], [sa, sb, sz], quats=q, opac=o)
    K, W = identity_cam(fx=f, fy=f, cx=32.5, cy=24.5)
    r = _frame(sc, K, W)
    p = r.proj[0]
    th = 2.0 * math.atan2(float(q[3]), float(q[0]))          # the angle of the fp32 quaternion
    c_, s_ = math.cos(th), math.sin(th)
    R2 = np.array([[c_, -s_], [s_, c_]])
    sa32, sb32 = float(np.float32(sa)), float(np.float32(sb))
    S2 = (f / z) ** 2 * R2 @ np.diag([sa32 ** 2, sb32 ** 2]) @ R2.T + 0.3 * np.eye(2)
    inv = np.linalg.inv(S2)
    assert p[oracle.F_SXX] == pytest.approx(S2[0, 0], rel=1e-10)
    assert p[oracle.F_SYY] == pytest.approx(S2[1, 1], rel=1e-10)
    assert p[oracle.F_SXY] == pytest.approx(S2[0, 1], rel=1e-9, abs=1e-12)
    assert p[oracle.F_A] == pytest.approx(inv[0, 0], rel=1e-9)
    assert p[oracle.F_B] == pytest.approx(inv[0, 1], rel=1e-9)
    assert p[oracle.F_C] == pytest.approx(inv[1, 1], rel=1e-9)
    o32 = float(np.float32(o))
    for dpx, dpy in ((2, 1), (-2, 1), (1, -2), (3, 3), (-3, 2)):
        px, py = 32 + dpx, 24 + dpy
        d = np.array([p[oracle.F_U] - (px + 0.5), p[oracle.F_V] - (py + 0.5)])
        a_exp = min(0.99, o32 * math.exp(-0.5 * d @ inv @ d))
        if a_exp >= 1 / 255:
            assert r.alpha[py, px] == pytest.approx(a_exp, rel=1e-9)
        else:
            assert r.alpha[py, px] == 0.0


# ---------------------------------------------------------------- pin 8b (special case, R4)
def test_pin8b_near_far_cull_boundary():
    """Reading R4 on the fp32 key: keep iff near < z <= far.  Gaussians exactly at near and far
    and one ulp on either side (identity camera: the R11 key is z exactly): at near culled,
    one ulp beyond near kept, at far kept, one ulp beyond far culled; the image shows only the
    kept ones (a culled Gaussian's pixels stay background)."""
    near, far = np.float32(1.0), np.float32(5.0)
    zs = np.float32([near, np.nextafter(near, np.float32(9)), far, np.nextafter(far, np.float32(9))])
    xs = np.float32([-0.3, -0.1, 0.1, 0.3]) * zs
    sc = scene_from(np.stack([xs, np.zeros(4, np.float32), zs], 1), np.repeat(0.02 * zs[:, None], 3, 1), opac=0.9)
    K, W = identity_cam(fx=100, fy=100, cx=32, cy=24)
    prm = oracle.RenderParams(64, 48, near=float(near), far=float(far))
    r = _frame(sc, K, W, prm)
    assert r.zbits.view(np.float32).tolist() == zs.tolist()
    assert r.valid.tolist() == [False, True, True, False]
    for i, kept in enumerate([False, True, True, False]):
        u = int(np.floor(r.proj[i, oracle.F_U])); v = int(np.floor(r.proj[i, oracle.F_V]))
        assert (r.alpha[v, u] > 0.5) == kept, i


# ---------------------------------------------------------------- reading R28 (error bound)
def test_r28_position_bound_covers_a_binary32_projection():
    """Reading R28's position term: F_EU / F_EV bound |u_f32 - u| and |v_f32 - v| for a binary32
    evaluation of the projection chain (x, y, z by the R11-style fma chain of the pose and
    camera rows — mini.depth_key_f32 applied to each camera row — then u = fma(f, x * rn(1/z), c)),
    over random bodies, poses, DR cameras and means spanning a room-sized scene; and the bound
    is not vacuous (within 8x of the worst observed error)."""
    rng = np.random.default_rng(28)
    worst = 0.0
    for trial in range(60):
        W = np.zeros((3, 4), np.float32)
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        W[:, :3] = synth._quat_to_mat(q)
        W[:, 3] = rng.normal(0, 2, 3)
        n = 400
        body = rng.integers(-1, 3, n)
        sc = scene_from(rng.uniform(-3, 3, (n, 3)), 0.02, body=body, n_bodies=3)
        pose = random_pose(rng, 3)
        pose[:, :3] *= 10
        K = np.float32([rng.uniform(50, 600), rng.uniform(50, 600), 320, 240])
        proj, zb, valid = oracle.project(sc, pose, K, W, oracle.RenderParams(640, 480, near=0.05))
        for i in np.nonzero(valid)[0]:
            p = None if body[i] < 0 else pose[body[i]]
            rows = [mini.depth_key_f32(W[[1, 2, r]], p, sc.means[i][None])[0] for r in (0, 1)]
            z32 = zb[i:i + 1].view(np.float32)[0]
            iz = np.float32(1.0 / np.float64(z32))
            u32 = mini.fma32(K[0], np.float32(rows[0] * iz), K[2])
            v32 = mini.fma32(K[1], np.float32(rows[1] * iz), K[3])
            for val, f, fe in ((u32, oracle.F_U, oracle.F_EU), (v32, oracle.F_V, oracle.F_EV)):
                err = abs(float(val) - proj[i, f])
                assert err <= proj[i, fe], (trial, i, err, proj[i, fe])
                worst = max(worst, err / proj[i, fe])
    assert worst >= 1.0 / 8.0, worst


def test_r28_mask_monotone_in_the_bound_and_empty_without_it():
    """margin_scale = 0 disables the mask (no pixel masked, no termination test flagged); the
    masked set only grows with the bound; unmasked pixels are identical (the bound never
    changes what is composited)."""
    cfg = synth.CONFIGS["T1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg, [0])
    prm = oracle.RenderParams(cfg.width, cfg.height)
    fr = [oracle.render_frame(sc, b.poses[0], b.intrinsics[0, 0], b.w2c[0, 0], prm, margin_scale=k)
          for k in (0.0, 1.0, 30.0)]
    assert not fr[0].masked.any() and not fr[0].term_near.any() and not fr[0].eT.any()
    assert np.all(fr[1].masked <= fr[2].masked) and np.all(fr[1].term_near <= fr[2].term_near)
    assert fr[2].masked.sum() > fr[1].masked.sum() > 0
    for f in fr[1:]:
        assert np.array_equal(f.rgb, fr[0].rgb) and np.array_equal(f.alpha, fr[0].alpha)
