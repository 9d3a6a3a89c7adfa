"""Seeded workload generators: determinism and env-slice independence."""
import numpy as np

import synth


def test_scene_deterministic_and_shapes():
    cfg = synth.CONFIGS["T1"]
    a, b = synth.make_scene(cfg), synth.make_scene(cfg)
    assert a.n == cfg.n_gaussians
    assert a.sh.shape == (cfg.n_gaussians, (cfg.sh_degree + 1) ** 2, 3)
    for f in ("means", "scales", "quats", "opacities", "sh", "body_id"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert np.all(a.scales > 0) and np.all((a.opacities > 0) & (a.opacities <= 1))
    assert set(np.unique(a.body_id)) == set(range(-1, cfg.n_bodies))
    # static first, bodies contiguous
    assert np.all(np.diff(a.body_id) >= 0)


def test_env_inputs_independent_of_batch_and_slice():
    cfg = synth.CONFIGS["C2"]
    full = synth.make_batch(cfg, np.arange(8), step=3)
    part = synth.make_batch(cfg, np.arange(5, 8), step=3)
    assert np.array_equal(full.poses[5:], part.poses)
    assert np.array_equal(full.w2c[5:], part.w2c)
    assert np.array_equal(full.intrinsics[5:], part.intrinsics)


def test_env_slices_partition():
    for B in (1, 7, 64, 1024):
        for G in (1, 2, 3, 8):
            sl = [synth.env_slice(B, r, G) for r in range(G)]
            assert sl[0][0] == 0 and sl[-1][1] == B
            assert all(sl[i][1] == sl[i + 1][0] for i in range(G - 1))


def test_camera_dr_ranges():
    """Per-env camera DR: |dt| <= 0.02 m per axis, rotation <= 5 deg."""
    cfg = synth.CONFIGS["C4"]
    K, W = synth.make_cameras(cfg, np.arange(16))
    for c, (eye0, tgt) in enumerate(synth.NOMINAL_CAMS[: cfg.n_cams]):
        R0 = synth._look_at_c2w(eye0, tgt).T
        for e in range(16):
            R = W[e, c, :, :3].astype(np.float64)
            eye = -R.T @ W[e, c, :, 3]
            assert np.all(np.abs(eye - np.array(eye0)) <= 0.02 + 1e-5)
            cosang = (np.trace(R @ R0.T) - 1) / 2
            assert np.degrees(np.arccos(np.clip(cosang, -1, 1))) <= 5.0 + 1e-3
            assert np.allclose(R @ R.T, np.eye(3), atol=1e-6)


def test_pose_quaternions_unit_and_chain_links():
    cfg = synth.CONFIGS["C3"]
    p = synth.make_poses(cfg, np.arange(4), step=7)
    assert p.shape == (4, cfg.n_bodies, 7)
    assert np.allclose(np.linalg.norm(p[..., 3:], axis=-1), 1, atol=1e-6)
    d = np.linalg.norm(np.diff(p[..., :3].astype(np.float64), axis=1), axis=-1)
    assert np.allclose(d, 0.3, atol=1e-5)


def test_sample_pixels_stratified_and_full_tiles():
    """SURVEY d.6 sample: one pixel per cell of a 64x64 grid + every pixel of 2 tiles."""
    for W, H in ((640, 480), (128, 128), (1280, 720), (224, 224), (17, 9)):
        px, py, n = synth.sample_pixels(W, H, seed=3)
        g = (min(64, W), min(64, H))
        assert n == g[0] * g[1]
        assert px.min() >= 0 and px.max() < W and py.min() >= 0 and py.max() < H
        bx = (np.arange(g[0] + 1) * W) // g[0]        # cell boundaries
        by = (np.arange(g[1] + 1) * H) // g[1]
        cx, cy = np.searchsorted(bx, px[:n], side="right") - 1, np.searchsorted(by, py[:n], side="right") - 1
        assert len(set(zip(cx.tolist(), cy.tolist()))) == n     # one pixel in every cell
        tiles = set(((py[n:] // 16) * ((W + 15) // 16) + px[n:] // 16).tolist())
        assert len(tiles) == min(2, ((W + 15) // 16) * ((H + 15) // 16))
        for t in tiles:   # each drawn tile complete (ragged edges included)
            x0, y0 = (t % ((W + 15) // 16)) * 16, (t // ((W + 15) // 16)) * 16
            size = (min(x0 + 16, W) - x0) * (min(y0 + 16, H) - y0)
            assert np.sum(((py[n:] // 16) * ((W + 15) // 16) + px[n:] // 16) == t) == size
    a, b = synth.sample_pixels(640, 480, 5), synth.sample_pixels(640, 480, 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
