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
