"""§8(f) row 4 — batched ray-cast LiDAR (gsb_lidar_create / gsb_render_lidar, reading R32)
against the CPU oracle (oracle.lidar_frame: brute force per ray over every Gaussian in
(bits(rho_f32), id) order), element by element on every ray.

Bars (the camera bars of BASELINE.json north_star with range for depth): |d alpha| <= 2e-3,
|d range| <= 1e-3 range + 1e-6 on rays outside the reading-R28 threshold-margin mask.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from tests import gpu_util as gu
from tests.helpers import scene_from

pytestmark = pytest.mark.gpu

MASK_CAP = oracle.MASK_CAP


def _sensors(cfg, env_ids, with_body=True):
    """sensor 0: world-fixed per env; sensor 1: on body 0 (R29 mount) when the scene has bodies."""
    Wsens = synth.lidar_world_sensor(cfg, env_ids)
    if not with_body or cfg.n_bodies == 0:
        return Wsens[:, None].copy(), None
    mount = synth.lidar_body_mount()
    sx = np.stack([Wsens, np.broadcast_to(mount, Wsens.shape)], 1).copy()
    return sx, np.int32([-1, 0])


def _gpu_lidar(g, lid, poses, sx, sensor_body, near=0.01, far=1000.0):
    B, S = sx.shape[0], sx.shape[1]
    rng_t = torch.full((B, S, lid.n_rays), float("nan"), device="cuda")
    alp_t = torch.full((B, S, lid.n_rays), float("nan"), device="cuda")
    lid.render(gu.to_dev(poses), gu.to_dev(sx), rng_t, alp_t, sensor_body=sensor_body, near=near, far=far)
    torch.cuda.synchronize()
    return rng_t.cpu().numpy(), alp_t.cpu().numpy()


def _w2s(sx, sensor_body, poses, e, s):
    if sensor_body is not None and sensor_body[s] >= 0:
        return oracle.compose_w2c(poses[e][sensor_body[s]], sx[e, s])   # R29, bit-identical to K0
    return sx[e, s]


def _compare(g_rng, g_alp, ref: oracle.LidarResult, rays=None):
    if rays is not None:
        g_rng, g_alp = g_rng[rays], g_alp[rays]
    ok = ~ref.masked
    d_r = np.abs(g_rng - ref.range)
    d_a = np.abs(g_alp - ref.alpha)
    bar_r = oracle.TOL_DEPTH_REL * np.abs(ref.range) + oracle.TOL_DEPTH_ABS
    return dict(masked_frac=float(ref.masked.mean()),
                max_alpha=float(d_a[ok].max()) if ok.any() else 0.0,
                max_range_excess=float((d_r - bar_r)[ok].max()) if ok.any() else -1.0,
                alpha_fail=int((d_a[ok] > oracle.TOL_ALPHA).sum()),
                range_fail=int((d_r > bar_r)[ok].sum()),
                hit_frac=float((ref.alpha > 0.5).mean()),
                masked_max_alpha=float(d_a[~ok].max()) if (~ok).any() else 0.0)


def _check(res, tag):
    print(tag, res)
    assert res["alpha_fail"] == 0 and res["range_fail"] == 0, (tag, res)
    assert res["masked_frac"] <= MASK_CAP, (tag, res)


PATTERNS = {
    "rotating": lambda: synth.lidar_pattern("rotating", 16, 256),
    "solid_state": lambda: synth.lidar_pattern("solid_state", 24, 96),
    "non_repetitive": lambda: synth.lidar_pattern("non_repetitive", n_points=1500, step=3),
    "height_scan": lambda: synth.lidar_pattern("height_scan", 11, 17),
    "random": lambda: synth.lidar_pattern("random", n_points=2048, seed=4),
}


@pytest.mark.parametrize("cfg_name,pattern", [("T1", "rotating"), ("T2", "non_repetitive"), ("T5", "solid_state"),
                                              ("T3", "random"), ("T1", "height_scan"), ("T4", "random")])
def test_lidar_matches_oracle(cfg_name, pattern):
    cfg = synth.CONFIGS[cfg_name]
    scene = synth.make_scene(cfg)
    B = cfg.n_envs
    poses = synth.make_poses(cfg, np.arange(B), 1)
    sx, sb = _sensors(cfg, np.arange(B))
    dirs = PATTERNS[pattern]()
    g = gsb.Scene.from_synth(scene)
    lid = gsb.Lidar(g, dirs)
    g_rng, g_alp = _gpu_lidar(g, lid, poses, sx, sb)
    info = lid.info()
    assert info["keys"] > 0
    hit = 0.0
    for e in range(B):
        for s in range(sx.shape[1]):
            ref = oracle.lidar_frame(scene, poses[e], _w2s(sx, sb, poses, e, s), dirs)
            res = _compare(g_rng[e, s], g_alp[e, s], ref)
            _check(res, f"{cfg_name}/{pattern} env {e} sensor {s} {info}")
            hit = max(hit, res["hit_frac"])
    assert hit > 0.05   # the rays do see the scene


def test_lidar_closed_form_scene_and_edges():
    """Hand-built scene: Gaussians straddling the azimuth seam (+-180 deg) and the poles, one
    around the sensor, one behind near-plane; every ray compared with the oracle; a batch of
    0 envs is a no-op; bad arguments fail."""
    means = [[-3.0, 0.001, 0.0], [-3.0, -0.001, 0.2], [0.0, 0.0, 2.5], [0.0, 0.0, -2.5], [0.0, 0.0, 0.0],
             [2.0, 0.5, 0.1], [0.004, 0.0, 0.0]]
    scales = [[0.3, 0.3, 0.3], [0.05, 0.4, 0.05], [0.5, 0.5, 0.2], [0.2, 0.2, 0.2], [1.5, 1.5, 1.5],
              [0.1, 0.02, 0.3], [0.002, 0.002, 0.002]]
    sc = scene_from(means, scales, opac=[0.9, 0.8, 0.7, 0.95, 0.05, 0.6, 0.9])
    dirs = synth.lidar_pattern("random", n_points=4000, seed=9)
    g = gsb.Scene.from_synth(sc)
    sx = np.hstack([np.eye(3), np.zeros((3, 1))]).astype(np.float32)[None, None].copy()
    for n_az, n_el in [(0, 0), (7, 5), (256, 1), (1, 256)]:
        lid = gsb.Lidar(g, dirs, n_az, n_el)
        g_rng, g_alp = _gpu_lidar(g, lid, np.zeros((1, 0, 7), np.float32), sx, None)
        ref = oracle.lidar_frame(sc, np.zeros((0, 7), np.float32), sx[0, 0], dirs)
        _check(_compare(g_rng[0, 0], g_alp[0, 0], ref), f"edges n_az={n_az} n_el={n_el} {lid.info()}")
        lid.close()
    lid = gsb.Lidar(g, dirs)
    out = torch.zeros((0, 1, lid.n_rays), device="cuda")
    lid.render(None, gu.to_dev(sx[:0]), out)     # 0 envs
    with pytest.raises(gsb.GsbError):
        gsb.Lidar(g, np.float32([[1.0, 1.0, 0.0]]))      # not a unit vector
    with pytest.raises(gsb.GsbError):
        lid.render(None, gu.to_dev(sx), torch.zeros((1, 1, lid.n_rays), device="cuda"), near=1.0, far=0.5)


def test_lidar_slicing_bit_identical():
    """An env slice renders bit-identically to the same envs inside a larger batch."""
    cfg = synth.CONFIGS["T2"]
    scene = synth.make_scene(cfg)
    ids = np.arange(4)
    poses = synth.make_poses(cfg, ids, 2)
    sx, sb = _sensors(cfg, ids)
    dirs = synth.lidar_pattern("rotating", 8, 128)
    g = gsb.Scene.from_synth(scene)
    lid = gsb.Lidar(g, dirs)
    r_all, a_all = _gpu_lidar(g, lid, poses, sx, sb)
    r_sl, a_sl = _gpu_lidar(g, lid, poses[1:3], sx[1:3], sb)
    assert np.array_equal(r_all[1:3].view(np.uint32), r_sl.view(np.uint32))
    assert np.array_equal(a_all[1:3].view(np.uint32), a_sl.view(np.uint32))


def test_lidar_c3_full_size_sampled_rays():
    """The bench workload (C3 scene, 520 k Gaussians, a 32 x 1024 rotating LiDAR on body 0 of
    every env): 3 envs x 384 sampled rays against the oracle, in the bench's launch
    configuration (all 1024 envs in one call)."""
    cfg = synth.CONFIGS["C3"]
    scene = synth.make_scene(cfg)
    B = cfg.n_envs
    poses = synth.make_poses(cfg, np.arange(B), 0)
    mount = synth.lidar_body_mount()[None].copy()
    dirs = synth.lidar_pattern("rotating", 32, 1024)
    g = gsb.Scene.from_synth(scene)
    lid = gsb.Lidar(g, dirs)
    rng_t = torch.zeros((B, 1, lid.n_rays), device="cuda")
    alp_t = torch.zeros((B, 1, lid.n_rays), device="cuda")
    lid.render(gu.to_dev(poses), gu.to_dev(mount), rng_t, alp_t, sensor_body=[0])
    torch.cuda.synchronize()
    r = np.random.default_rng(0)
    for e in (0, B // 2, B - 1):
        rays = np.sort(r.choice(lid.n_rays, 384, replace=False))
        w2s = oracle.compose_w2c(poses[e][0], mount[0])
        ref = oracle.lidar_frame(scene, poses[e], w2s, dirs[rays])
        res = _compare(rng_t[e, 0].cpu().numpy(), alp_t[e, 0].cpu().numpy(), ref, rays)
        _check(res, f"C3 lidar env {e} {lid.info()}")


def test_lidar_many_sensors_max_grid_single_ray():
    """Sixteen sensors per env (alternating world-fixed and body-mounted on different bodies),
    the largest cell grid (256 x 256), and a one-ray pattern: every ray against the oracle."""
    cfg = synth.CONFIGS["T4"]
    scene = synth.make_scene(cfg)
    B, S = cfg.n_envs, 16
    poses = synth.make_poses(cfg, np.arange(B), 3)
    Wsens = synth.lidar_world_sensor(cfg, np.arange(B))
    mount = synth.lidar_body_mount()
    sx = np.zeros((B, S, 3, 4), np.float32)
    sb = np.full(S, -1, np.int32)
    for s in range(S):
        if s % 2:
            sb[s] = s % cfg.n_bodies
            sx[:, s] = mount
        else:
            sx[:, s] = Wsens
    g = gsb.Scene.from_synth(scene)
    for dirs, grid in ((synth.lidar_pattern("random", n_points=3000, seed=11), (256, 256)),
                       (np.float32([[0.6, 0.0, -0.8]]), (0, 0))):
        lid = gsb.Lidar(g, dirs, *grid)
        g_rng, g_alp = _gpu_lidar(g, lid, poses, sx, sb)
        for e in range(B):
            for s in range(S):
                ref = oracle.lidar_frame(scene, poses[e], _w2s(sx, sb, poses, e, s), dirs)
                _check(_compare(g_rng[e, s], g_alp[e, s], ref), f"sensors env {e} sensor {s} {lid.info()}")
        lid.close()


def test_lidar_empty_scene_and_culled_ranges():
    """N = 0: every ray returns range 0, alpha 0.  A near/far window excluding every Gaussian
    gives the same; a window keeping some matches the oracle with the same near/far."""
    sc = scene_from(np.zeros((0, 3)), np.zeros((0, 3)))
    g = gsb.Scene.from_synth(sc)
    dirs = synth.lidar_pattern("rotating", 4, 32)
    lid = gsb.Lidar(g, dirs)
    sx = np.hstack([np.eye(3), np.zeros((3, 1))]).astype(np.float32)[None, None].copy()
    r, a = _gpu_lidar(g, lid, np.zeros((1, 0, 7), np.float32), sx, None)
    assert (r == 0).all() and (a == 0).all()
    cfg = synth.CONFIGS["T3"]
    scene = synth.make_scene(cfg)
    g2 = gsb.Scene.from_synth(scene)
    lid2 = gsb.Lidar(g2, dirs)
    sx2 = synth.lidar_world_sensor(cfg, [0])[:, None].copy()
    r, a = _gpu_lidar(g2, lid2, np.zeros((1, 0, 7), np.float32), sx2, None, near=900.0, far=1000.0)
    assert (r == 0).all() and (a == 0).all()
    r, a = _gpu_lidar(g2, lid2, np.zeros((1, 0, 7), np.float32), sx2, None, near=2.0, far=4.0)
    ref = oracle.lidar_frame(scene, np.zeros((0, 7), np.float32), sx2[0, 0], dirs, near=2.0, far=4.0)
    _check(_compare(r[0, 0], a[0, 0], ref), "near/far window")
