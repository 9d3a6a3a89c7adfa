"""§8(f) row 2 — static-camera background pre-binning (gsb_prebin_static / gsb_render_static).

With cameras fixed in the world, the static (body -1) Gaussians are projected, binned and sorted
once per camera; each render bins only the robot Gaussians and K4 merges the two (zbits, id)
ordered lists per tile.  Keys are unique (reading R10), so the merge IS the sort of the union:
every output must be bit-identical to gsb_render with the same cameras broadcast over the envs,
and (through that, and directly on T7) match the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _static_batch(cfg, step=0):
    Ks, Ws = synth.static_cameras(cfg)
    B = cfg.n_envs
    K = np.broadcast_to(Ks, (B,) + Ks.shape).copy()
    W = np.broadcast_to(Ws, (B,) + Ws.shape).copy()
    return Ks, Ws, synth.Batch(synth.make_poses(cfg, np.arange(B), step), K, W)


def _render_static(g, cfg, poses, bg=(0.0, 0.0, 0.0), stats=False):
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    rgb = torch.full((B, C, 3, H, W), float("nan"), device="cuda")
    dep = torch.full((B, C, H, W), float("nan"), device="cuda")
    alp = torch.full((B, C, H, W), float("nan"), device="cuda")
    nev = torch.full((B, C, H, W), -7, dtype=torch.int32, device="cuda")
    g.render_static(gu.to_dev(poses), gsb.RenderParams(W, H, background=bg, stats=stats), rgb, dep, alp, nev)
    torch.cuda.synchronize()
    return dict(rgb=rgb.cpu().numpy(), depth=dep.cpu().numpy(), alpha=alp.cpu().numpy(), n_eval=nev.cpu().numpy())


def _assert_identical(a, b):
    for k in ("rgb", "depth", "alpha", "n_eval"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", ["T1", "T2", "T3", "T4", "T6", "T7"])
def test_static_render_bit_identical_to_broadcast_render(name):
    cfg = synth.CONFIGS[name]
    sc = synth.make_scene(cfg)
    Ks, Ws, b = _static_batch(cfg)
    ref = gu.gpu_render(sc, b, cfg.width, cfg.height, stats=True)
    g = ref["scene"]
    g.prebin_static(Ks, Ws, gsb.RenderParams(cfg.width, cfg.height))
    g.reserve(cfg.n_envs, cfg.n_cams, cfg.width, cfg.height)
    out = _render_static(g, cfg, b.poses, stats=True)
    _assert_identical(out, ref)
    assert g.stats() == ref["stats"]
    # a later physics step with the same pre-binning (the point of pre-binning)
    _, _, b5 = _static_batch(cfg, step=5)
    ref5 = gu.gpu_render(sc, b5, cfg.width, cfg.height, gscene=g)
    _assert_identical(_render_static(g, cfg, b5.poses), ref5)


def test_static_robot_heavy_lists_match_oracle_and_chunking():
    """T7: thousands of robot Gaussians in a few tiles (robot lists beyond K4's fused-sort
    capacity -> sorted in HBM, merged positions in global scratch); every frame against the
    oracle, and chunk / key-capacity invariance of the static path."""
    cfg = synth.CONFIGS["T7"]
    sc = synth.make_scene(cfg)
    Ks, Ws, b = _static_batch(cfg)
    g = gsb.Scene.from_synth(sc)
    g.prebin_static(Ks, Ws, gsb.RenderParams(cfg.width, cfg.height))
    g.reserve(cfg.n_envs, cfg.n_cams, cfg.width, cfg.height)
    prm = gsb.RenderParams(cfg.width, cfg.height, timing=True)
    out = _render_static(g, cfg, b.poses)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    rgb = torch.empty((B, C, 3, H, W), device="cuda")
    g.render_static(gu.to_dev(b.poses), prm, rgb)
    torch.cuda.synchronize()
    assert g.timings()["max_list"] > 1024, "T7 must exercise robot lists sorted in HBM"
    rec, zb, va = gu.gpu_project(g, b, W, H)
    kap = gu.kappa_f32(sc)
    for e in range(B):
        ref = oracle.render_frame(sc, b.poses[e], Ks[0], Ws[0], oracle.RenderParams(W, H))
        r = gu.compare_frame(out, e, 0, ref, W, H, gpu_rec=rec[e], gpu_zb=zb[e], gpu_valid=va[e], kap=kap)
        print("T7 static", e, r)
        assert r["rgb_fail"] == 0 and r["dep_fail"] == 0 and r["alp_fail"] == 0 and r["n_eval_fail"] == 0, r
    # chunk of one frame and a key capacity forcing one frame per pass: bit-identical
    g2 = gsb.Scene.from_synth(sc)
    g2.prebin_static(Ks, Ws, gsb.RenderParams(W, H))
    g2.reserve(B, C, W, H, 1, 60000)
    _assert_identical(_render_static(g2, cfg, b.poses), out)


def test_static_background_and_errors():
    cfg = synth.CONFIGS["T1"]
    sc = synth.make_scene(cfg)
    Ks, Ws, b = _static_batch(cfg)
    g = gsb.Scene.from_synth(sc)
    g.reserve(cfg.n_envs, cfg.n_cams, cfg.width, cfg.height)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    rgb = torch.empty((B, C, 3, H, W), device="cuda")
    with pytest.raises(gsb.GsbError) as ei:   # no pre-binning yet
        g.render_static(gu.to_dev(b.poses), gsb.RenderParams(W, H), rgb)
    assert ei.value.status == 1
    # pre-binning from HOST arrays, before the (re-)reservation
    g.prebin_static(Ks, Ws, gsb.RenderParams(W, H))
    g.reserve(B, C, W, H)
    with pytest.raises(gsb.GsbError) as ei:   # image size differs from the pre-binning
        g.render_static(gu.to_dev(b.poses), gsb.RenderParams(W - 1, H), rgb)
    assert ei.value.status == 2
    with pytest.raises(gsb.GsbError) as ei:   # SH degree differs
        g.render_static(gu.to_dev(b.poses), gsb.RenderParams(W, H, sh_degree=0), rgb)
    assert ei.value.status == 2
    # background colour may differ from the pre-binning's: identical to gsb_render with it
    bg = (0.2, 0.4, 0.6)
    ref = gu.gpu_render(sc, b, W, H, bg=bg)
    _assert_identical(_render_static(g, cfg, b.poses, bg=bg), ref)
    # pre-binning from DEVICE tensors gives the same result
    g.prebin_static(gu.to_dev(Ks), gu.to_dev(Ws), gsb.RenderParams(W, H))
    _assert_identical(_render_static(g, cfg, b.poses, bg=bg), ref)


@pytest.mark.parametrize("path", ["split", "fused"])
@pytest.mark.parametrize("name", ["T2", "T6", "T7"])
def test_static_merge_both_k4_paths_bit_identical(name, path, monkeypatch):
    """The merge runs in the split path (K4a writes the merged list, K4b decodes background
    entries) or in the fused kernel, chosen by list length; force each: bit-identical to
    gsb_render on the broadcast cameras."""
    monkeypatch.setenv("GSB_K4_SPLIT_MIN", "0" if path == "split" else "1000000000")
    cfg = synth.CONFIGS[name]
    sc = synth.make_scene(cfg)
    Ks, Ws, b = _static_batch(cfg)
    ref = gu.gpu_render(sc, b, cfg.width, cfg.height)
    g = ref["scene"]
    g.prebin_static(Ks, Ws, gsb.RenderParams(cfg.width, cfg.height))
    g.reserve(cfg.n_envs, cfg.n_cams, cfg.width, cfg.height)
    _assert_identical(_render_static(g, cfg, b.poses), ref)


@pytest.mark.parametrize("name", ["T2", "T5", "T7"])
def test_static_per_env_cameras_bit_identical(name):
    """GSB_FLAG_STATIC_PER_ENV: every env has its own domain-randomised camera, fixed over the
    episode, pre-binned once; rendering env e with pre-binned camera e is bit-identical to
    gsb_render with the same per-env cameras, at two physics steps and for an env prefix."""
    cfg = synth.CONFIGS[name]
    sc = synth.make_scene(cfg)
    B = cfg.n_envs + 2
    ids = np.arange(B)
    K, Wc = synth.make_cameras(cfg, ids)
    K, Wc = K[:, :1].copy(), Wc[:, :1].copy()          # one camera per env
    g = gsb.Scene.from_synth(sc)
    g.prebin_static(K[:, 0].copy(), Wc[:, 0].copy(), gsb.RenderParams(cfg.width, cfg.height))
    g.reserve(B, 1, cfg.width, cfg.height)
    H, W = cfg.height, cfg.width
    for step in (0, 4):
        b = synth.Batch(synth.make_poses(cfg, ids, step), K, Wc)
        ref = gu.gpu_render(sc, b, W, H, gscene=g, stats=True)
        for n in (B, B - 1):
            rgb = torch.full((n, 1, 3, H, W), float("nan"), device="cuda")
            dep = torch.full((n, 1, H, W), float("nan"), device="cuda")
            alp = torch.full((n, 1, H, W), float("nan"), device="cuda")
            nev = torch.full((n, 1, H, W), -7, dtype=torch.int32, device="cuda")
            g.render_static(gu.to_dev(b.poses[:n]), gsb.RenderParams(W, H, static_per_env=True, stats=True), rgb, dep,
                            alp, nev)
            torch.cuda.synchronize()
            out = dict(rgb=rgb.cpu().numpy(), depth=dep.cpu().numpy(), alpha=alp.cpu().numpy(), n_eval=nev.cpu().numpy())
            _assert_identical(out, {k: v[:n] for k, v in ref.items() if k in ("rgb", "depth", "alpha", "n_eval")})
            if n == B:
                assert g.stats() == ref["stats"]
    with pytest.raises(gsb.GsbError):   # more envs than pre-binned cameras
        g.reserve(B + 1, 1, W, H)
        g.render_static(gu.to_dev(synth.make_poses(cfg, np.arange(B + 1), 0)),
                        gsb.RenderParams(W, H, static_per_env=True), torch.zeros((B + 1, 1, 3, H, W), device="cuda"))
