"""§8(f) row 3 — renderer-driven pruning scores (GSB_FLAG_SCORES, reading R30) and
filter_template semantics (gsb_filter_scene), against the oracle.

Score bar: per Gaussian, over all frames of the batch, w_sum within 1e-3 relative + 1e-5
absolute of the oracle's fp64 sum (fp32 weights, fp32 atomic accumulation in unfixed order) and
w_max within 2e-4 relative + 1e-6 — for every Gaussian not "touched" by an R28 threshold-margin
pixel (where either side of a flip is correct, so its weight there is not unique).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _render(g, b, W, H, scores=False, bg=(0.0, 0.0, 0.0)):
    B, C = b.intrinsics.shape[:2]
    rgb = torch.empty((B, C, 3, H, W), device="cuda")
    dep = torch.empty((B, C, H, W), device="cuda")
    alp = torch.empty((B, C, H, W), device="cuda")
    nev = torch.empty((B, C, H, W), dtype=torch.int32, device="cuda")
    g.render(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c),
             gsb.RenderParams(W, H, background=bg, scores=scores), rgb, dep, alp, nev)
    torch.cuda.synchronize()
    return dict(rgb=rgb.cpu().numpy(), depth=dep.cpu().numpy(), alpha=alp.cpu().numpy(), n_eval=nev.cpu().numpy())


@pytest.mark.parametrize("path", ["split", "fused"])
@pytest.mark.parametrize("name", ["T1", "T2", "T6"])
def test_scores_match_oracle(name, path, monkeypatch):
    """Both compositing paths (K4b's per-warp atomics, the fused kernel's per-CTA shared sums)."""
    monkeypatch.setenv("GSB_K4_SPLIT_MIN", "0" if path == "split" else "1000000000")
    cfg = synth.CONFIGS[name]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    W, H = cfg.width, cfg.height
    g = gsb.Scene.from_synth(sc)
    g.reserve(cfg.n_envs, cfg.n_cams, W, H)
    plain = _render(g, b, W, H)
    g.scores_reset()
    scored = _render(g, b, W, H, scores=True)
    for k in plain:   # the score variant composites exactly like the plain one
        assert np.array_equal(plain[k], scored[k]), k
    ws, wm = (t.cpu().numpy().astype(np.float64) for t in g.scores())
    ref_s, ref_m = np.zeros(sc.n), np.zeros(sc.n)
    touched = np.zeros(sc.n, bool)
    alpha_sum = 0.0
    for e in range(cfg.n_envs):
        for c in range(cfg.n_cams):
            s_, m_, t_, _ = oracle.frame_scores(sc, b.poses[e], b.intrinsics[e, c], b.w2c[e, c],
                                                oracle.RenderParams(W, H))
            ref_s += s_
            ref_m = np.maximum(ref_m, m_)
            touched |= t_
            alpha_sum += float(scored["alpha"][e, c].astype(np.float64).sum())
    ok = ~touched
    err_s = np.abs(ws - ref_s)
    err_m = np.abs(wm - ref_m)
    print(name, "touched", int(touched.sum()), "of", sc.n, "scored", int((ref_s > 0).sum()),
          "max rel sum err", float((err_s[ok] / np.maximum(ref_s[ok], 1e-30)).max(initial=0)),
          "max abs max err", float(err_m[ok].max(initial=0)))
    assert (err_s[ok] <= 1e-3 * ref_s[ok] + 1e-5).all()
    assert (err_m[ok] <= 2e-4 * ref_m[ok] + 1e-6).all()
    assert ok[ref_s > 0].mean() >= 0.5   # most scored Gaussians are checked exactly
    assert ((ws > 0) == (ref_s > 0))[ok].all()
    # per-pixel partition identity on the device: sum of all weights = sum of alpha
    assert ws.sum() == pytest.approx(alpha_sum, rel=1e-4)
    # accumulation across renders, and reset
    _render(g, b, W, H, scores=True)
    ws2, wm2 = (t.cpu().numpy().astype(np.float64) for t in g.scores())
    np.testing.assert_allclose(ws2, 2 * ws, rtol=1e-5, atol=1e-6)
    np.testing.assert_array_equal(wm2, wm)
    g.scores_reset()
    ws3, wm3 = g.scores()
    assert float(ws3.abs().max()) == 0.0 and float(wm3.abs().max()) == 0.0


def _subset(sc: synth.Scene, keep):
    return synth.Scene(sc.means[keep], sc.scales[keep], sc.quats[keep], sc.opacities[keep], sc.sh[keep],
                       sc.sh_degree, sc.body_id[keep], sc.n_bodies)


def test_filter_scene_template_semantics():
    """predicate true -> identical; false -> empty (background); keep every
    other -> the result renders bit-identically to a scene built from the subset directly."""
    cfg = synth.CONFIGS["T1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    W, H = cfg.width, cfg.height
    g = gsb.Scene.from_synth(sc)
    g.reserve(cfg.n_envs, cfg.n_cams, W, H)
    full = _render(g, b, W, H)
    g_all = g.filter(np.ones(sc.n, bool))
    g_all.reserve(cfg.n_envs, cfg.n_cams, W, H)
    out = _render(g_all, b, W, H)
    for k in full:
        assert np.array_equal(out[k], full[k]), k
    g_none = g.filter(np.zeros(sc.n, bool))
    assert g_none.n == 0
    g_none.reserve(cfg.n_envs, cfg.n_cams, W, H)
    bg = (0.25, 0.5, 0.75)
    out = _render(g_none, b, W, H, bg=bg)
    assert np.array_equal(out["rgb"], np.broadcast_to(np.float32(bg)[None, None, :, None, None], out["rgb"].shape))
    assert not out["depth"].any() and not out["alpha"].any()
    keep = np.arange(sc.n) % 2 == 0
    g_half = g.filter(keep)
    g_half.reserve(cfg.n_envs, cfg.n_cams, W, H)
    direct = gsb.Scene.from_synth(_subset(sc, keep))
    direct.reserve(cfg.n_envs, cfg.n_cams, W, H)
    a, d = _render(g_half, b, W, H), _render(direct, b, W, H)
    for k in a:
        assert np.array_equal(a[k], d[k]), k
    with pytest.raises(ValueError):
        g.filter(np.ones(sc.n - 1, bool))


def test_score_pruning_beats_random_pruning():
    """The mechanism the paper relies on: keeping the 30% highest-score Gaussians (fewer
    than the ones these views blend at all, so blended ones go too) changes the rendered frames
    far less than keeping a random 30% (PSNR against the full render, same views)."""
    cfg = synth.CONFIGS["T2"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    W, H = cfg.width, cfg.height
    g = gsb.Scene.from_synth(sc)
    g.reserve(cfg.n_envs, cfg.n_cams, W, H)
    g.scores_reset()
    full = _render(g, b, W, H, scores=True)["rgb"]
    ws, _ = g.scores()
    keep_s = gsb.prune_mask(ws, 0.3)
    assert keep_s.sum() < int((ws > 0).sum().item())
    keep_r = np.random.default_rng(5).permutation(sc.n) < keep_s.sum()

    def psnr(keep):
        gp = g.filter(keep)
        gp.reserve(cfg.n_envs, cfg.n_cams, W, H)
        img = _render(gp, b, W, H)["rgb"]
        mse = float(((img.astype(np.float64) - full) ** 2).mean())
        return 10 * np.log10(1.0 / max(mse, 1e-20))

    p_s, p_r = psnr(keep_s), psnr(keep_r)
    print("PSNR score-pruned", p_s, "random-pruned", p_r, "never-blended", int((ws == 0).sum().item()))
    assert p_s > p_r + 3.0
