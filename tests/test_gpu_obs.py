"""§8(f) row 4 — observation epilogue (gsb_render_obs / gsb_render_obs_host, reading R31):
image DR + uint8 RGB + fp16 depth fused into K4's store, against oracle/obs.py.

Bars: where the epilogue's input is exactly known (background-only frames: c = bg in binary32)
the codes, noise included, are bit-exact; on rendered scenes the integer code is decided by
each side in binary32 from its own composite, so codes agree within 1 (a composite within
~1e-5 of a rounding boundary may round either way), exactly on >= 99.5 % of unmasked pixels.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from oracle import obs as obs_oracle
from tests import gpu_util as gu
from tests.helpers import scene_from

pytestmark = pytest.mark.gpu


def _dr(rng, B, C, noise=True):
    d = np.stack([rng.uniform(0.6, 1.6, (B, C)), rng.uniform(0.5, 1.5, (B, C)), rng.uniform(-0.1, 0.1, (B, C)),
                  rng.uniform(0.0, 0.05, (B, C)) if noise else np.zeros((B, C))], -1)
    return d.astype(np.float32)


def _obs_render(g, b, W, H, dr, seed, step, env_offset=0, f16=True, bg=(0.0, 0.0, 0.0)):
    B, C = b.intrinsics.shape[:2]
    rgb8 = torch.full((B, C, 3, H, W), 77, dtype=torch.uint8, device="cuda")
    dep = torch.full((B, C, H, W), -1, dtype=torch.float16 if f16 else torch.float32, device="cuda")
    g.render_obs(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c), gsb.RenderParams(W, H, background=bg),
                 rgb8, dep, image_dr=None if dr is None else gu.to_dev(dr), seed=seed, step=step,
                 env_offset=env_offset, depth_f16=f16)
    torch.cuda.synchronize()
    return rgb8.cpu().numpy(), dep.cpu().numpy()


def test_obs_bit_exact_on_known_composites():
    """Empty scene: every pixel's composite is the background exactly, so the R31 codes (DR and
    counter-based noise included) must match the oracle bit for bit, for several backgrounds,
    seeds, steps and env offsets; depth is +0 in fp16."""
    sc = scene_from(np.zeros((0, 3)), np.zeros((0, 3)))
    B, C, H, W = 3, 2, 37, 53
    K = np.tile(np.float32([50, 50, 26.5, 18.5]), (B, C, 1))
    Wc = np.zeros((B, C, 3, 4), np.float32)
    Wc[..., :3, :3] = np.eye(3)
    b = synth.Batch(np.zeros((B, 0, 7), np.float32), K, Wc)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H)
    rng = np.random.default_rng(3)
    for trial in range(6):
        bg = tuple(rng.uniform(0, 1, 3))
        dr = _dr(rng, B, C, noise=trial != 0)
        seed, step, off = int(rng.integers(0, 2 ** 32)), int(rng.integers(0, 2 ** 32)), int(rng.integers(0, 5000))
        q, d = _obs_render(g, b, W, H, dr, seed, step, env_offset=off, bg=bg)
        rgb = np.broadcast_to(np.float32(bg)[None, :, None, None], (B * C, 3, H, W))
        ref, ref_d = obs_oracle.epilogue(rgb, np.zeros((B * C, H, W)), dr.reshape(B * C, 4), seed, step, off * C)
        np.testing.assert_array_equal(q.reshape(B * C, 3, H, W), ref)
        np.testing.assert_array_equal(d.reshape(B * C, H, W).view(np.uint16), ref_d.view(np.uint16))
    # identity DR (NULL) = textbook 8-bit encoding of the background
    q, _ = _obs_render(g, b, W, H, None, 0, 0, bg=(0.2, 0.5, 1.0))
    assert (q[:, :, 0] == 51).all() and (q[:, :, 1] == 128).all() and (q[:, :, 2] == 255).all()


@pytest.mark.parametrize("name", ["T1", "T5"])
def test_obs_codes_match_oracle_on_rendered_frames(name):
    cfg = synth.CONFIGS[name]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H)
    dr = _dr(np.random.default_rng(11), B, C)
    bg = (0.1, 0.2, 0.3)
    q, d16 = _obs_render(g, b, W, H, dr, seed=123, step=4, bg=bg)
    exact = total = 0
    for e in range(B):
        for c in range(C):
            ref = oracle.render_frame(sc, b.poses[e], b.intrinsics[e, c], b.w2c[e, c],
                                      oracle.RenderParams(W, H, bg=bg))
            rq, rd = obs_oracle.epilogue(ref.rgb.transpose(2, 0, 1)[None], ref.depth[None], dr[e, c][None], 123, 4,
                                         e * C + c)
            ok = ~ref.masked
            diff = np.abs(q[e, c].astype(int) - rq[0].astype(int))
            assert diff[:, ok].max() <= 1, (e, c)
            exact += int((diff[:, ok] == 0).sum())
            total += int(diff[:, ok].size)
            dg = d16[e, c].astype(np.float64)
            tol = 1e-3 * ref.depth + 1e-6 + np.abs(rd[0].astype(np.float64)) * 2.0 ** -11
            assert (np.abs(dg - ref.depth)[ok] <= tol[ok]).all(), (e, c)
    print(name, "exact code fraction", exact / total)
    assert exact / total >= 0.995


def test_obs_host_path_slicing_and_fp32_depth():
    cfg = synth.CONFIGS["T1"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H, host_io=True)
    dr = _dr(np.random.default_rng(12), B, C)
    q, d16 = _obs_render(g, b, W, H, dr, seed=9, step=2)
    # host buffers: identical
    hq = torch.empty((B, C, 3, H, W), dtype=torch.uint8).pin_memory()
    hd = torch.empty((B, C, H, W), dtype=torch.float16).pin_memory()
    g.render_obs_host(torch.from_numpy(b.poses), torch.from_numpy(b.intrinsics), torch.from_numpy(b.w2c),
                      gsb.RenderParams(W, H), hq, hd, image_dr=torch.from_numpy(dr), seed=9, step=2)
    assert np.array_equal(hq.numpy(), q) and np.array_equal(hd.numpy().view(np.uint16), d16.view(np.uint16))
    # an env slice rendered alone with its env_offset reproduces its frames (noise keyed globally)
    sl = synth.Batch(b.poses[1:], b.intrinsics[1:], b.w2c[1:])
    qs, _ = _obs_render(g, sl, W, H, dr[1:], seed=9, step=2, env_offset=1)
    assert np.array_equal(qs, q[1:])
    # fp32 depth option = the plain render's depth, bit for bit
    _, d32 = _obs_render(g, b, W, H, dr, seed=9, step=2, f16=False)
    plain = gu.gpu_render(sc, b, W, H, gscene=g)
    assert np.array_equal(d32, plain["depth"])
    with pytest.raises(gsb.GsbError):
        g.render_obs(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c), gsb.RenderParams(W, H), None)


# ---------------------------------------------------------------- reading R33: motion blur
def _encode(rgb, blur=None, dr=None, depth=None, seed=0, step=0, env_offset=0, f16=True):
    B, C, _, H, W = rgb.shape
    out = torch.full((B, C, 3, H, W), 77, dtype=torch.uint8, device="cuda")
    od = None
    if depth is not None:
        od = torch.full((B, C, H, W), -1, dtype=torch.float16 if f16 else torch.float32, device="cuda")
    gsb.obs_encode(gu.to_dev(rgb), out, depth=None if depth is None else gu.to_dev(depth), out_depth=od,
                   blur=None if blur is None else gu.to_dev(np.asarray(blur, np.int32)),
                   image_dr=None if dr is None else gu.to_dev(dr), seed=seed, step=step, env_offset=env_offset,
                   depth_f16=f16)
    torch.cuda.synchronize()
    return out.cpu().numpy(), (None if od is None else od.cpu().numpy())


def test_obs_encode_blur_bit_exact_on_seeded_frames():
    """gsb_obs_encode (K6) on seeded fp32 frames (inputs, not renders): blur (R33) + DR + noise
    (R31) codes bit-exact against the oracle for random extents incl. 0, negative, long and
    beyond the +-64 clamp; fp16 and fp32 depth pass-through."""
    rng = np.random.default_rng(21)
    B, C, H, W = 3, 2, 45, 70
    for trial in range(4):
        rgb = rng.uniform(-0.05, 1.05, (B, C, 3, H, W)).astype(np.float32)
        depth = rng.uniform(0.1, 9.0, (B, C, H, W)).astype(np.float32)
        blur = rng.integers(-12, 13, (B, C, 2)).astype(np.int32)
        blur[0, 0] = (0, 0)
        if trial == 3:
            blur[1, 1] = (70, -3)   # clamped to (64, -3)
        dr = _dr(rng, B, C, noise=trial % 2 == 1)
        seed, step, off = int(rng.integers(0, 2 ** 32)), trial, int(rng.integers(0, 100))
        q, d = _encode(rgb, blur, dr, depth, seed, step, off, f16=trial != 2)
        bl = np.clip(blur.reshape(B * C, 2), -64, 64)
        ref, ref_d = obs_oracle.epilogue(obs_oracle.motion_blur(rgb.reshape(B * C, 3, H, W), bl), depth.reshape(B * C, H, W),
                                         dr.reshape(B * C, 4), seed, step, off * C)
        np.testing.assert_array_equal(q.reshape(B * C, 3, H, W), ref)
        if trial != 2:
            np.testing.assert_array_equal(d.reshape(B * C, H, W).view(np.uint16), ref_d.view(np.uint16))
        else:
            np.testing.assert_array_equal(d, depth)


def test_obs_encode_without_blur_equals_fused_epilogue():
    """Rendering fp32 then encoding without blur gives exactly the codes of the fused epilogue
    (gsb_render_obs): both apply the same R31 op chain to the same composite."""
    cfg = synth.CONFIGS["T5"]
    sc = synth.make_scene(cfg)
    b = synth.make_batch(cfg, step=1)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H)
    rng = np.random.default_rng(5)
    dr = _dr(rng, B, C)
    q_fused, d_fused = _obs_render(g, b, W, H, dr, 123, 9, env_offset=4)
    out = gu.gpu_render(sc, b, W, H, gscene=g)
    q, d = _encode(out["rgb"], None, dr, out["depth"], 123, 9, 4)
    np.testing.assert_array_equal(q, q_fused)
    np.testing.assert_array_equal(d.view(np.uint16), d_fused.view(np.uint16))


def test_obs_blur_of_rendered_frames_within_one_code():
    """Render + blur + encode against oracle render + blur + encode on T1 frames: each side
    decides the code from its own blurred composite, so codes agree within 1 wherever every
    tap's pixel is outside the R28 mask, and exactly on >= 99 % of them."""
    cfg = synth.CONFIGS["T1"]
    sc = synth.make_scene(cfg)
    b = synth.make_batch(cfg, step=0)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    out = gu.gpu_render(sc, b, W, H)
    blur = np.array([[(5, 2), (-3, 0)], [(0, 7), (4, -4)], [(9, 1), (0, 0)]], np.int32)[:B, :C]
    q, _ = _encode(out["rgb"], blur)
    n_ok = n_exact = 0
    for e in range(B):
        for c in range(C):
            ref = oracle.render_frame(sc, b.poses[e], b.intrinsics[e, c], b.w2c[e, c], oracle.RenderParams(W, H))
            ref_rgb = ref.rgb.transpose(2, 0, 1)[None]
            rq, _ = obs_oracle.epilogue(obs_oracle.motion_blur(ref_rgb, blur[e, c][None]), None, None)
            # pixels all of whose taps are unmasked
            taps = obs_oracle.blur_taps(*blur[e, c])
            clean = np.ones((H, W), bool)
            ys, xs = np.arange(H)[:, None], np.arange(W)[None, :]
            for ox, oy in taps:
                clean &= ~ref.masked[np.clip(ys + oy, 0, H - 1), np.clip(xs + ox, 0, W - 1)]
            dq = np.abs(q[e, c].astype(int) - rq[0].astype(int)).max(axis=0)
            assert dq[clean].max() <= 1
            n_ok += int(clean.sum())
            n_exact += int((dq[clean] == 0).sum())
    assert n_exact >= 0.99 * n_ok
