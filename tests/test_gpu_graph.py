"""GSB_FLAG_FIXED_PLAN: a render whose launch sequence depends only on the call's shapes (no host
synchronisation, no data-dependent launch choice), so it can be captured in a CUDA graph and
replayed with new poses in place (the per-step S_t transfer of Alg. 1, then one replay).
Outputs must be bit-identical to the regular render; a chunk beyond the key capacity raises the
overflow flag instead of writing out of bounds."""
import numpy as np
import pytest
import torch

import paper_2604_25459_b200 as gsb
import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def _bufs(B, C, H, W):
    return (torch.full((B, C, 3, H, W), float("nan"), device="cuda"),
            torch.full((B, C, H, W), float("nan"), device="cuda"),
            torch.full((B, C, H, W), -7, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("name,chunk", [("T1", 0), ("T2", 0), ("T6", 0), ("T2", 1), ("C1", 0)])
def test_fixed_plan_bit_identical_to_regular(name, chunk):
    cfg = synth.CONFIGS[name]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    ref = gu.gpu_render(sc, b, W, H, chunk_frames=chunk)
    g = ref["scene"]
    rgb, dep, nev = _bufs(B, C, H, W)
    g.render(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c), gsb.RenderParams(W, H, fixed_plan=True),
             rgb, dep, None, nev)
    torch.cuda.synchronize()
    assert not g.overflow()
    assert np.array_equal(rgb.cpu().numpy(), ref["rgb"])
    assert np.array_equal(dep.cpu().numpy(), ref["depth"])
    assert np.array_equal(nev.cpu().numpy(), ref["n_eval"])


def test_graph_capture_and_replay_with_new_poses():
    """Capture one fixed-plan render in a CUDA graph, then for three physics steps copy the new
    poses into the captured input tensor and replay: every replay equals a regular render of
    that step, bit for bit."""
    cfg = synth.CONFIGS["T1"]
    sc = synth.make_scene(cfg)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    b0 = synth.make_batch(cfg, step=0)
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H)
    poses = gu.to_dev(b0.poses)
    intr, w2c = gu.to_dev(b0.intrinsics), gu.to_dev(b0.w2c)
    rgb, dep, nev = _bufs(B, C, H, W)
    prm = gsb.RenderParams(W, H, fixed_plan=True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):   # warm-up (kernel attributes, grids) outside the capture
        g.render(poses, intr, w2c, prm, rgb, dep, None, nev)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        g.render(poses, intr, w2c, prm, rgb, dep, None, nev)
    for step in (1, 5, 9):
        bs = synth.make_batch(cfg, step=step)
        poses.copy_(gu.to_dev(bs.poses))
        graph.replay()
        torch.cuda.synchronize()
        ref = gu.gpu_render(sc, bs, W, H)
        assert np.array_equal(rgb.cpu().numpy(), ref["rgb"]), step
        assert np.array_equal(dep.cpu().numpy(), ref["depth"]), step
        assert np.array_equal(nev.cpu().numpy(), ref["n_eval"]), step
    assert not g.overflow()


def test_fixed_plan_overflow_flag_instead_of_out_of_bounds():
    cfg = synth.CONFIGS["T2"]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    B, C, H, W = cfg.n_envs, cfg.n_cams, cfg.height, cfg.width
    g = gsb.Scene.from_synth(sc)
    g.reserve(B, C, W, H, 0, 1000)    # far below the frames' keys
    rgb, dep, nev = _bufs(B, C, H, W)
    g.render(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c), gsb.RenderParams(W, H, fixed_plan=True),
             rgb, dep, None, nev)
    torch.cuda.synchronize()
    assert g.overflow()
    assert not g.overflow()            # reset by the read
    with pytest.raises(gsb.GsbError):  # the regular render reports the capacity error itself
        g.render(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c), gsb.RenderParams(W, H), rgb)
    with pytest.raises(gsb.GsbError):  # STATS needs the host readback the fixed plan avoids
        g.render(gu.to_dev(b.poses), gu.to_dev(b.intrinsics), gu.to_dev(b.w2c),
                 gsb.RenderParams(W, H, fixed_plan=True, stats=True), rgb)
