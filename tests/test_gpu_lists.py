"""Integer parity of the PRODUCTION binning + tile sort (SURVEY §8(c) c.3 "per-(f, t) counts,
offsets and id lists given the oracle's fp32 projected values"; readings R9, R10).

gsb_debug_tile_lists runs K2b emission and the sort that really feeds compositing in gsb_render
— K4a's warp-per-list counting sort (<= 512 keys), its CTA-per-list index counting sort (<= 4096;
also the legacy CTA counting sort of the LiDAR path), the HBM radix beyond, and the fused K4's
in-CTA sorts (count and packed radix) — with keys carrying the
record slot (the render's default: equal-depth runs re-ordered by creation id) or the id.  The
inputs are the oracle's projections rounded to fp32, laid out in a random internal (slot)
order, so every depth tie must be broken through the slot -> id map.  Every (frame, tile) list
must equal oracle/binning.py's bit for bit; at full size (C3, C4) that is every tile of frames
{0, B/2, B-1} (all cameras)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_25459_b200 as gsb
import synth
from oracle import binning
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu

VARIANTS = {1: "K4a warp + long CTA", 2: "K4a packed", 3: "fused K4 small", 4: "fused K4 packed",
            5: "K4a CTA count"}


def _oracle_fp32(sc, b, cfg, frames):
    """The oracle's projected values rounded to fp32 ([F, N] by creation id) for frames (e, c)."""
    F, N = len(frames), sc.n
    arr = {k: np.zeros((F, N), np.float32) for k in ("u", "v", "sxx", "syy", "kappa")}
    zb = np.zeros((F, N), np.uint32)
    va = np.zeros((F, N), np.uint8)
    prm = oracle.RenderParams(cfg.width, cfg.height)
    for f, (e, c) in enumerate(frames):
        proj, z, v = oracle.project(sc, b.poses[e], b.intrinsics[e, c], b.w2c[e, c], prm)
        arr["u"][f], arr["v"][f] = proj[:, oracle.F_U], proj[:, oracle.F_V]
        arr["sxx"][f], arr["syy"][f] = proj[:, oracle.F_SXX], proj[:, oracle.F_SYY]
        arr["kappa"][f] = proj[:, oracle.F_KAPPA]
        zb[f], va[f] = z, v
    return arr, zb, va


def _run(arr, zb, va, W, H, perm, variant, key_mode, cap):
    """Inputs permuted into slot order (slot j holds Gaussian perm[j]); returns GPU lists."""
    d = {k: gu.to_dev(np.ascontiguousarray(x[:, perm])) for k, x in arr.items()}
    return gsb.debug_tile_lists(d["u"], d["v"], d["sxx"], d["syy"], d["kappa"],
                                gu.to_dev(np.ascontiguousarray(zb[:, perm]).view(np.int32)),
                                gu.to_dev(np.ascontiguousarray(va[:, perm])),
                                gu.to_dev(perm.astype(np.int32)), W, H, cap=cap, variant=variant, key_mode=key_mode)


def _check(arr, zb, va, W, H, variants, key_modes=(0, 1), seed=0, expect_auto=None):
    offs_ref, ids_ref = binning.bin_frames(arr["u"], arr["v"], arr["sxx"], arr["syy"], arr["kappa"], zb, va, W, H)
    N = zb.shape[1]
    perm = np.random.default_rng(seed).permutation(N)
    for variant in variants:
        for km in key_modes:
            offs, ids, ran = _run(arr, zb, va, W, H, perm, variant, km, cap=int(ids_ref.size) + 16)
            torch.cuda.synchronize()
            if variant == 0 and expect_auto is not None:
                assert ran == expect_auto, (ran, expect_auto)
            assert np.array_equal(offs.cpu().numpy(), offs_ref), (variant, km)
            got = ids.cpu().numpy().view(np.uint32)
            bad = np.nonzero(got != ids_ref)[0]
            assert bad.size == 0, (VARIANTS.get(ran), km, bad.size, bad[:5])
    return offs_ref


@pytest.mark.parametrize("name", ["C1", "T1", "T2", "T4", "T6"])
def test_production_tile_lists_small_configs(name):
    """All frames of the parity configs through every sort variant and both key kinds."""
    cfg = synth.CONFIGS[name]
    sc, b = synth.make_scene(cfg), synth.make_batch(cfg)
    frames = [(e, c) for e in range(cfg.n_envs) for c in range(cfg.n_cams)]
    arr, zb, va = _oracle_fp32(sc, b, cfg, frames)
    _check(arr, zb, va, cfg.width, cfg.height, variants=(0, 1, 2, 3, 4, 5), seed=len(name))
    # K4b block masks ride in the keys' low bits through K4a's warp / index / HBM sorts
    _check(arr, zb, va, cfg.width, cfg.height, variants=(1, 2), key_modes=(2,), seed=len(name))


@pytest.mark.parametrize("size", [32, 64, 160])
def test_production_tile_lists_ties_and_oversize_lists(size):
    """32x32: > 4096 keys in one tile (the HBM radix of every variant); 64x64: ~500-1000-key lists
    (K4a's index counting sort); 160x160: ~100-300-key lists (K4a's warp path) — all with many
    exactly equal depths (equal-depth runs longer than 32, the re-keyed fallback, and short runs
    fixed in place)."""
    rng = np.random.default_rng(3)
    F, N, W, H = 2, 9000, size, size
    arr = {"u": rng.uniform(2, W - 2, (F, N)), "v": rng.uniform(2, H - 2, (F, N)), "sxx": rng.uniform(0.5, 3, (F, N)),
           "syy": rng.uniform(0.5, 3, (F, N)), "kappa": rng.uniform(0.5, 8, (F, N))}
    arr = {k: x.astype(np.float32) for k, x in arr.items()}
    if size == 32:   # one tile with > 4096 keys
        arr["u"][:, ::4] = rng.uniform(4, 12, (F, (N + 3) // 4))
        arr["v"][:, ::4] = rng.uniform(4, 12, (F, (N + 3) // 4))
    z = rng.choice(np.float32([1.0, 1.5, 2.0, 2.25]), (F, N)).astype(np.float32)
    z[:, ::3] = rng.uniform(0.5, 5, (F, (N + 2) // 3)).astype(np.float32)
    z[:, 1::7] = np.float32(3.0) + np.float32(2 ** -20) * rng.integers(0, 3, (F, len(range(1, N, 7))))
    zb = z.view(np.uint32)
    va = (rng.random((F, N)) < 0.95).astype(np.uint8)
    offs = _check(arr, zb, va, W, H, variants=(1, 2, 3, 4, 5), seed=5)
    _check(arr, zb, va, W, H, variants=(1, 2), key_modes=(2,), seed=5)   # with block masks
    L = np.diff(offs, axis=1)
    if size == 32:
        assert L.max() > 4096
    elif size == 64:
        assert L.min() > 512 and L.max() <= 4096
    else:
        assert L.max() <= 1024 and L.mean() > 100


@pytest.mark.slow
@pytest.mark.parametrize("name,auto", [("C3", 1), ("C4", 2)])
def test_production_tile_lists_full_size(name, auto):
    """Every tile of frames {0, B/2, B-1} (all cameras) at full size: the variant gsb_render picks
    for the config (C3: K4a warp sort, a CTA with the HBM radix for each > 1024-key list; C4: K4a
    packed) and the other K4a variants, with slot keys and id keys."""
    cfg = synth.CONFIGS[name]
    sc = synth.make_scene(cfg)
    envs = [0, cfg.n_envs // 2, cfg.n_envs - 1]
    b = synth.make_batch(cfg, envs)
    frames = [(k, c) for k in range(len(envs)) for c in range(cfg.n_cams)]
    arr, zb, va = _oracle_fp32(sc, b, cfg, frames)
    offs = _check(arr, zb, va, cfg.width, cfg.height, variants=(0, 1, 2, 5), seed=11, expect_auto=auto)
    L = np.diff(offs, axis=1)
    print(name, "keys", int(L.sum()), "longest list", int(L.max()), "lists > 1024:", int((L > 1024).sum()))
