"""Reading R31 — observation epilogue (§8(f) row 4): image domain randomisation and uint8 /
fp16 encoding of a rendered frame — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names the image DR but gives no formulas: "variations in brightness, contrast and
exposure" and "injection of image noise and motion blur".  Reading R31 fixes,
per frame f with parameters (gain, contrast, brightness, noise_std) and per pixel/channel value c
(the fp32 composite C + T bg), every op in binary32 round-to-nearest, in this order:

    e = c * gain                      exposure as a linear gain (2^EV)
    k = (e - 0.5) * contrast + 0.5    contrast about mid-grey (a fixed pivot: per-pixel, no image mean)
    b = k + brightness                additive brightness
    v = b + (z * s3) * noise_std      z: Irwin-Hall(4) integer noise, s3 = sqrt(3) / 2^22 (unit variance)
    q = rint(clamp(v, 0, 1) * 255)    round half to even; NaN -> 0
    depth16 = float16(depth_f32)      round to nearest even

The noise is counter-based so that both sides (and any sharding) draw the same numbers: with
mix32 the 'lowbias32' integer hash (x ^= x>>16; x *= 0x7feb352d; x ^= x>>15; x *= 0x846ca68b;
x ^= x>>16), the global frame index g = env_offset * C + f, and idx = ((g H + y) W + x) 3 + ch,
    base = mix32(lo32(idx) ^ mix32(hi32(idx) ^ mix32(seed ^ mix32(step))))
    u_j  = mix32(base + j * 0x9E3779B9) >> 10      (j = 0..3, 22-bit uniforms)
    z    = float(u_0 + u_1 + u_2 + u_3) - 2^23     (exact in binary32).
With noise_std = 0 the noise term is skipped (it would add +0).

Reading R33 — motion blur ("injection of image noise and motion blur"; no formula): a
per-frame linear box blur of the composite c along an integer pixel motion (bx, by), applied
BEFORE R31 (blur happens during the exposure, noise and encoding after it); depth is not
blurred.  With L = max(|bx|, |by|) + 1 taps (L = 1: identity), tap k = 0..L-1 sits at
    o_k(b) = floor((2 k b + (L-1)) / (2 (L-1))) - floor(b / 2)      (integer arithmetic)
i.e. k b / (L-1) rounded half up, shifted to centre the segment; samples clamp to the image
edge; in binary32 RN:  acc = ((c_0 + c_1) + c_2) + ...  in tap order, blurred = acc / L.
"""
from __future__ import annotations

import numpy as np

S3 = np.float32(np.sqrt(3.0)) / np.float32(2.0 ** 22)   # exact: power-of-two divisor
_M1, _M2, _GOLD = np.uint32(0x7FEB352D), np.uint32(0x846CA68B), np.uint32(0x9E3779B9)


def mix32(x):
    """lowbias32 integer hash on uint32 arrays (wrap-around arithmetic)."""
    x = np.asarray(x, np.uint32).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= _M1
        x ^= x >> np.uint32(15)
        x *= _M2
        x ^= x >> np.uint32(16)
    return x


def noise_z(seed: int, step: int, gframe, y, x, ch, H: int, W: int) -> np.ndarray:
    """Irwin-Hall(4) integer noise z (float32) at the given global frame / pixel / channel."""
    idx = ((np.asarray(gframe, np.uint64) * np.uint64(H) + np.asarray(y, np.uint64)) * np.uint64(W)
           + np.asarray(x, np.uint64)) * np.uint64(3) + np.asarray(ch, np.uint64)
    lo = (idx & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (idx >> np.uint64(32)).astype(np.uint32)
    k = mix32(np.uint32(seed) ^ mix32(np.uint32(step)))
    base = mix32(lo ^ mix32(hi ^ k))
    s = np.zeros(base.shape, np.uint32)
    with np.errstate(over="ignore"):
        for j in range(4):
            s += mix32(base + np.uint32(j) * _GOLD) >> np.uint32(10)
    return s.astype(np.float32) - np.float32(2.0 ** 23)


def epilogue(rgb, depth, dr, seed: int = 0, step: int = 0, frame_offset: int = 0):
    """R31 on frames: rgb [F,3,H,W] and depth [F,H,W] (any float type; rounded to binary32 first),
    dr [F,4] (gain, contrast, brightness, noise_std) or None.  Returns (uint8 [F,3,H,W],
    float16 [F,H,W] or None)."""
    c = np.asarray(rgb, np.float32)
    F, _, H, W = c.shape
    if dr is None:
        dr = np.tile(np.float32([1.0, 1.0, 0.0, 0.0]), (F, 1))
    dr = np.asarray(dr, np.float32).reshape(F, 4)
    g, k, b, n = (dr[:, i][:, None, None, None] for i in range(4))
    e = c * g
    v = (e - np.float32(0.5)) * k + np.float32(0.5)
    v = v + b
    if (dr[:, 3] != 0).any():
        f, ch, y, x = np.meshgrid(np.arange(F), np.arange(3), np.arange(H), np.arange(W), indexing="ij")
        z = noise_z(seed, step, f + frame_offset, y, x, ch, H, W)
        add = (z * S3) * n
        v = np.where(n != 0, v + add, v)
    v = np.where(np.isnan(v), np.float32(0), v)
    v = np.clip(v, np.float32(0), np.float32(1))
    q = np.rint(v * np.float32(255)).astype(np.uint8)
    d16 = None
    if depth is not None:
        with np.errstate(over="ignore"):   # beyond 65504 rounds to inf, as IEEE requires
            d16 = np.asarray(depth, np.float32).astype(np.float16)
    return q, d16


def blur_taps(bx: int, by: int):
    """Reading R33 tap offsets [(ox_k, oy_k)] of one frame (integer arithmetic)."""
    L = max(abs(int(bx)), abs(int(by))) + 1
    if L == 1:
        return [(0, 0)]
    d = 2 * (L - 1)
    return [((2 * k * bx + (L - 1)) // d - bx // 2, (2 * k * by + (L - 1)) // d - by // 2) for k in range(L)]


def motion_blur(rgb, blur):
    """Reading R33 on frames rgb [F,3,H,W] (rounded to binary32) with blur [F,2] int (bx, by):
    binary32 sequential tap sum over edge-clamped samples, then one division by L."""
    c = np.asarray(rgb, np.float32)
    F, _, H, W = c.shape
    out = np.empty_like(c)
    ys, xs = np.arange(H)[:, None], np.arange(W)[None, :]
    for f in range(F):
        taps = blur_taps(int(blur[f][0]), int(blur[f][1]))
        acc = np.zeros((3, H, W), np.float32)
        for ox, oy in taps:
            yy = np.clip(ys + oy, 0, H - 1)
            xx = np.clip(xs + ox, 0, W - 1)
            acc = acc + c[f][:, yy, xx]
        out[f] = acc / np.float32(len(taps))
    return out
