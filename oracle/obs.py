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
With noise_std = 0 the noise term is skipped (it would add +0).  Motion blur needs a pixel
neighbourhood and is not part of this epilogue.
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
