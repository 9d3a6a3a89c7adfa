"""Integer-path (binning) oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Given projected values ROUNDED TO fp32 (u, v, Sigma2D_xx, Sigma2D_yy, kappa, zbits, valid),
compute every Gaussian's tile rectangle with the exact fp32 formula of reading R9 and
build, per (frame, tile), the list of ids sorted by (zbits, id) (reading R10; north_star
"deterministic tie-break on Gaussian id").  The GPU's gsb_debug_bin_sort must reproduce
these lists bit-exactly.

R9: rx = sqrt_rn(kappa*Sxx); xl = (u - rx) - 0.5f; xh = (u + rx) - 0.5f;
px_lo = max(ceil(xl), 0); px_hi = min(floor(xh), W-1) (clamped in float); non-finite
or px_lo > px_hi => culled; same for y; tiles [px_lo>>4, px_hi>>4]; tile id = ty*ceil(W/16)+tx.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def rects_f32(u, v, sxx, syy, kappa, valid, width, height):
    """Per-Gaussian (tx0, tx1, ty0, ty1, ok) by reading R9, all binary32 (numpy float32
    ops are IEEE round-to-nearest; np.sqrt on float32 is correctly rounded)."""
    f = np.float32
    u, v = np.asarray(u, f), np.asarray(v, f)
    sxx, syy, kappa = np.asarray(sxx, f), np.asarray(syy, f), np.asarray(kappa, f)
    with np.errstate(all="ignore"):
        rx = np.sqrt(kappa * sxx)
        ry = np.sqrt(kappa * syy)
        xl = (u - rx) - f(0.5)
        xh = (u + rx) - f(0.5)
        yl = (v - ry) - f(0.5)
        yh = (v + ry) - f(0.5)
        fin = np.isfinite(xl) & np.isfinite(xh) & np.isfinite(yl) & np.isfinite(yh)
        pxl = np.maximum(np.ceil(xl), f(0.0))
        pxh = np.minimum(np.floor(xh), f(width - 1))
        pyl = np.maximum(np.ceil(yl), f(0.0))
        pyh = np.minimum(np.floor(yh), f(height - 1))
    ok = np.asarray(valid, bool) & fin & (pxl <= pxh) & (pyl <= pyh)
    big = np.float32(2 ** 30)
    pxl, pxh = np.clip(np.where(ok, pxl, 0), -big, big), np.clip(np.where(ok, pxh, 0), -big, big)
    pyl, pyh = np.clip(np.where(ok, pyl, 0), -big, big), np.clip(np.where(ok, pyh, 0), -big, big)
    pxl, pxh, pyl, pyh = (a.astype(np.int64) for a in (pxl, pxh, pyl, pyh))
    return pxl >> 4, pxh >> 4, pyl >> 4, pyh >> 4, ok


def bin_frame(u, v, sxx, syy, kappa, zbits, valid, width, height):
    """One frame: returns (offsets [T_t+1] int64, ids [K] uint32)."""
    tw = (width + TILE - 1) // TILE
    th = (height + TILE - 1) // TILE
    T = tw * th
    tx0, tx1, ty0, ty1, ok = rects_f32(u, v, sxx, syy, kappa, valid, width, height)
    zbits = np.asarray(zbits, np.uint32)
    tiles, ids = [], []
    for i in np.nonzero(ok)[0]:
        for ty in range(ty0[i], ty1[i] + 1):
            for tx in range(tx0[i], tx1[i] + 1):
                tiles.append(ty * tw + tx)
                ids.append(i)
    tiles = np.asarray(tiles, np.int64)
    ids = np.asarray(ids, np.int64)
    if ids.size:
        order = np.lexsort((ids, zbits[ids], tiles))     # tile, then (zbits, id)
        tiles, ids = tiles[order], ids[order]
    counts = np.bincount(tiles, minlength=T) if tiles.size else np.zeros(T, np.int64)
    offsets = np.zeros(T + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    return offsets, ids.astype(np.uint32)


def bin_frames(u, v, sxx, syy, kappa, zbits, valid, width, height):
    """[F,N] inputs -> (offsets [F,T_t+1] absolute into ids, ids [sum K])."""
    F = u.shape[0]
    offs, all_ids, base = [], [], 0
    for f in range(F):
        o, ids = bin_frame(u[f], v[f], sxx[f], syy[f], kappa[f], zbits[f], valid[f], width, height)
        offs.append(o + base)
        all_ids.append(ids)
        base += ids.size
    return np.stack(offs), (np.concatenate(all_ids) if all_ids else np.zeros(0, np.uint32))
