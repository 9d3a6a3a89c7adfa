"""Pins of the reading-R33 motion blur oracle (oracle/obs.py; "image noise and motion
blur") against the textbook definition (a normalised line kernel convolved with edge
replication: scipy.ndimage.correlate, mode="nearest"), closed forms and invariants."""
import numpy as np
import pytest
from scipy import ndimage

from oracle import obs


@pytest.mark.parametrize("bx,by", [(0, 0), (4, 0), (0, -5), (3, 2), (-7, 3), (6, -6), (1, 0), (-2, -9)])
def test_taps_form_a_centred_digital_line(bx, by):
    """L = max(|bx|,|by|)+1 taps, consecutive taps are 8-connected neighbours, the segment spans
    exactly (bx, by), the dominant axis steps by one pixel per tap, and it is centred."""
    t = np.array(obs.blur_taps(bx, by))
    L = max(abs(bx), abs(by)) + 1
    assert len(t) == L
    if L > 1:
        st = np.diff(t, axis=0)
        assert np.abs(st).max() <= 1
        assert tuple(t[-1] - t[0]) == (bx, by)
        dom = 0 if abs(bx) >= abs(by) else 1
        assert (np.abs(st[:, dom]) == 1).all()
        # centred: the midpoint of the segment is within half a pixel of the origin
        assert np.abs((t[0] + t[-1]) / 2.0).max() <= 0.5


@pytest.mark.parametrize("bx,by", [(5, 0), (0, 3), (4, -2), (-6, 5)])
def test_blur_equals_normalised_line_kernel_correlation(bx, by):
    """R33 == scipy.ndimage.correlate with weight 1/L at each tap offset and edge replication
    (fp64 library reference; agreement to binary32 rounding)."""
    rng = np.random.default_rng(1)
    F, H, W = 1, 23, 31
    img = rng.uniform(0, 1, (F, 3, H, W)).astype(np.float32)
    got = obs.motion_blur(img, [(bx, by)])
    taps = obs.blur_taps(bx, by)
    r = max(max(abs(a), abs(b)) for a, b in taps)
    k = np.zeros((2 * r + 1, 2 * r + 1))
    for ox, oy in taps:
        k[r + oy, r + ox] += 1.0 / len(taps)
    for ch in range(3):
        ref = ndimage.correlate(img[0, ch].astype(np.float64), k, mode="nearest")
        np.testing.assert_allclose(got[0, ch], ref, atol=3e-7)


def test_blur_impulse_constant_and_identity():
    """An impulse far from the edges becomes L pixels of 1/L along the (mirrored) taps; a
    constant 0.5 image stays exactly 0.5; (0, 0) is the identity bit for bit."""
    H, W = 32, 40
    img = np.zeros((1, 3, H, W), np.float32)
    img[0, :, 16, 20] = 1.0
    out = obs.motion_blur(img, [(6, 0)])
    taps = obs.blur_taps(6, 0)
    row = out[0, 0, 16]
    hit = np.nonzero(row)[0]
    assert sorted(hit.tolist()) == sorted(20 - ox for ox, _ in taps)
    assert np.allclose(row[hit], np.float32(1.0) / np.float32(7))
    assert out[0, 0].sum() == pytest.approx(1.0, abs=1e-6)
    c = np.full((2, 3, H, W), 0.5, np.float32)
    assert (obs.motion_blur(c, [(9, -4), (3, 3)]) == np.float32(0.5)).all()
    rng = np.random.default_rng(2)
    x = rng.uniform(0, 1, (2, 3, H, W)).astype(np.float32)
    assert np.array_equal(obs.motion_blur(x, [(0, 0), (0, 0)]).view(np.uint32), x.view(np.uint32))


def test_blur_preserves_mass_in_the_interior():
    """Away from the edges a normalised kernel preserves the total (fp64 sum)."""
    rng = np.random.default_rng(3)
    H, W = 40, 40
    img = np.zeros((1, 3, H, W), np.float32)
    img[0, :, 10:30, 10:30] = rng.uniform(0, 1, (3, 20, 20))
    out = obs.motion_blur(img, [(5, 3)])
    assert out.astype(np.float64).sum() == pytest.approx(img.astype(np.float64).sum(), rel=1e-6)
