"""16-byte ring descriptors (features.py), computed by the `k_descriptors` kernel.

gray = rint(0.299 R + 0.587 G + 0.114 B) (fp64), biased Sobel
clip(rint(128 + g/4)), entry 2i = gx and 2i+1 = gy at SAMPLE_OFFSETS[i],
128 off-image; the valid interior has margin 3 (features.py:19-104).
"""

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload
from .sampling import bilinear, flatten_channels

DESCRIPTOR_LENGTH = 16
DESCRIPTOR_MARGIN = 3
SAMPLE_OFFSETS = ((0, -2), (1, -1), (2, 0), (1, 1), (0, 2), (-1, 1), (-2, 0), (-1, -1))
GRAY_WEIGHTS = (0.299, 0.587, 0.114)


def _run(images, want_gray=False, want_sobel=False):
    """images: (K, H, W, C) uint8 host or device -> device desc (+ gray, sobel)."""
    t = require_cuda()
    x = upload(images) if not hasattr(images, "is_cuda") or not images.is_cuda else images
    if x.dim() == 3:
        x = x.unsqueeze(-1)
    k, h, w, c = x.shape
    desc = empty((k, h, w, DESCRIPTOR_LENGTH), t.uint8)
    gray = empty((k, h, w), t.uint8) if want_gray else None
    sob = empty((k, h, w, 2), t.uint8) if want_sobel else None
    N.check(N.lib().st_descriptors(N.ptr(x), k, h, w, c, N.ptr(desc), N.ptr(gray), N.ptr(sob),
                                   N.stream_handle()))
    return desc, gray, sob


def rgb_to_gray(image):
    img = np.asarray(image)
    if img.ndim == 2:
        return img.astype(np.uint8, copy=False)
    _, gray, _ = _run(img[None], want_gray=True)
    return download(gray)[0]


def sobel_responses(gray):
    g = np.asarray(gray)
    if g.ndim != 2:
        raise ValueError("sobel_responses wants a grayscale image")
    _, _, sob = _run(g.astype(np.uint8)[None], want_sobel=True)
    s = download(sob)[0]
    return s[..., 0].copy(), s[..., 1].copy()


@dataclass
class DescriptorMap:
    """Dense descriptors of one view: data (h, w, 16) uint8, valid (h, w) bool."""

    data: np.ndarray
    valid: np.ndarray

    @property
    def shape(self):
        return self.data.shape[:2]

    def flat32(self):
        cached = getattr(self, "_flat32", None)
        if cached is None:
            cached = flatten_channels(self.data)
            self._flat32 = cached
        return cached


def _valid_mask(h, w):
    m = DESCRIPTOR_MARGIN
    valid = np.zeros((h, w), dtype=bool)
    valid[m:h - m, m:w - m] = True
    return valid


def compute_descriptors(gray):
    g = np.asarray(gray)
    h, w = g.shape[:2]
    if h < 2 * DESCRIPTOR_MARGIN + 1 or w < 2 * DESCRIPTOR_MARGIN + 1:
        raise ValueError(f"image too small for descriptors (needs at least "
                         f"{2 * DESCRIPTOR_MARGIN + 1} pixels per side)")
    desc, _, _ = _run(g[None])
    return DescriptorMap(data=download(desc)[0], valid=_valid_mask(h, w))


def sample_descriptors(dmap, u, v):
    h, w = dmap.shape
    flat, fh, fw = dmap.flat32()
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    m = DESCRIPTOR_MARGIN
    valid = (u >= m) & (u <= w - m - 1) & (v >= m) & (v <= h - m - 1)
    return bilinear(flat, fh, fw, u, v), valid


# The two helpers below belong to the support-harvest stage (prior.py), which
# is upstream of the accelerated path; they stay plain numpy.
def descriptor_distance(a, b):
    return np.abs(np.asarray(a, np.int32) - np.asarray(b, np.int32)).sum(axis=-1)


def texture_energy(dmap):
    return np.abs(dmap.data.astype(np.int32) - 128).sum(axis=2)
