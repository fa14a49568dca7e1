"""Bilinear sampling over flattened planes (sampling.py), on the GPU.

`bilinear` keeps the reference contract: (h*w, c) float32 plane, continuous
(u, v), non-finite coordinates map to 0, coordinates are clipped, result is
(n, c) float64 -- fp32 tap differences, fp64 lerp (sampling.py:21-55).
"""

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload


def flatten_channels(image):
    """(h, w) or (h, w, c) -> (float32 (h*w, c), h, w) (sampling.py:12-18)."""
    a = np.asarray(image)
    if a.ndim == 2:
        a = a[:, :, None]
    h, w, c = a.shape
    return np.ascontiguousarray(a.reshape(h * w, c), dtype=np.float32), h, w


def bilinear(flat, height, width, u, v):
    t = require_cuda()
    flat = np.asarray(flat, dtype=np.float32)
    if flat.ndim == 1:
        flat = flat[:, None]
    c = flat.shape[1]
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).ravel())
    n = u.size
    out = empty((n, c), t.float64)
    if n:
        g = upload(flat)
        du, dv = upload(u), upload(v)
        N.check(N.lib().st_bilinear(N.ptr(g), int(height), int(width), c, N.ptr(du), N.ptr(dv),
                                    n, N.ptr(out), N.stream_handle()))
    return download(out)
