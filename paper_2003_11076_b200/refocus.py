"""See-through composition from the static rays (refocus.py), on the GPU.

`synthesize` = `k_refocus` (Eq. 2 fp64 average of static in-bounds rays,
provenance 255/0/128, n_rays) followed by `k_median_small` (clipped-window
median rewriting every non-COPIED pixel) -- refocus.py:24-148.
"""

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload
from .frame import device_frame
from .solver import STATUS_VALID  # noqa: F401  (re-export parity with the reference)

PROV_FALLBACK = 0
PROV_COPIED = 128
PROV_REFOCUSED = 255


def _rig_of(frame, rig):
    h, w = frame.shape
    return N.make_rig(rig, w, h)


def _refocus_list(frame, rig, pix, d, static_bits, min_static_rays):
    t = require_cuda()
    dev = device_frame(frame, refresh=("images",))
    pix = np.asarray(pix, dtype=np.int64).ravel()
    n = pix.size
    rgb = empty((n, 3), t.uint8)
    cnt = empty((n,), t.int32)
    prov = empty((n,), t.uint8)
    tot = empty((n, 3), t.float64)
    if n:
        bits = np.asarray(static_bits, dtype=np.uint32).ravel().view(np.int32)
        N.invoke("st_refocus_pixels", dev.images, _rig_of(frame, rig), upload(pix),
                 upload(np.asarray(d, np.float64).ravel()), upload(bits), n,
                 int(min_static_rays), rgb, cnt, prov, tot)
    return download(rgb), download(cnt), download(prov), download(tot)


def gather_static_colors(frame, rig, pix, d, static_bits):
    """(color_sum (n, 3) f64, count (n,) int32) (refocus.py:24-49)."""
    _, cnt, _, tot = _refocus_list(frame, rig, pix, d, static_bits, 1 << 30)
    return tot, cnt


def refocus_pixel(frame, rig, u, v, d, static_bits, min_static_rays=2):
    """Single-pixel reference path: (rgb uint8[3], ray count, provenance)."""
    if not np.isscalar(static_bits):
        static_bits = sum(1 << k for k, b in enumerate(static_bits) if b)
    w = frame.shape[1]
    rgb, cnt, prov, _ = _refocus_list(frame, rig, [int(v) * w + int(u)], [float(d)],
                                      [static_bits], min_static_rays)
    return rgb[0].copy(), int(cnt[0]), int(prov[0])


def median_filter(image, radius):
    """Per-channel median over border-clipped windows, rint half-even (refocus.py:68-106)."""
    img = np.asarray(image)
    if radius <= 0:
        return img.copy()
    t = require_cuda()
    h, w = img.shape[:2]
    c = img.shape[2] if img.ndim == 3 else 1
    if img.dtype != np.uint8:
        raise ValueError("median_filter expects a uint8 image")
    src = upload(img.reshape(h, w, c))
    out = empty((h, w, c), t.uint8)
    N.check(N.lib().st_median(N.ptr(src), h, w, c, int(radius), N.ptr(out), N.stream_handle()))
    return download(out).reshape(img.shape)


def synthesize_device(frame, rig, values, status, static_bits, min_static_rays=2,
                      median_radius=1, copy_mask=None):
    """Device-tensor variant used by `reconstruct` (no host round trips)."""
    t = require_cuda()
    dev = device_frame(frame, refresh=("images",))
    h, w = frame.shape
    img = empty((h, w, 3), t.uint8)
    prov = empty((h, w), t.uint8)
    nr = empty((h, w), t.uint8)
    scratch = empty((h, w, 3), t.uint8) if median_radius > 0 else None
    cm = None
    if copy_mask is not None:
        cm = copy_mask if isinstance(copy_mask, t.Tensor) else upload(
            np.asarray(copy_mask, dtype=bool).astype(np.uint8))
    N.check(N.lib().st_synthesize(N.ptr(dev.images), _rig_of(frame, rig), N.ptr(values),
                                  N.ptr(status), N.ptr(static_bits), int(min_static_rays),
                                  int(median_radius), N.ptr(cm), N.ptr(img), N.ptr(prov),
                                  N.ptr(nr), N.ptr(scratch), N.stream_handle()))
    return img, prov, nr


def synthesize(frame, rig, disparity, seg, min_static_rays=2, median_radius=1, copy_mask=None):
    """Dense see-through composition (refocus.py:109-148)."""
    values = upload(np.asarray(disparity.values, dtype=np.float32))
    status = upload(np.asarray(disparity.status, dtype=np.uint8))
    bits = upload(np.asarray(seg.static_bits, dtype=np.uint32).view(np.int32))
    img, prov, nr = synthesize_device(frame, rig, values, status, bits, min_static_rays,
                                      median_radius, copy_mask)
    from .device import download_many
    img, prov, nr = download_many((img, prov, nr))
    return img, prov, nr
