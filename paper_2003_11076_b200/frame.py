"""LightFieldFrame (frame.py:10-52) with a device-resident mirror.

A frame's descriptors are computed on the GPU once and cached, exactly as the
reference caches them (frame.py:46-52, computed from the images at first
use).  The arrays the reference re-reads on every call are re-uploaded on
every call: the priors at solver construction (solver.py:182) and the
images in synthesize (refocus.py:24-49), so a caller that edits a frame's
arrays in place sees the same results as with the reference.
"""

from dataclasses import dataclass, field

import numpy as np

from .features import DescriptorMap, _run, _valid_mask
from .device import download, require_cuda, upload


@dataclass
class LightFieldFrame:
    images: list
    priors: list
    _descriptors: list = field(init=False, repr=False, default=None)
    _dev: object = field(init=False, repr=False, default=None)

    def __post_init__(self):
        if len(self.images) != len(self.priors):
            raise ValueError("one prior map per view is required")
        if len(self.images) < 2:
            raise ValueError("a light-field frame needs at least two views")
        base = self.images[0].shape[:2]
        for i, (img, pri) in enumerate(zip(self.images, self.priors)):
            if img.shape[:2] != base or pri.shape != base:
                raise ValueError(f"view {i}: shape mismatch with view 0")
            if pri.min() < 0.0 or pri.max() > 1.0:
                raise ValueError(f"view {i}: prior values outside [0, 1]")

    @property
    def num_views(self):
        return len(self.images)

    @property
    def shape(self):
        return self.images[0].shape[:2]

    def gray(self, k):
        from .features import rgb_to_gray
        return rgb_to_gray(self.images[k])

    def descriptors(self, k):
        if self._descriptors is None:
            self._descriptors = [None] * self.num_views
        if self._descriptors[k] is None:
            d = device_frame(self)
            h, w = self.shape
            self._descriptors[k] = DescriptorMap(data=download(d.desc[k]), valid=_valid_mask(h, w))
        return self._descriptors[k]


class DeviceFrame:
    """(K,H,W,3) u8 images, (K,H,W) f32 priors, (K,H,W,16) u8 descriptors on the GPU."""

    def __init__(self, images, priors):
        t = require_cuda()
        from .device import upload_views
        self.images = (upload(images, np.uint8) if isinstance(images, t.Tensor)
                       else upload_views(images, np.uint8))
        self.priors = (upload(priors, np.float32) if isinstance(priors, t.Tensor)
                       else upload_views(priors, np.float32))
        if self.images.dim() == 3:
            self.images = self.images.unsqueeze(-1).expand(-1, -1, -1, 3).contiguous()
        self.K, self.H, self.W = (int(x) for x in self.images.shape[:3])
        self.desc, _, _ = _run(self.images)

    def refresh(self, frame, what):
        """Re-upload `what` ("images" / "priors") from the host frame."""
        t = torch_of()
        for name in what:
            src = getattr(frame, name)
            dst = getattr(self, name)
            if isinstance(src, t.Tensor):
                dst.copy_(src.reshape(dst.shape))
                continue
            dt = np.uint8 if name == "images" else np.float32
            for k, a in enumerate(src):
                a = np.ascontiguousarray(a, dtype=dt)
                if name == "images" and a.ndim == 2:
                    a = np.repeat(a[:, :, None], 3, axis=2)
                dst[k].copy_(t.from_numpy(a))


def torch_of():
    from .device import torch
    return torch()


def device_frame(frame, refresh=()):
    """Device mirror of any LightFieldFrame-like object (cached on our own
    frames; `refresh` names the arrays to re-upload into a cached mirror)."""
    cached = getattr(frame, "_dev", None)
    if cached is not None:
        if refresh:
            cached.refresh(frame, refresh)
        return cached
    d = DeviceFrame(frame.images, frame.priors)
    if isinstance(frame, LightFieldFrame):
        frame._dev = d
    return d
