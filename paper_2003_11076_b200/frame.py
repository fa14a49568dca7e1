"""LightFieldFrame (frame.py:10-52) with a device-resident mirror.

A frame's K views and priors are uploaded once and its descriptors are
computed on the GPU once; every solver / refocus call on the same frame
reuses the device copies (the reference caches descriptors the same way,
frame.py:46-52).
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
        self.images = upload(images if isinstance(images, t.Tensor) else np.stack(images), np.uint8)
        self.priors = upload(priors if isinstance(priors, t.Tensor) else np.stack(priors),
                             np.float32)
        if self.images.dim() == 3:
            self.images = self.images.unsqueeze(-1).expand(-1, -1, -1, 3).contiguous()
        self.K, self.H, self.W = (int(x) for x in self.images.shape[:3])
        self.desc, _, _ = _run(self.images)


def device_frame(frame):
    """Device mirror of any LightFieldFrame-like object (cached on our own frames)."""
    cached = getattr(frame, "_dev", None)
    if cached is not None:
        return cached
    d = DeviceFrame(frame.images, frame.priors)
    if isinstance(frame, LightFieldFrame):
        frame._dev = d
    return d
