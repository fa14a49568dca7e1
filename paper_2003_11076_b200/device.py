"""Device-memory plumbing: torch CUDA tensors in, pinned host buffers out.

PyTorch is used only for device allocation, streams and pinned host memory;
every computation on the product path runs in the native CUDA library.
"""

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("seethrough_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    from . import _native
    _native.lib()
    return t


def dev():
    return torch().device("cuda", torch().cuda.current_device())


def upload(a, dtype=None):
    """numpy (or torch CPU) -> contiguous CUDA tensor on the current stream."""
    t = torch()
    if isinstance(a, t.Tensor):
        x = a
    else:
        arr = np.asarray(a)
        if dtype is not None and arr.dtype != dtype:
            arr = arr.astype(dtype)
        x = t.from_numpy(np.ascontiguousarray(arr))
    if x.device.type != "cuda":
        # pinned sources (see pinned_empty) copy asynchronously by DMA
        x = x.to(dev(), non_blocking=x.is_pinned())
    return x.contiguous()


def empty(shape, dtype):
    t = torch()
    return t.empty(shape, dtype=dtype, device=dev())


def pinned_empty(shape, np_dtype):
    """numpy array backed by page-locked memory (torch's caching host allocator)."""
    t = torch()
    tt = t.empty(shape, dtype=_TORCH_OF[np.dtype(np_dtype)], pin_memory=t.cuda.is_available())
    return tt.numpy()


def download(x, out=None):
    """CUDA tensor -> numpy, through pinned memory, synchronising the stream."""
    t = torch()
    if out is None:
        host = t.empty(tuple(x.shape), dtype=x.dtype, pin_memory=True)
    else:
        host = out
    host.copy_(x, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return host.numpy()


def upload_views(views, np_dtype):
    """A list of equally shaped host arrays -> one (K, ...) CUDA tensor, each
    view copied straight into its slice (no host-side np.stack)."""
    t = torch()
    first = np.asarray(views[0])
    out = t.empty((len(views),) + first.shape, dtype=_TORCH_OF[np.dtype(np_dtype)], device=dev())
    for k, v in enumerate(views):
        a = np.ascontiguousarray(v, dtype=np_dtype)
        out[k].copy_(t.from_numpy(a), non_blocking=False)
    return out


def download_many(xs):
    """Several CUDA tensors -> numpy arrays through ONE pinned block, one
    synchronisation (the arrays are views of distinct parts of the block)."""
    t = torch()
    sizes = [x.numel() * x.element_size() for x in xs]
    offs, total = [], 0
    for n in sizes:
        offs.append(total)
        total += (n + 255) & ~255
    block = t.empty((max(total, 1),), dtype=t.uint8, pin_memory=True)
    outs = []
    for x, o, n in zip(xs, offs, sizes):
        h = block[o:o + n].view(x.dtype).view(x.shape)
        h.copy_(x, non_blocking=True)
        outs.append(h)
    t.cuda.current_stream().synchronize()
    return [h.numpy() for h in outs]


def _torch_dtypes():
    t = torch()
    return {np.dtype(np.uint8): t.uint8, np.dtype(np.int32): t.int32,
            np.dtype(np.int64): t.int64, np.dtype(np.uint32): t.uint32,
            np.dtype(np.float32): t.float32, np.dtype(np.float64): t.float64,
            np.dtype(np.bool_): t.bool}


class _LazyDT(dict):
    def __missing__(self, key):
        self.update(_torch_dtypes())
        return dict.__getitem__(self, key)


_TORCH_OF = _LazyDT()


def tdtype(np_dtype):
    return _TORCH_OF[np.dtype(np_dtype)]
