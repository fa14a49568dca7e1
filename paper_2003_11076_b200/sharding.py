"""Multi-GPU decompositions of the hot path.

* Frame-parallel (BASELINE C5): every rank reconstructs its own frames; no
  collective on the data path (see bench.py).
* Row bands (C3/C4): every rank holds the frame, solves the pixels of its
  band of reference rows (an explicit active mask for `st_solve`), and the
  per-iteration statistics -- energy sums and changed/active counts -- are
  summed across ranks through `st_solve`'s reduce callback, so the
  reference's GLOBAL convergence rule (solver.py:473-485) and the EMStats
  means are those of the whole frame.  Pixels are independent within an
  iteration (solver.py:30-32) and the support groups and surface are built
  from the whole frame, so a banded solve reproduces the single-device
  solve exactly.  The bands are then gathered to every rank.
"""

import numpy as np


def band_rows(height, world, rank):
    """Contiguous, balanced [r0, r1) row range of `rank`."""
    base, extra = divmod(height, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def band_mask(height, width, world, rank):
    m = np.zeros((height, width), dtype=np.uint8)
    r0, r1 = band_rows(height, world, rank)
    m[r0:r1] = 1
    return m


class CollectiveReduce:
    """`st_reduce_fn` implemented with torch.distributed (sum, in place).

    The callback receives a small double array per EM iteration; integer
    counts stay exact below 2^53.
    """

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.device = device or ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
        self.calls = 0

    def __call__(self, values, n, user):
        t = self.torch
        try:
            buf = t.tensor([values[i] for i in range(n)], dtype=t.float64, device=self.device)
            self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)
            host = buf.cpu().tolist()
            for i in range(n):
                values[i] = host[i]
            self.calls += 1
            return 0
        except Exception:  # noqa: BLE001 -- report failure to the C side
            return 1


def gather_bands(local, height, world, rank, group=None):
    """Assemble a full-frame array from every rank's band rows (all ranks get it).

    local: this rank's full-size (H, ...) array whose band rows are valid.
    """
    import torch
    import torch.distributed as dist
    r0, r1 = band_rows(height, world, rank)
    rows = band_rows(height, world, 0)[1] - band_rows(height, world, 0)[0]  # largest band
    a = np.ascontiguousarray(local)
    tail = a.shape[1:]
    pad = np.zeros((rows,) + tail, dtype=a.dtype)
    pad[:r1 - r0] = a[r0:r1]
    as_bytes = torch.from_numpy(pad.view(np.uint8).reshape(rows, -1).copy())
    backend = dist.get_backend(group)
    if backend == "nccl":
        as_bytes = as_bytes.cuda()
    out = [torch.empty_like(as_bytes) for _ in range(world)]
    dist.all_gather(out, as_bytes, group=group)
    full = np.empty_like(a)
    for r in range(world):
        s0, s1 = band_rows(height, world, r)
        blk = out[r].cpu().numpy().reshape((rows,) + (-1,)).view(a.dtype).reshape((rows,) + tail)
        full[s0:s1] = blk[:s1 - s0]
    return full


def solve_band(solver, world, rank, dynamic_only=False, group=None, forced_iters=0):
    """Banded `DisparitySolver.solve`: returns full-frame (DisparityMap,
    SegmentationState, EMStats) on every rank, identical to a single-device
    solve of the whole frame."""
    import torch
    from .device import download
    from .solver import DisparityMap, SegmentationState
    h, w = solver.height, solver.width
    mask = band_mask(h, w, world, rank)
    if dynamic_only:
        ref = solver.frame.priors[solver.rig.ref_index]
        mask &= (np.asarray(ref, dtype=np.float32) < np.float32(solver.params.threshold))
    red = CollectiveReduce(group)
    (values, status, sbits, vbits), stats = solver.solve_device(
        active_mask=mask, forced_iters=forced_iters, reduce=red)
    torch.cuda.synchronize()
    parts = [download(x) for x in (values, status, sbits, vbits)]
    values, status, sbits, vbits = (gather_bands(p, h, world, rank, group) for p in parts)
    return (DisparityMap(values=values, status=status),
            SegmentationState(static_bits=sbits.view(np.uint32), valid_bits=vbits.view(np.uint32)),
            stats)
