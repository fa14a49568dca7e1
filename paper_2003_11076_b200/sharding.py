"""Multi-GPU decompositions of the hot path.

* Frame-parallel (BASELINE C5): every rank reconstructs its own frames; no
  collective on the data path (bench.py, reconstruct_stream per rank).
* Row bands (BASELINE C3/C4): one frame split across ranks by rows of the
  reference view (`reconstruct_band`, `BandPipeline`).  Pixels are
  independent within an iteration (solver.py:30-32) and on a rectified rig
  (A = I, b = (bx, 0, 0); the synthetic linear array) every sample of a
  band row reads the SAME row of every view, so a rank only needs:
    - its band [r0, r1) plus the median's halo rows (solved too: halo pixels
      are pure per-pixel functions of the same global iteration count, so
      they equal the neighbour's own -- no halo exchange),
    - the 3-row descriptor halo (Sobel + ring offsets, features.py:9-11) of
      the input views: only those rows are copied host -> device,
    - the support list (KB-scale, replicated) and the surface raster (the
      Qhull walk replay runs over the whole frame on every rank: measured,
      see DESIGN.md §7).
  Collectives (torch.distributed; NCCL over NVLink on the GPU box):
    1. per EM iteration, an all-gather of every shard's 96-byte statistics
       record, stream-ordered inside st_solve_rows (k_band_control sums
       the records in rank order on the device), so the reference's GLOBAL
       convergence rule (solver.py:473-485) and the EMStats means hold
       across bands with no host round trip per iteration beyond reading
       the stop flag;
    2. the output band gather to rank `dst` (point-to-point sends of each
       artefact's band rows straight into the destination's full-frame
       buffers: one NCCL group).
  Non-rectified rigs fall back to full-frame inputs per rank (the warped
  rows of a band can lie anywhere); only the solve and refocus are banded.
"""

import ctypes

import numpy as np

from . import _native as N
from .device import empty, require_cuda


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


DESC_HALO = 3   # features.py:20 DESCRIPTOR_MARGIN: Sobel (1) + ring offsets (2)


def is_rectified(rig):
    """Every view warps rows onto themselves: A = I, b = (bx, 0, 0)
    (the st_api.cu make_ctx test)."""
    for k in range(len(rig)):
        a, b = rig.warp_coefficients(k)
        a = np.asarray(a, dtype=np.float64).reshape(9)
        b = np.asarray(b, dtype=np.float64).reshape(3)
        if not (np.array_equal(a, np.eye(3).reshape(9)) and b[1] == 0.0 and b[2] == 0.0
                and abs(b[0]) < 1e300):
            return False
    return True


def band_extents(height, world, rank, median_radius=1, rectified=True):
    """Row ranges of one band: `rows` (its own, counted in the statistics),
    `solve` (+ the median's halo), `desc` (descriptors computed), `images`
    and `priors` (host rows copied to the device)."""
    r0, r1 = band_rows(height, world, rank)
    mr = max(int(median_radius), 0)
    e0, e1 = max(0, r0 - mr), min(height, r1 + mr)
    if rectified:
        d0, d1 = max(0, e0 - 1), min(height, e1 + 1)
        i0, i1 = max(0, d0 - DESC_HALO), min(height, d1 + DESC_HALO)
        p0, p1 = d0, d1
    else:
        d0, d1 = i0, i1 = p0, p1 = 0, height
    return {"rows": (r0, r1), "solve": (e0, e1), "desc": (d0, d1), "images": (i0, i1),
            "priors": (p0, p1)}


# -- collectives ------------------------------------------------------------------------

class RecordExchange:
    """st_exchange_fn: all-gather of the shards' statistics records.

    NCCL: `all_gather_into_tensor` on the solve stream (stream-ordered, no
    host synchronisation).  gloo (tests, CPU-staged): a blocking gather
    through host memory."""

    def __init__(self, send, recv, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.send, self.recv, self.group = send, recv, group
        self.nccl = dist.get_backend(group) == "nccl"
        self.calls = 0
        self.error = None
        self.fn = N.EXCHANGE_FN(self._call)

    def _call(self, stream, user):
        try:
            if self.nccl:
                self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            else:
                import torch
                world = self.dist.get_world_size(self.group)
                host = self.send.cpu()
                outs = [torch.empty_like(host) for _ in range(world)]
                self.dist.all_gather(outs, host, group=self.group)
                self.recv.copy_(torch.cat(outs).to(self.recv.device))
            self.calls += 1
            return 0
        except Exception as exc:  # noqa: BLE001 -- reported through the C return code
            self.error = exc
            return 1


def gather_rows(arrays, height, world, rank, dst=0, group=None):
    """Send each full-frame device array's band rows to rank `dst`, which
    receives every other band straight into its own arrays' rows."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return
    nccl = dist.get_backend(group) == "nccl"
    bands = [band_rows(height, world, r) for r in range(world)]
    if nccl:
        ops = []
        for a in arrays:
            if rank == dst:
                for r in range(world):
                    if r != dst and bands[r][1] > bands[r][0]:
                        ops.append(dist.P2POp(dist.irecv, a[bands[r][0]:bands[r][1]], r,
                                              group=group))
            elif bands[rank][1] > bands[rank][0]:
                ops.append(dist.P2POp(dist.isend, a[bands[rank][0]:bands[rank][1]], dst,
                                      group=group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return
    # gloo: CPU staging
    for a in arrays:
        if rank == dst:
            for r in range(world):
                if r == dst or bands[r][1] <= bands[r][0]:
                    continue
                buf = torch.empty_like(a[bands[r][0]:bands[r][1]], device="cpu")
                dist.recv(buf, src=r, group=group)
                a[bands[r][0]:bands[r][1]].copy_(buf)
        elif bands[rank][1] > bands[rank][0]:
            dist.send(a[bands[rank][0]:bands[rank][1]].cpu().contiguous(), dst=dst, group=group)


# -- the band pipeline ----------------------------------------------------------------------

class BandPipeline:
    """One rank's share of a row-band sharded frame of shape (K, H, W).

    Buffers are full-frame sized (global pixel indexing everywhere), but a
    frame only moves and computes its band's rows (+ halos)."""

    def __init__(self, rig, width, height, params=None, prior_params=None, group=None,
                 median_radius=1, guard_bytes=0):
        from .prior import PriorParams
        from .reconstruct import FramePipeline
        from .solver import SolverParams
        import torch.distributed as dist
        t = require_cuda()
        self.t = t
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.params = params or SolverParams()
        self.prior_params = prior_params or PriorParams()
        self.pipe = FramePipeline(rig, width, height, self.params, self.prior_params,
                                  guard_bytes=guard_bytes)
        self.K, self.H, self.W = self.pipe.K, self.pipe.H, self.pipe.W
        self.rectified = is_rectified(rig)
        self.median_radius = int(median_radius)
        self.ext = band_extents(self.H, self.world, self.rank, median_radius, self.rectified)
        nrec = int(N.lib().st_band_record_bytes())
        self.rec_send = empty((nrec,), t.uint8)
        self.rec_recv = empty((self.world * nrec,), t.uint8)
        self.exchange = RecordExchange(self.rec_send, self.rec_recv, group) \
            if self.world > 1 else None
        self.mu_unsafe = empty((1,), t.int32)
        self.retries = 0  # frames redone with the whole-frame surface raster

    # -- inputs -------------------------------------------------------------------------

    def load(self, images, priors):
        """Copy the band's input rows (host numpy (K,H,W,3)/(K,H,W) arrays or
        per-view lists; pinned sources copy by DMA)."""
        t = self.t
        i0, i1 = self.ext["images"]
        p0, p1 = self.ext["priors"]
        for dst, src, dt, (a, b) in ((self.pipe.images, images, np.uint8, (i0, i1)),
                                     (self.pipe.priors, priors, np.float32, (p0, p1))):
            for k in range(self.K):
                s = src[k]
                if isinstance(s, t.Tensor):
                    dst[k, a:b].copy_(s[a:b], non_blocking=True)
                else:
                    dst[k, a:b].copy_(t.from_numpy(np.ascontiguousarray(s[a:b], dtype=dt)),
                                      non_blocking=True)

    def h2d_bytes(self):
        i0, i1 = self.ext["images"]
        p0, p1 = self.ext["priors"]
        return self.K * self.W * ((i1 - i0) * 3 + (p1 - p0) * 4)

    # -- the frame ----------------------------------------------------------------------

    def run(self, tri_dev, dynamic_only=False, forced_iters=0):
        """Descriptors of the band rows, surface raster and support groups
        (whole frame), the banded EM with the per-iteration exchange, and
        the refocus + median of the band; on the current stream."""
        t = self.t
        pipe = self.pipe
        K, H, W = self.K, self.H, self.W
        p = N.make_params(self.params, self.prior_params, forced_iters, False)
        main = t.cuda.current_stream()
        ready = t.cuda.Event()
        ready.record(main)
        need = int(N.lib().st_mu_raster_workspace(W, H, tri_dev.n_tri))
        if pipe.mu_ws.numel() < need:
            pipe.mu_ws = pipe._empty((need,), t.uint8)
        e0, e1 = self.ext["solve"]
        banded_mu = self.world > 1 and (e0 > 0 or e1 < H)
        with t.cuda.stream(pipe.side):
            pipe.side.wait_event(ready)
            if banded_mu:
                # the band's solved rows only (+ 2 halo rows of walks); the
                # flag rides in the first statistics record (ST_EAGAIN below)
                N.invoke("st_mu_raster_rows", tri_dev.st, W, H, float(self.prior_params.d_max),
                         pipe.mu, pipe.mu_ws, pipe.mu_ws.numel(), e0, e1, self.mu_unsafe)
                pipe.frame.mu_unsafe = self.mu_unsafe.data_ptr()
            else:
                N.invoke("st_mu_raster", tri_dev.st, W, H, float(self.prior_params.d_max),
                         pipe.mu, pipe.mu_ws, pipe.mu_ws.numel())
                pipe.frame.mu_unsafe = None
            mu_done = t.cuda.Event()
            mu_done.record(pipe.side)
        need = int(N.lib().st_support_workspace(tri_dev.n_sup, W, H,
                                                float(self.prior_params.neighborhood_radius)))
        if pipe.sup_ws.numel() < need:
            pipe.sup_ws = pipe._empty((need,), t.uint8)
        d0, d1 = self.ext["desc"]
        with t.cuda.stream(pipe.side2):
            pipe.side2.wait_event(ready)
            N.invoke("st_descriptors_rows", pipe.images, K, H, W, pipe.desc, d0, d1)
            e0, e1 = self.ext["solve"]
            N.invoke("st_support_build_rows", tri_dev.sup_uv, tri_dev.sup_d, tri_dev.n_sup, W,
                     H, p, pipe.frame, pipe.sup_ws, pipe.sup_ws.numel(), None, e0, e1)
            pre_done = t.cuda.Event()
            pre_done.record(pipe.side2)
        main.wait_event(pre_done)
        main.wait_event(mu_done)
        r0, r1 = self.ext["rows"]
        ex = self.exchange
        fn = ex.fn if ex is not None else N.EXCHANGE_FN()

        def solve():
            rc = N.lib().st_solve_rows(
                pipe.frame, pipe.rig, p, int(bool(dynamic_only)), r0, r1, e0, e1,
                N.ptr(pipe.values), N.ptr(pipe.status), N.ptr(pipe.sbits), N.ptr(pipe.vbits),
                N.ptr(pipe.stats_dev), N.ptr(pipe.solve_ws), pipe.solve_ws.numel(), fn, None,
                self.world, N.ptr(self.rec_send), N.ptr(self.rec_recv), N.stream_handle())
            if rc and ex is not None and ex.error is not None:
                raise ex.error
            N.check(rc)

        try:
            solve()
        except N.BandRetry:
            # some shard's row-window raster was not exact (every shard sees
            # the same gathered records, so all of them retry together)
            self.retries += 1
            N.invoke("st_mu_raster", tri_dev.st, W, H, float(self.prior_params.d_max), pipe.mu,
                     pipe.mu_ws, pipe.mu_ws.numel())
            pipe.frame.mu_unsafe = None
            solve()
        copy = None
        if dynamic_only:
            N.invoke("st_copy_mask", pipe.priors[pipe.rig.ref_index], H * W,
                     float(self.params.threshold), pipe.copy)
            copy = pipe.copy
        N.invoke("st_synthesize_rows", pipe.images, pipe.rig, pipe.values, pipe.status,
                 pipe.sbits, int(self.params.min_static_rays), self.median_radius, copy,
                 pipe.image, pipe.prov, pipe.n_rays, pipe.scratch, r0, r1, e0, e1)

    def outputs(self):
        pipe = self.pipe
        return [pipe.values, pipe.status, pipe.sbits, pipe.vbits, pipe.image, pipe.prov,
                pipe.n_rays]

    def gather(self, dst=0):
        """The artefact bands onto rank `dst` (stream-ordered under NCCL)."""
        gather_rows(self.outputs(), self.H, self.world, self.rank, dst, self.group)

    def stats(self):
        from .solver import _stats_of
        raw = self.pipe.stats_dev.cpu().numpy()
        return _stats_of(N.StStats.from_buffer_copy(raw.tobytes()))

    def fetch(self):
        """D2H of the full-frame artefacts (rank `dst` after gather())."""
        from .reconstruct import _outputs_of
        host = self.pipe.fetch()
        return _outputs_of(self.pipe, self.stats(), host)


_BANDS = {}


def band_pipeline(rig, width, height, params, prior_params, group=None, median_radius=1):
    import torch.distributed as dist
    from .reconstruct import _rig_key
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    key = (_rig_key(rig, width, height, params, prior_params), id(group), world, rank,
           int(median_radius))
    p = _BANDS.get(key)
    if p is None:
        if len(_BANDS) > 2:
            _BANDS.clear()
        p = _BANDS[key] = BandPipeline(rig, width, height, params, prior_params, group,
                                       median_radius)
    return p


def reconstruct_band(frame, rig, tri, params=None, prior_params=None, group=None,
                     dynamic_only=False, median_radius=1, forced_iters=0, dst=0):
    """`reconstruct` of one frame split into row bands across the ranks of
    `group` (one GPU each).  Every rank passes the same frame and
    triangulation; rank `dst` returns the full-frame Reconstruction (the
    single-device result, bit for bit), the others return None."""
    from .prior import TriDevice
    from .solver import _check_views
    if frame.num_views != len(rig):
        raise ValueError("frame view count does not match the rig")
    _check_views(frame.num_views)
    h, w = frame.shape
    bp = band_pipeline(rig, w, h, params, prior_params, group, median_radius)
    bp.load(frame.images, frame.priors)
    td = TriDevice(tri)
    bp.run(td, dynamic_only=dynamic_only, forced_iters=forced_iters)
    bp.gather(dst)
    if bp.rank != dst:
        bp.t.cuda.current_stream().synchronize()
        return None
    rec = bp.fetch()
    td.check()
    return rec


def solve_band(solver, world=None, rank=None, dynamic_only=False, group=None, forced_iters=0):
    """Banded `DisparitySolver.solve` on a solver whose frame is on every
    rank: returns full-frame (DisparityMap, SegmentationState, EMStats) on
    every rank, identical to a single-device solve of the whole frame."""
    import torch
    import torch.distributed as dist
    from .device import download
    from .solver import DisparityMap, SegmentationState, _stats_of
    t = require_cuda()
    world = dist.get_world_size(group) if world is None else world
    rank = dist.get_rank(group) if rank is None else rank
    h, w = solver.height, solver.width
    r0, r1 = band_rows(h, world, rank)
    values = empty((h, w), t.float32)
    status = empty((h, w), t.uint8)
    sbits = empty((h, w), t.int32)
    vbits = empty((h, w), t.int32)
    stats_dev = empty((ctypes.sizeof(N.StStats),), t.uint8)
    nbytes = int(N.lib().st_solve_workspace(w, h, solver.num_views))
    ws = empty((nbytes,), t.uint8)
    nrec = int(N.lib().st_band_record_bytes())
    send = empty((nrec,), t.uint8)
    recv = empty((world * nrec,), t.uint8)
    ex = RecordExchange(send, recv, group) if world > 1 else None
    p = N.make_params(solver.params, solver.prior_params, forced_iters)
    rc = N.lib().st_solve_rows(solver._frame, solver._rig, p, int(bool(dynamic_only)), r0, r1,
                               r0, r1, N.ptr(values), N.ptr(status), N.ptr(sbits), N.ptr(vbits),
                               N.ptr(stats_dev), N.ptr(ws), ws.numel(),
                               ex.fn if ex is not None else N.EXCHANGE_FN(), None, world,
                               N.ptr(send), N.ptr(recv), N.stream_handle())
    if rc and ex is not None and ex.error is not None:
        raise ex.error
    N.check(rc)
    outs = [values, status, sbits, vbits]
    if world > 1:
        # every rank gets the whole frame: each band from its owner
        for src in range(world):
            s0, s1 = band_rows(h, world, src)
            for a in outs:
                if dist.get_backend(group) == "nccl":
                    dist.broadcast(a[s0:s1], src=src, group=group)
                else:
                    buf = a[s0:s1].cpu()
                    dist.broadcast(buf, src=src, group=group)
                    a[s0:s1].copy_(buf)
    torch.cuda.synchronize()
    stats = _stats_of(N.StStats.from_buffer_copy(download(stats_dev).tobytes()))
    stats.support_records = solver._support_records
    return (DisparityMap(values=download(values), status=download(status)),
            SegmentationState(static_bits=download(sbits).view(np.uint32),
                              valid_bits=download(vbits).view(np.uint32)),
            stats)
