"""Frame reconstruction: solve + see-through refocus, device-resident.

`FramePipeline` is the fused form of the reference pipeline's two hot stages
(pipeline.py:247-261: `DisparitySolver(...).solve()` then `synthesize(...)`)
for a stream of frames of one shape: every device buffer (descriptors, mu,
support lists, EM state, outputs, workspaces) is allocated once and reused,
so a frame costs its H2D copy, the kernels and the D2H of the artefacts.
`reconstruct` is the one-call host API on top of it.
"""

from dataclasses import dataclass

import os

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload
from .prior import PriorParams, TriDevice
from .solver import (DisparityMap, EMStats, SegmentationState, SolverParams, _check_views,
                     _stats_of)


class AsyncStats:
    """EM statistics still on the device (st_solve_async): resolved from the
    raw st_stats bytes that FramePipeline.fetch_async brings back
    (support_records is -1: the asynchronous support build does not read
    its record count back)."""

    def __init__(self, support_records):
        self.support_records = support_records

    def resolve(self, raw):
        s = N.StStats.from_buffer_copy(raw.tobytes())
        s.support_records = self.support_records
        return _stats_of(s)


@dataclass
class Reconstruction:
    disparity: DisparityMap
    segmentation: SegmentationState
    stats: EMStats
    image: np.ndarray
    provenance: np.ndarray
    n_rays: np.ndarray


class FramePipeline:
    """Persistent device buffers for frames of shape (K, H, W)."""

    def __init__(self, rig, width, height, params=None, prior_params=None, guard_bytes=0):
        t = require_cuda()
        self.t = t
        # guard_bytes > 0 (tests): every device buffer sits between two guard
        # zones of a known pattern; check_guards() finds out-of-bounds writes
        self.guard_bytes = int(guard_bytes)
        self._guards = []
        self.K = len(rig)
        _check_views(self.K)
        self.W, self.H = int(width), int(height)
        self.params = params or SolverParams()
        self.prior_params = prior_params or PriorParams()
        self.rig_obj = rig
        self.rig = N.make_rig(rig, self.W, self.H)
        K, H, W = self.K, self.H, self.W
        self.images = self._empty((K, H, W, 3), t.uint8)
        self.priors = self._empty((K, H, W), t.float32)
        self.desc = self._empty((K, H, W, 16), t.uint8)
        self.mu = self._empty((H * W,), t.float64)
        self.mu_ws = self._empty((1,), t.uint8)
        self.sup_ws = self._empty((1,), t.uint8)
        self.solve_ws = self._empty((int(N.lib().st_solve_workspace(W, H, K)),), t.uint8)
        self.values = self._empty((H, W), t.float32)
        self.status = self._empty((H, W), t.uint8)
        self.sbits = self._empty((H, W), t.int32)
        self.vbits = self._empty((H, W), t.int32)
        self.image = self._empty((H, W, 3), t.uint8)
        self.prov = self._empty((H, W), t.uint8)
        self.n_rays = self._empty((H, W), t.uint8)
        self.scratch = self._empty((H, W, 3), t.uint8)
        self.copy = self._empty((H, W), t.uint8)
        self.stats_dev = self._empty((N.C.sizeof(N.StStats),), t.uint8)
        self.frame = N.StFrame()
        self.frame.images = self.images.data_ptr()
        self.frame.priors = self.priors.data_ptr()
        self.frame.desc = self.desc.data_ptr()
        self.frame.mu = self.mu.data_ptr()
        # the surface raster is a latency-bound pointer chase on the pre-solve
        # critical path: its stream gets the higher priority, so its blocks are
        # scheduled ahead of the descriptor / support-group kernels
        prio = int(os.environ.get("ST_SIDE_PRIORITY", "-1"))
        self.side = t.cuda.Stream(priority=prio)
        self.side2 = t.cuda.Stream()
        # the slot's EM + refocus stream in reconstruct_stream: the slots'
        # frames are independent, so several are in flight at once (the EM's
        # later iterations are small latency-bound grids that leave most SMs
        # to the other frames)
        self.compute = t.cuda.Stream()

    def _empty(self, shape, dtype):
        if not self.guard_bytes:
            return empty(shape, dtype)
        t = self.t
        n = int(np.prod(shape)) * t.empty((), dtype=dtype).element_size()
        g = (self.guard_bytes + 255) & ~255
        raw = empty((n + 2 * g,), t.uint8)
        raw.fill_(0xA5)
        self._guards.append((raw, g, n))
        return raw[g:g + n].view(dtype).view(shape)

    def check_guards(self):
        """Number of guard-zone bytes overwritten since allocation (0 = none)."""
        bad = 0
        for raw, g, n in self._guards:
            bad += int((raw[:g] != 0xA5).sum()) + int((raw[g + n:] != 0xA5).sum())
        return bad

    # -- inputs ---------------------------------------------------------------------

    def load(self, images, priors):
        """Copy a frame into the input buffers (async DMA when the host side is pinned)."""
        t = self.t
        self._desc_ready = False
        for dst, src, dt in ((self.images, images, np.uint8), (self.priors, priors, np.float32)):
            if isinstance(src, t.Tensor):
                dst.copy_(src, non_blocking=True)
            elif isinstance(src, np.ndarray):
                dst.copy_(t.from_numpy(np.ascontiguousarray(src, dtype=dt)), non_blocking=True)
            else:
                # per-view host arrays: one native call for every view's copy
                views = [np.ascontiguousarray(a, dtype=dt) for a in src]
                per = dst[0].numel() * dst.element_size()
                if len(views) != dst.shape[0] or any(v.nbytes != per for v in views):
                    raise ValueError("frame views do not match the pipeline's shape")
                srcs, offs, sizes, n = N.gather_args(views, [k * per for k in range(len(views))])
                N.check(N.lib().st_h2d_gather(N.ptr(dst), srcs, offs, sizes, n,
                                              N.stream_handle()))
                self._hold = views  # (pageable sources: copied before the call returns)

    # -- the frame --------------------------------------------------------------------

    def harvest(self, threshold=None, stride=None, min_texture=None, counters=None):
        """Descriptors + the device support harvest of the loaded frame
        (st_harvest, prior.py:233-259 before deduplicate).  Enqueued on the
        current stream; returns (u, v, d, src, count) device tensors.
        counters: optional device int64[2] (candidates, reverse scans)."""
        from .prior import MIN_TEXTURE, SUPPORT_STRIDE, _grid_len
        t = self.t
        K, H, W = self.K, self.H, self.W
        thr = self.params.threshold if threshold is None else threshold
        stride = SUPPORT_STRIDE if stride is None else int(stride)
        mt = MIN_TEXTURE if min_texture is None else float(min_texture)
        if getattr(self, "_hv_key", None) != stride:
            lib = N.lib()
            cap = max(int(lib.st_harvest_capacity(K, W, H, stride)), 1)
            self.hv_ws = self._empty((max(int(lib.st_harvest_workspace(K, W, H, stride)), 1),),
                               t.uint8)
            self.hv_u = self._empty((cap,), t.int32)
            self.hv_v = self._empty((cap,), t.int32)
            self.hv_d = self._empty((cap,), t.float64)
            self.hv_src = self._empty((cap,), t.int32)
            self.hv_n = self._empty((1,), t.int64)
            self.cams = N.make_cams(self.rig_obj, W, H)
            self._hv_key = stride
        N.invoke("st_descriptors", self.images, K, H, W, 3, self.desc, None, None)
        self._desc_ready = True
        N.invoke("st_harvest", self.desc, self.priors, self.cams, float(self.prior_params.d_max),
                 _grid_len(self.prior_params.d_max), float(thr), stride, mt, self.hv_u,
                 self.hv_v, self.hv_d, self.hv_src, self.hv_n, counters, self.hv_ws,
                 self.hv_ws.numel())
        return self.hv_u, self.hv_v, self.hv_d, self.hv_src, self.hv_n

    def harvest_host(self, **kw):
        """harvest() + D2H + native dedup -> host (u, v, d, src) in the
        reference's final support order (prior.py:183-212)."""
        from .prior import deduplicate_arrays
        u, v, d, s, n = self.harvest(**kw)
        cnt = int(n.item())
        u, v, d, s = (download(x[:cnt]) for x in (u, v, d, s))
        keep = deduplicate_arrays(u, v, d, s, self.rig_obj.ref_index, self.W, self.H)
        return u[keep], v[keep], d[keep], s[keep]

    def run(self, tri_dev, dynamic_only=False, forced_iters=0, median_radius=1, timing=False,
            reduce=None, ready=None):
        """Descriptors, mu, support lists, EM, refocus + median for the loaded frame
        (descriptors are reused when harvest() already computed them).

        The pre-solve stages run on two side streams -- the surface raster
        (its Qhull-walk emulation is a long pointer chase) on one, the
        descriptors and the support candidate groups on the other -- and
        start at `ready` (default: now, on the current stream).  A caller
        that passes the event its frame's inputs were loaded on (see
        reconstruct_stream) lets them overlap the previous frame's EM."""
        p = N.make_params(self.params, self.prior_params, forced_iters, timing)
        K, H, W = self.K, self.H, self.W
        t = self.t
        main = t.cuda.current_stream()
        marks = []
        mark = (lambda: marks.append(self._event())) if timing else (lambda: None)
        mark()
        need = int(N.lib().st_mu_raster_workspace(W, H, tri_dev.n_tri))
        if self.mu_ws.numel() < need:
            self.mu_ws = self._empty((need,), t.uint8)
        if ready is None:
            ready = t.cuda.Event()
            ready.record(main)
        with t.cuda.stream(self.side):
            self.side.wait_event(ready)
            mu_start = self._event() if timing else None
            N.invoke("st_mu_raster", tri_dev.st, W, H, float(self.prior_params.d_max), self.mu,
                     self.mu_ws, self.mu_ws.numel())
            mu_done = self._event(timing=timing)
        need = int(N.lib().st_support_workspace(tri_dev.n_sup, W, H,
                                                float(self.prior_params.neighborhood_radius)))
        if self.sup_ws.numel() < need:
            self.sup_ws = self._empty((need,), t.uint8)
        # no host round trip unless a diagnostic path wants the record count
        # (dynamic_only: st_solve_rows reads the active-list size back once)
        run_async = not dynamic_only and reduce is None and not timing
        run_rows = bool(dynamic_only) and reduce is None and not timing
        rec = N.C.c_int64(-1)
        with t.cuda.stream(self.side2):
            self.side2.wait_event(ready)
            if getattr(self, "_desc_ready", False):
                self.side2.wait_stream(main)  # harvest() wrote them on the caller's stream
            else:
                N.invoke("st_descriptors", self.images, K, H, W, 3, self.desc, None, None)
            N.invoke("st_support_build", tri_dev.sup_uv, tri_dev.sup_d, tri_dev.n_sup, W, H, p,
                     self.frame, self.sup_ws, self.sup_ws.numel(),
                     None if (run_async or run_rows) else rec)
            pre_done = self._event(timing=False)
        self._desc_ready = False
        main.wait_event(pre_done)
        mark()
        main.wait_event(mu_done)
        mark()
        stats = N.StStats()
        if run_async:
            N.invoke("st_solve_async", self.frame, self.rig, p, self.values, self.status,
                     self.sbits, self.vbits, self.stats_dev, self.solve_ws,
                     self.solve_ws.numel())
        elif run_rows:
            N.check(N.lib().st_solve_rows(
                self.frame, self.rig, p, 1, 0, H, 0, H, N.ptr(self.values), N.ptr(self.status),
                N.ptr(self.sbits), N.ptr(self.vbits), N.ptr(self.stats_dev),
                N.ptr(self.solve_ws), self.solve_ws.numel(), N.EXCHANGE_FN(), None, 1, None,
                None, N.stream_handle()))
        else:
            cb = N.REDUCE_FN(reduce) if reduce is not None else N.REDUCE_FN()
            N.invoke("st_solve", self.frame, self.rig, p, int(bool(dynamic_only)), None,
                     self.values, self.status, self.sbits, self.vbits, stats, self.solve_ws,
                     self.solve_ws.numel(), cb, None)
        mark()
        stats.support_records = rec.value
        copy = None
        if dynamic_only:
            # pipeline.py:254-255: copy_mask = ref prior >= threshold (float32 compare)
            N.invoke("st_copy_mask", self.priors[self.rig.ref_index], H * W,
                     float(self.params.threshold), self.copy)
            copy = self.copy
        N.invoke("st_synthesize", self.images, self.rig, self.values, self.status, self.sbits,
                 int(self.params.min_static_rays), int(median_radius), copy, self.image,
                 self.prov, self.n_rays, self.scratch)
        mark()
        if run_async or run_rows:
            return AsyncStats(rec.value)
        out = _stats_of(stats)
        if timing:
            marks[-1].synchronize()
            names = ("descriptors_support", "mu_wait", "solve", "synthesize")
            out.stage_ms = {n: marks[i].elapsed_time(marks[i + 1]) for i, n in enumerate(names)}
            out.stage_ms["mu_raster_side_stream"] = mu_start.elapsed_time(mu_done)
        return out

    # -- native per-frame path (st_frame_run) -------------------------------------------

    def _plan_for(self, tri_dev, forced_iters, median_radius):
        t = self.t
        W, H = self.W, self.H
        lib = N.lib()
        P = getattr(self, "_plan", None)
        if P is None:
            P = N.StFramePlan()
            P.frame = self.frame
            P.rig = self.rig
            for name, x in (("values", self.values), ("status", self.status),
                            ("static_bits", self.sbits), ("valid_bits", self.vbits),
                            ("image", self.image), ("prov", self.prov), ("n_rays", self.n_rays),
                            ("scratch", self.scratch), ("stats_dev", self.stats_dev),
                            ("solve_ws", self.solve_ws)):
                setattr(P, name, x.data_ptr())
            P.solve_ws_bytes = self.solve_ws.numel()
            P.side_stream = self.side.cuda_stream
            P.side2_stream = self.side2.cuda_stream
            N.check(lib.st_frame_plan_init(N.C.byref(P)))
            self._plan = P
        P.params = N.make_params(self.params, self.prior_params, forced_iters, False)
        P.median_radius = int(median_radius)
        need = int(lib.st_mu_raster_workspace(W, H, tri_dev.n_tri))
        if self.mu_ws.numel() < need:
            self.mu_ws = self._empty((need,), t.uint8)
        need = int(lib.st_support_workspace(tri_dev.n_sup, W, H,
                                            float(self.prior_params.neighborhood_radius)))
        if self.sup_ws.numel() < need:
            self.sup_ws = self._empty((need,), t.uint8)
        P.mu_ws, P.mu_ws_bytes = self.mu_ws.data_ptr(), self.mu_ws.numel()
        P.sup_ws, P.sup_ws_bytes = self.sup_ws.data_ptr(), self.sup_ws.numel()
        P.main_stream = t.cuda.current_stream().cuda_stream
        P.descriptors_ready = 1 if getattr(self, "_desc_ready", False) else 0
        self._desc_ready = False
        return P

    def run_native(self, tri_dev, forced_iters=0, median_radius=1, ready=None, out_stream=None,
                   done=None):
        """run() + fetch_async() for the dense solve in one native call
        (st_frame_run): no per-stage Python, no host synchronisation.
        Returns (pinned host block or None, AsyncStats)."""
        t = self.t
        P = self._plan_for(tri_dev, forced_iters, median_radius)
        block = None
        if out_stream is not None:
            block = t.empty((int(N.lib().st_frame_host_bytes(self.W, self.H)),), dtype=t.uint8,
                            pin_memory=True)
            P.out_stream = out_stream.cuda_stream
        else:
            P.out_stream = None
        N.check(N.lib().st_frame_run(
            N.C.byref(P), N.C.byref(tri_dev.st), N.ptr(tri_dev.sup_uv), N.ptr(tri_dev.sup_d),
            int(tri_dev.n_sup), ready, None if block is None else N.C.c_void_p(block.data_ptr()),
            done))
        return block, AsyncStats(-1)

    def host_views(self, block):
        """The artefacts inside an st_frame_run host block (its layout)."""
        H, W = self.H, self.W
        specs = ((np.float32, (H, W)), (np.uint8, (H, W)), (np.uint32, (H, W)),
                 (np.uint32, (H, W)), (np.uint8, (H, W, 3)), (np.uint8, (H, W)),
                 (np.uint8, (H, W)), (np.uint8, (N.C.sizeof(N.StStats),)))
        raw = block.numpy()
        out, o = [], 0
        for dt, shape in specs:
            n = int(np.prod(shape)) * np.dtype(dt).itemsize
            out.append(raw[o:o + n].view(dt).reshape(shape))
            o += (n + 255) & ~255
        return out

    def __del__(self):
        P = getattr(self, "_plan", None)
        if P is not None:
            try:
                N.lib().st_frame_plan_destroy(N.C.byref(P))
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass

    def _event(self, timing=True):
        e = self.t.cuda.Event(enable_timing=timing)
        e.record(self.t.cuda.current_stream())
        return e

    # -- outputs ------------------------------------------------------------------------

    def device_bytes(self):
        """Device memory held by this pipeline (the cache's eviction weight)."""
        n = 0
        for x in vars(self).values():
            if hasattr(x, "is_cuda") and x.is_cuda:
                n += x.numel() * x.element_size()
        return n

    def output_bytes(self):
        return self.H * self.W * (4 + 1 + 4 + 4 + 3 + 1 + 1)

    def fetch(self):
        """D2H of every artefact into fresh pinned host buffers (torch's caching
        host allocator recycles them once the caller drops the arrays)."""
        host = self.fetch_async(self.t.cuda.current_stream())
        self.t.cuda.current_stream().synchronize()
        return host

    def fetch_async(self, stream):
        """Enqueue the D2H copies on `stream`; the arrays are valid once it syncs.

        One pinned block per frame (torch's caching host allocator recycles
        it once the caller drops the arrays), carved into the artefacts."""
        t = self.t
        devs = (self.values, self.status, self.sbits, self.vbits, self.image, self.prov,
                self.n_rays, self.stats_dev)
        offs, total = [], 0
        for d in devs:
            offs.append(total)
            total += (d.numel() * d.element_size() + 255) & ~255
        block = t.empty((total,), dtype=t.uint8, pin_memory=True)
        outs = []
        with t.cuda.stream(stream):
            for d, o in zip(devs, offs):
                n = d.numel() * d.element_size()
                h = block[o:o + n].view(d.dtype).view(d.shape)
                h.copy_(d, non_blocking=True)
                outs.append(h)
        return [h.numpy() for h in outs]


def _outputs_of(pipe, stats, host):
    values, status, sbits, vbits, img, prov, nr, raw_stats = host
    if isinstance(stats, AsyncStats):
        stats = stats.resolve(raw_stats)
    return Reconstruction(
        disparity=DisparityMap(values=values, status=status),
        segmentation=SegmentationState._device_result(sbits.view(np.uint32),
                                                      vbits.view(np.uint32)),
        stats=stats, image=img, provenance=prov, n_rays=nr)


def reconstruct_stream(items, rig, params=None, prior_params=None, dynamic_only=False,
                       median_radius=1, forced_iters=0):
    """Pipelined `reconstruct` over a sequence of (frame, tri) pairs.

    Yields one Reconstruction per frame, in order.  Device pipelines rotate
    (STREAM_SLOTS), each computing on its own stream, so several frames are
    in flight: a host thread uploads the next frames (pinned frames copy by
    DMA) and their triangulations on a copy stream, each frame's pre-solve
    stages, EM and refocus run on its slot's streams, and finished frames'
    artefacts stream back to pinned host memory on an output stream, in
    order; a frame is handed out once `depth` (STREAM_SLOTS - 1) later
    frames are enqueued.  Every frame gets the full per-frame work of
    `reconstruct`.

    ST_STREAM_COMPUTE selects the compute streams: "slot" (default, one per
    slot), an integer k (k slot streams in rotation) or "main" (the caller's
    stream: the frames' EMs serialised, frame i+1's pre-solve stages still
    overlapping frame i's EM); ST_STREAM_DEPTH the frames in flight
    (profiles/r02_stream_modes.txt).
    """
    import queue
    import threading

    t = require_cuda()
    params = params or SolverParams()
    prior_params = prior_params or PriorParams()
    it = iter(items)
    first = next(it, None)
    if first is None:
        return
    h, w = first[0].shape
    pipes = _stream_pipes(rig, w, h, params, prior_params)
    main = t.cuda.current_stream()
    copy_s, out_s = t.cuda.Stream(), t.cuda.Stream()
    n_slots = len(pipes)
    mode = os.environ.get("ST_STREAM_COMPUTE", "slot")
    compute_streams = ([main] if mode == "main" else
                       [x.compute for x in pipes][:n_slots if mode == "slot" else int(mode)])
    # frames enqueued ahead of the one being handed out (its D2H awaited):
    # concurrent compute streams need several in flight
    depth = int(os.environ.get("ST_STREAM_DEPTH",
                               "1" if len(compute_streams) == 1 else str(n_slots - 1)))
    depth = max(1, min(depth, n_slots - 1))
    free = [None] * n_slots      # event: pipe's inputs/outputs no longer in use
    free_lock = threading.Condition()
    q = queue.Queue(maxsize=max(1, len(pipes) - 1))  # prepared frames ahead of the consumer
    error = []

    device = t.cuda.current_device()

    import time
    prof = {} if os.environ.get("ST_STREAM_PROFILE") else None

    def tick(key, t0):
        if prof is not None:
            prof[key] = prof.get(key, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    stop = threading.Event()

    def put(item):
        while not stop.is_set():
            try:
                q.put(item, timeout=0.05)
                return True
            except queue.Full:
                continue
        return False

    def prep():
        t.cuda.set_device(device)
        try:
            for i, (frame, tri) in enumerate(_chain(first, it)):
                t0 = time.perf_counter()
                pipe = pipes[i % n_slots]
                with free_lock:
                    while i >= n_slots and free[i % n_slots] is None and not stop.is_set():
                        free_lock.wait()
                    if stop.is_set():
                        return
                    ev = free[i % n_slots]
                    free[i % n_slots] = None
                t0 = tick("prep_wait_free", t0)
                with t.cuda.stream(copy_s):
                    if ev is not None:
                        copy_s.wait_event(ev)
                    pipe.load(frame.images, frame.priors)
                    t0 = tick("prep_load", t0)
                    td = TriDevice(tri, slot=pipe)  # the slot's own staging + device buffer
                    t0 = tick("prep_tridevice", t0)
                    loaded = t.cuda.Event()
                    loaded.record(copy_s)
                # planes solved on the device only: numpy's singular-system
                # error is checked when the frame's outputs arrive
                if not put((pipe, td, loaded, tri.planes is None)):
                    return
        except Exception as exc:  # noqa: BLE001 -- surfaced in the consumer
            error.append(exc)
        put(None)

    worker = threading.Thread(target=prep, daemon=True)
    worker.start()
    from collections import deque
    pending = deque()
    i = 0
    try:
        while True:
            t0 = time.perf_counter()
            item = q.get()
            if item is None:
                break
            t0 = tick("main_wait_prep", t0)
            pipe, td, loaded, check = item
            cs = compute_streams[i % len(compute_streams)]
            cs.wait_event(loaded)
            for x in td.tensors():
                for st_ in (cs, pipe.side, pipe.side2):
                    x.record_stream(st_)
            # the frame's pre-solve stages start as soon as its inputs are on the
            # device, its EM on the slot's stream, concurrently with the frames
            # of the other slots
            if not dynamic_only:
                # one native call enqueues the whole frame and its D2H (st_frame_run)
                fetched = t.cuda.Event()
                fetched.record(out_s)  # creates the event; st_frame_run re-records it
                with t.cuda.stream(cs):
                    block, stats = pipe.run_native(td, forced_iters=forced_iters,
                                                   median_radius=median_radius, ready=loaded,
                                                   out_stream=out_s, done=fetched)
                host = pipe.host_views(block)
                t0 = tick("main_run", t0)
                with t.cuda.stream(out_s):
                    flags = None
                    if check and td.flags is not None:
                        flags = t.empty((1,), dtype=t.int32, pin_memory=True)
                        flags.copy_(td.flags, non_blocking=True)
                        fetched = t.cuda.Event()
                        fetched.record(out_s)
            else:
                with t.cuda.stream(cs):
                    stats = pipe.run(td, dynamic_only=dynamic_only, forced_iters=forced_iters,
                                     median_radius=median_radius, ready=loaded)
                t0 = tick("main_run", t0)
                done = t.cuda.Event()
                done.record(cs)
                with t.cuda.stream(out_s):
                    out_s.wait_event(done)
                    host = pipe.fetch_async(out_s)
                    flags = None
                    if check and td.flags is not None:
                        flags = t.empty((1,), dtype=t.int32, pin_memory=True)
                        flags.copy_(td.flags, non_blocking=True)
                    fetched = t.cuda.Event()
                    fetched.record(out_s)
            with free_lock:
                free[i % n_slots] = fetched
                free_lock.notify_all()
            t0 = tick("main_fetch_enqueue", t0)
            pending.append((pipe, stats, fetched, host, flags))
            i += 1
            if len(pending) > depth:
                out = _finish(pending.popleft())
                t0 = tick("main_finish_prev", t0)
                yield out
                t0 = time.perf_counter()
        if error:
            raise error[0]
        while pending:
            yield _finish(pending.popleft())
    finally:
        # normal end, an error, or a consumer that stopped early (generator
        # close): stop the prep thread, let the device finish every enqueued
        # copy into pinned host blocks before they can be recycled, and hand
        # the pipelines back
        stop.set()
        with free_lock:
            free_lock.notify_all()
        while True:
            try:
                q.get_nowait()
            except queue.Empty:
                break
        worker.join()
        for s_ in [copy_s, main, out_s] + compute_streams:
            s_.synchronize()
        pipes.busy = False
        if prof is not None:
            print("reconstruct_stream profile (s, summed over frames):",
                  {k: round(v, 4) for k, v in sorted(prof.items())}, f"frames={i}", flush=True)


def _finish(pending):
    pipe, stats, fetched, host, flags = pending
    fetched.synchronize()
    if flags is not None and int(flags[0]) & 1:
        raise ValueError("degenerate support set: zero-area triangle")
    return _outputs_of(pipe, stats, host)


def reconstruct_frames(frames, rig, params=None, prior_params=None, dynamic_only=False,
                       median_radius=1, forced_iters=0, workers=None, inflight=None):
    """The reference pipeline's compute stages (pipeline.py:233-261) over a
    stream of raw frames: device harvest + native dedup per frame on a side
    stream, host Qhull in a process pool (several frames in flight), then
    the pipelined device solve + refocus of reconstruct_stream.  Yields one
    Reconstruction per frame, in order."""
    from collections import deque

    from .qhull_pool import delaunay_tables, make_pool, prior_of
    t = require_cuda()
    params = params or SolverParams()
    prior_params = prior_params or PriorParams()

    def triangulated():
        it = iter(frames)
        first = next(it, None)
        if first is None:
            return
        h, w = first.shape
        hp = FramePipeline(rig, w, h, params, prior_params)
        hs = t.cuda.Stream()
        pool, n = make_pool(workers)
        depth = inflight or n + 2
        q = deque()
        try:
            for frame in _chain(first, it):
                if frame.num_views != len(rig):
                    raise ValueError("frame view count does not match the rig")
                with t.cuda.stream(hs):
                    hp.load(frame.images, frame.priors)
                    u, v, d, _ = hp.harvest_host()
                q.append((frame, pool.submit(delaunay_tables, u, v, d, w, h)))
                if len(q) >= depth:
                    f0, fut = q.popleft()
                    yield f0, prior_of(fut.result())
            while q:
                f0, fut = q.popleft()
                yield f0, prior_of(fut.result())
        finally:
            for _, fut in q:
                fut.cancel()

    yield from reconstruct_stream(triangulated(), rig, params, prior_params,
                                  dynamic_only=dynamic_only, median_radius=median_radius,
                                  forced_iters=forced_iters)


def _chain(first, rest):
    yield first
    yield from rest


_PIPES = None
_STREAM_PIPES = None
CACHE_BYTES = int(os.environ.get("ST_PIPE_CACHE_BYTES", str(8 << 30)))  # device bytes kept


class _PipePair(list):
    busy = False


# Frames in flight.  A frame's H2D may start once its slot's previous frame
# has left (its D2H done); with too few slots that gate, not the link or the
# kernels, sets the stream's period (3 slots: H2D + pre-solve chain per frame)
STREAM_SLOTS = int(os.environ.get("ST_STREAM_SLOTS", "5"))


def _rig_key(rig, w, h, params, prior_params):
    """Cache key on the rig's CONTENTS (its st_rig bytes: view count, reference
    view, warp tables, view sizes), not on the object: pipeline.run_reconstruct
    loads a fresh rig for every call (geometry.py:326 load_calibration)."""
    return (bytes(N.make_rig(rig, w, h)), w, h, repr(params), repr(prior_params))


def _adopt(pipe, rig):
    """A cached pipeline serving a content-equal rig object: host-side users of
    the rig (harvest cameras, ref_index) follow the caller's object."""
    if pipe.rig_obj is not rig:
        pipe.rig_obj = rig
        pipe._hv_key = None
    return pipe


class _Cache:
    """LRU of device pipelines bounded by device bytes (CACHE_BYTES)."""

    def __init__(self):
        from collections import OrderedDict
        self.items = OrderedDict()

    def get(self, key):
        v = self.items.get(key)
        if v is not None:
            self.items.move_to_end(key)
        return v

    def put(self, key, value, nbytes):
        self.items[key] = (value, nbytes)
        self.items.move_to_end(key)
        total = sum(b for _, b in self.items.values())
        for k in list(self.items):
            if total <= CACHE_BYTES or k == key:
                break
            v, b = self.items[k]
            if getattr(v, "busy", False):
                continue
            del self.items[k]
            total -= b


def _stream_pipes(rig, w, h, params, prior_params):
    """The rotating pipelines of reconstruct_stream, kept across calls; a set
    in use by a running stream is never handed out twice."""
    global _STREAM_PIPES
    if _STREAM_PIPES is None:
        _STREAM_PIPES = _Cache()
    key = _rig_key(rig, w, h, params, prior_params)
    hit = _STREAM_PIPES.get(key)
    if hit is not None and not hit[0].busy:
        p = hit[0]
        for x in p:
            _adopt(x, rig)
    else:
        p = _PipePair(FramePipeline(rig, w, h, params, prior_params)
                      for _ in range(STREAM_SLOTS))
        if hit is None:
            _STREAM_PIPES.put(key, p, sum(x.device_bytes() for x in p))
    p.busy = True
    return p


def _pipeline_for(rig, w, h, params, prior_params):
    global _PIPES
    if _PIPES is None:
        _PIPES = _Cache()
    key = _rig_key(rig, w, h, params, prior_params)
    hit = _PIPES.get(key)
    if hit is not None:
        return _adopt(hit[0], rig)
    p = FramePipeline(rig, w, h, params, prior_params)
    _PIPES.put(key, p, p.device_bytes())
    return p


def reconstruct(frame, rig, tri, params=None, prior_params=None, dynamic_only=False,
                median_radius=1, forced_iters=0):
    """em_solve + synthesize in one device pass: host frame in, host artefacts out.

    dynamic_only follows pipeline.py:252-258 (only pixels whose reference
    prior is below the threshold are solved; the rest are copied through).
    forced_iters > 0 runs exactly that many EM iterations (non-reference
    bench mode).  Returned arrays are fresh copies (the reference's "new
    arrays out" contract).
    """
    params = params or SolverParams()
    prior_params = prior_params or PriorParams()
    if frame.num_views != len(rig):
        raise ValueError("frame view count does not match the rig")
    h, w = frame.shape
    pipe = _pipeline_for(rig, w, h, params, prior_params)
    pipe.load(frame.images, frame.priors)
    td = TriDevice(tri)
    if not dynamic_only:
        cur = pipe.t.cuda.current_stream()
        block, stats = pipe.run_native(td, forced_iters=forced_iters, median_radius=median_radius,
                                       out_stream=cur)
        cur.synchronize()
        return _outputs_of(pipe, stats, pipe.host_views(block))
    stats = pipe.run(td, dynamic_only=dynamic_only, forced_iters=forced_iters,
                     median_radius=median_radius)
    return _outputs_of(pipe, stats, pipe.fetch())


def reconstruct_frame(frame, rig, params=None, prior_params=None, dynamic_only=False,
                      median_radius=1, forced_iters=0, timings=None):
    """The reference pipeline's compute stages from a raw frame
    (pipeline.py:233-261): collect_support (device harvest + native dedup),
    triangulate (host Qhull, like the reference), em_solve + synthesize
    (device).  Returns (Reconstruction, TriangulationPrior).  `timings`
    (optional dict) receives host wall-clock seconds per stage."""
    import time

    from .prior import triangulate_arrays
    t = require_cuda()
    params = params or SolverParams()
    prior_params = prior_params or PriorParams()
    if frame.num_views != len(rig):
        raise ValueError("frame view count does not match the rig")
    h, w = frame.shape
    pipe = _pipeline_for(rig, w, h, params, prior_params)
    clock = time.perf_counter
    t0 = clock()
    pipe.load(frame.images, frame.priors)
    u, v, d, _ = pipe.harvest_host()
    t1 = clock()
    tri = triangulate_arrays(u, v, d, w, h, planes=False)
    t2 = clock()
    td = TriDevice(tri)
    stats = pipe.run(td, dynamic_only=dynamic_only, forced_iters=forced_iters,
                     median_radius=median_radius)
    rec = _outputs_of(pipe, stats, pipe.fetch())
    td.check()  # the planes were solved on the device: surface numpy's error here
    t3 = clock()
    if timings is not None:
        timings.update(support=t1 - t0, triangulate=t2 - t1, solve_refocus=t3 - t2)
    del t
    return rec, tri
