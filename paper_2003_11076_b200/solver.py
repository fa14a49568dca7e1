"""EM estimation of background disparity and per-ray static masks (solver.py).

Drop-in for the reference's DisparitySolver / em_solve / e_step /
masked_variance with the same signatures, dtypes and error messages.  All
per-pixel work runs in the CUDA library:

- `solve()` is one native call (`st_solve`): initial masks, then per
  iteration the M-step kernel (candidate argmin with the previous-disparity
  energy and changed count fused in) and the E-step kernel (2^K mask argmax),
  with the reference's global convergence rule between iterations.
- the per-method API (`m_step`, `e_step_at`, `gather_rays`, `initial_masks`,
  `pixel_energy`) launches the same kernels on explicit pixel lists.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload
from .features import DESCRIPTOR_LENGTH
from .frame import device_frame
from .prior import PriorParams, candidate_disparities, mu_raster_device

VARIANCE_CEILING = float(DESCRIPTOR_LENGTH) * 127.5 ** 2
MAX_ENUMERATED_VIEWS = 12
STATUS_VALID = 0
STATUS_LOW_TEXTURE = 1
STATUS_NO_STATIC_EVIDENCE = 2


@dataclass
class SolverParams:
    beta: float = 1.0 / (DESCRIPTOR_LENGTH * 20.0 ** 2)
    threshold: float = 0.7
    max_iters: int = 5
    min_static_rays: int = 2
    epsilon_prior: float = 0.01


@dataclass
class DisparityMap:
    values: np.ndarray   # (h, w) float32
    status: np.ndarray   # (h, w) uint8


@dataclass
class SegmentationState:
    static_bits: np.ndarray  # (h, w) uint32
    valid_bits: np.ndarray   # (h, w) uint32

    def __post_init__(self):
        if (self.static_bits & ~self.valid_bits).any():
            raise ValueError("static rays must be a subset of valid rays")

    @classmethod
    def _device_result(cls, static_bits, valid_bits):
        """Wrap the E-step's outputs without the subset scan (solver.py:78-81):
        the kernels only ever set static bits of valid rays."""
        obj = cls.__new__(cls)
        obj.static_bits = static_bits
        obj.valid_bits = valid_bits
        return obj


@dataclass
class EMStats:
    iterations_run: int = 0
    converged_after: int = None
    mean_energy: list = field(default_factory=list)
    prev_energy: list = field(default_factory=list)
    changed_fraction: list = field(default_factory=list)


def _check_views(k):
    if k > MAX_ENUMERATED_VIEWS:
        raise ValueError(f"mask enumeration is exponential; refusing {k} views "
                         f"(limit {MAX_ENUMERATED_VIEWS})")


def masked_variance(descriptors, mask):
    """solver.py:93-107 (two-pass, fp64), evaluated by `k_masked_variance`."""
    f = np.asarray(descriptors, dtype=np.float64)
    m = np.asarray(mask, dtype=bool)
    if int(m.sum()) < 1:
        raise ValueError("masked variance needs at least one selected ray")
    t = require_cuda()
    k = f.shape[0]
    out = empty((1,), t.float64)
    N.invoke("st_masked_variance", upload(f.reshape(1, k, -1)),
             upload(m.reshape(1, k).astype(np.uint8)), 1, k, out)
    return float(download(out)[0])


def e_step(descriptors, valid, static_prob, params):
    """solver.py:115-157: hard 2^K mask argmax per instance, on the GPU."""
    f = np.asarray(descriptors, dtype=np.float64)
    n, k, _ = f.shape
    _check_views(k)
    t = require_cuda()
    out = empty((n,), t.int32)
    if n:
        p = N.make_params(params, PriorParams())
        N.invoke("st_e_step", upload(f), upload(np.asarray(valid, dtype=bool).astype(np.uint8)),
                 upload(np.asarray(static_prob, dtype=np.float64)), n, k, p, out)
    return download(out).view(np.uint32).copy()


class DisparitySolver:
    """Per-frame device context (solver.py:162-502)."""

    def __init__(self, frame, rig, tri, params=None, prior_params=None):
        self.frame = frame
        self.rig = rig
        self.tri = tri
        self.params = params or SolverParams()
        self.prior_params = prior_params or PriorParams()
        self.height, self.width = frame.shape
        self.num_views = frame.num_views
        if self.num_views != len(rig):
            raise ValueError("frame view count does not match the rig")
        _check_views(self.num_views)
        self._t = require_cuda()
        self._dev = device_frame(frame, refresh=("priors",))
        self._rig = N.make_rig(rig, self.width, self.height)
        self._p = N.make_params(self.params, self.prior_params)
        self._mu = mu_raster_device(tri, self.width, self.height,
                                    clip_dmax=float(self.prior_params.d_max))
        self._sup_ws = None
        self._frame = None
        self._support_records = 0
        self._build_support()
        self._mu_host = None

    # -- device context -----------------------------------------------------------

    def _build_support(self):
        t = self._t
        pts, disps = self.tri.support_points()
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        disps = np.ascontiguousarray(disps, dtype=np.float64).ravel()
        n = int(disps.size)
        fr = N.StFrame()
        fr.images = self._dev.images.data_ptr()
        fr.priors = self._dev.priors.data_ptr()
        fr.desc = self._dev.desc.data_ptr()
        fr.mu = self._mu.data_ptr()
        nbytes = int(N.lib().st_support_workspace(n, self.width, self.height,
                                                  float(self.prior_params.neighborhood_radius)))
        self._sup_ws = empty((max(nbytes, 1),), t.uint8)
        self._sup_in = (upload(pts) if n else None, upload(disps) if n else None)
        rec = N.C.c_int64(0)
        N.check(N.lib().st_support_build(N.ptr(self._sup_in[0]), N.ptr(self._sup_in[1]), n,
                                         self.width, self.height, self._p, fr,
                                         N.ptr(self._sup_ws), self._sup_ws.numel(), rec,
                                         N.stream_handle()))
        self._support_records = rec.value
        self._frame = fr

    @property
    def mu(self):
        """Clipped surface raster, flat (h*w,) float64 (solver.py:185-186)."""
        if self._mu_host is None:
            self._mu_host = download(self._mu)
        return self._mu_host

    def _pix(self, pix):
        return upload(np.ascontiguousarray(np.asarray(pix, dtype=np.int64).ravel()))

    # -- gathering helpers --------------------------------------------------------

    def gather_rays(self, pix, d):
        t = self._t
        pix = np.asarray(pix, dtype=np.int64).ravel()
        n, k = pix.size, self.num_views
        desc = empty((n, k, DESCRIPTOR_LENGTH), t.float64)
        valid = empty((n, k), t.uint8)
        q = empty((n, k), t.float64)
        if n:
            N.invoke("st_gather_rays", self._frame, self._rig, self._pix(pix),
                     upload(np.asarray(d, dtype=np.float64).ravel()), n, desc, valid, q)
        return download(desc), download(valid).astype(bool), download(q)

    def _energy(self, pix, d, static_bits):
        t = self._t
        pix = np.asarray(pix, dtype=np.int64).ravel()
        n = pix.size
        e = empty((n,), t.float64)
        real = empty((n,), t.uint8)
        if n:
            bits = np.asarray(static_bits, dtype=np.uint32).ravel().view(np.int32)
            N.invoke("st_energy", self._frame, self._rig, self._p, self._pix(pix),
                     upload(np.asarray(d, dtype=np.float64).ravel()), upload(bits), n, e, real)
        return download(e), download(real).astype(bool)

    def pixel_energy(self, u, v, d, static_mask):
        if not np.isscalar(static_mask):
            static_mask = sum(1 << k for k, b in enumerate(static_mask) if b)
        pix = np.array([int(v) * self.width + int(u)], dtype=np.int64)
        e, _ = self._energy(pix, np.array([float(d)]), np.array([static_mask], dtype=np.uint32))
        return float(e[0])

    def pixel_candidates(self, u, v):
        """Candidate disparities of one pixel (host bookkeeping, solver.py:274-282)."""
        mu = float(self.mu[int(v) * self.width + int(u)])
        pts, disps = self.tri.support_points()
        r = self.prior_params.neighborhood_radius
        near = (np.abs(pts[:, 0] - u) <= r) & (np.abs(pts[:, 1] - v) <= r)
        d2 = (pts[near, 0] - u) ** 2 + (pts[near, 1] - v) ** 2
        return candidate_disparities(mu, disps[near][d2 <= r * r], self.prior_params)

    # -- the two steps -------------------------------------------------------------

    def m_step(self, active, static_bits_flat):
        t = self._t
        active = np.asarray(active, dtype=np.int64).ravel()
        n = active.size
        d = empty((n,), t.float64)
        e = empty((n,), t.float64)
        st = empty((n,), t.uint8)
        if n:
            bits = upload(np.asarray(static_bits_flat, dtype=np.uint32).ravel().view(np.int32))
            N.invoke("st_m_step", self._frame, self._rig, self._p, self._pix(active), n, bits,
                     d, e, st)
        return download(d), download(e), download(st)

    def e_step_at(self, active, d_active):
        t = self._t
        active = np.asarray(active, dtype=np.int64).ravel()
        n = active.size
        s = empty((n,), t.int32)
        v = empty((n,), t.int32)
        if n:
            N.invoke("st_e_step_at", self._frame, self._rig, self._p, self._pix(active),
                     upload(np.asarray(d_active, np.float64).ravel()), n, s, v)
        return download(s).view(np.uint32).copy(), download(v).view(np.uint32).copy()

    def initial_masks(self, pix):
        t = self._t
        pix = np.asarray(pix, dtype=np.int64).ravel()
        n = pix.size
        s = empty((n,), t.int32)
        v = empty((n,), t.int32)
        if n:
            N.invoke("st_initial_masks", self._frame, self._rig, self._p, self._pix(pix), n, s,
                     v)
        return download(s).view(np.uint32).copy(), download(v).view(np.uint32).copy()

    # -- full EM loop ------------------------------------------------------------------

    def solve_device(self, dynamic_only=False, active_mask=None, forced_iters=0, reduce=None,
                     timing=False):
        """Run st_solve; returns device tensors + EMStats (no host copies)."""
        t = self._t
        h, w = self.height, self.width
        values = empty((h, w), t.float32)
        status = empty((h, w), t.uint8)
        sbits = empty((h, w), t.int32)
        vbits = empty((h, w), t.int32)
        nbytes = int(N.lib().st_solve_workspace(w, h, self.num_views))
        ws = getattr(self, "_solve_ws", None)
        if ws is None or ws.numel() < nbytes:
            ws = self._solve_ws = empty((nbytes,), t.uint8)
        p = N.make_params(self.params, self.prior_params, forced_iters, timing)
        if reduce is None and active_mask is None and not timing:
            # no host round trip per iteration: the device-side control of
            # st_solve_async (dense) / st_solve_rows (dynamic_only)
            sdev = empty((N.C.sizeof(N.StStats),), t.uint8)
            if dynamic_only:
                N.check(N.lib().st_solve_rows(
                    self._frame, self._rig, p, 1, 0, h, 0, h, N.ptr(values), N.ptr(status),
                    N.ptr(sbits), N.ptr(vbits), N.ptr(sdev), N.ptr(ws), ws.numel(),
                    N.EXCHANGE_FN(), None, 1, None, None, N.stream_handle()))
            else:
                N.invoke("st_solve_async", self._frame, self._rig, p, values, status, sbits,
                         vbits, sdev, ws, ws.numel())
            stats = N.StStats.from_buffer_copy(download(sdev).tobytes())
            stats.support_records = self._support_records
            return (values, status, sbits, vbits), _stats_of(stats)
        stats = N.StStats()
        am = upload(np.asarray(active_mask, dtype=np.uint8).ravel()) if active_mask is not None \
            else None
        cb = N.REDUCE_FN(reduce) if reduce is not None else N.REDUCE_FN()
        N.check(N.lib().st_solve(self._frame, self._rig, p, int(bool(dynamic_only)), N.ptr(am),
                                 N.ptr(values), N.ptr(status), N.ptr(sbits), N.ptr(vbits), stats,
                                 N.ptr(ws), ws.numel(), cb, None, N.stream_handle()))
        stats.support_records = self._support_records
        return (values, status, sbits, vbits), _stats_of(stats)

    def solve(self, dynamic_only=False):
        from .device import download_many
        (values, status, sbits, vbits), stats = self.solve_device(dynamic_only)
        values, status, sbits, vbits = download_many((values, status, sbits, vbits))
        disparity = DisparityMap(values=values, status=status)
        # the E-step only sets static bits of valid rays (no host subset scan)
        seg = SegmentationState._device_result(sbits.view(np.uint32), vbits.view(np.uint32))
        return disparity, seg, stats


def _stats_of(s):
    it = s.iterations_run
    st = EMStats(iterations_run=it,
                 converged_after=None if s.converged_after < 0 else s.converged_after)
    st.mean_energy = [float(s.mean_energy[i]) for i in range(it)]
    n_prev = max(0, it - 1)
    st.prev_energy = [float(s.prev_energy[i]) for i in range(n_prev)]
    st.changed_fraction = [float(s.changed_fraction[i]) for i in range(n_prev)]
    st.active_pixels = int(s.active_pixels)
    st.candidates_total = int(s.candidates_total)
    st.energy_evals = int(s.energy_evals)
    st.hopeless_msteps = int(s.hopeless_msteps)
    st.energy_samples = int(s.energy_samples)
    st.prev_evals = int(s.prev_evals)
    st.msteps = int(s.msteps)
    st.esteps = int(s.esteps)
    st.support_records = int(s.support_records)
    st.kernel_ms = [float(x) for x in s.kernel_ms]
    st.kernel_launches = [int(x) for x in s.kernel_launches]
    return st


def em_solve(frame, rig, tri, params=None, prior_params=None, dynamic_only=False):
    """solver.py:505-508."""
    solver = DisparitySolver(frame, rig, tri, params=params, prior_params=prior_params)
    return solver.solve(dynamic_only=dynamic_only)
