"""Piecewise-planar disparity prior: parameters, triangulated surface, densities.

The support-point harvest and the Delaunay triangulation (prior.py:51-360)
are the upstream stage of the accelerated path and stay on the host
(`triangulate` uses scipy Qhull like the reference).  What the solver
consumes every frame runs on the device: the dense surface raster mu
(`TriangulationPrior.disparity_map` -> `st_mu_raster`) and the support
candidate lists (`st_support_build`).
"""

from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass
class PriorParams:
    """prior.py:33-40."""
    sigma: float = 2.0
    gamma: float = 0.05
    d_max: float = 64.0
    neighborhood_radius: float = 20.0


@dataclass
class SupportPoint:
    u: int
    v: int
    d: float
    source_view: int


def delaunay_of(tri):
    """The scipy Delaunay lookup behind a TriangulationPrior (rebuilt if absent)."""
    dl = getattr(tri, "_lookup", None)
    if dl is None or not hasattr(dl, "neighbors"):
        from scipy.spatial import Delaunay
        dl = Delaunay(np.asarray(tri.points, dtype=np.float64))
        if not np.array_equal(dl.simplices.astype(np.int32),
                              np.asarray(tri.triangles, dtype=np.int32)):
            raise ValueError("triangles are not the Delaunay triangulation of the points")
        try:
            tri._lookup = dl
        except AttributeError:
            pass
    return dl


class _Staging:
    """Two reusable page-locked staging buffers for the triangulation tables."""

    def __init__(self):
        self.bufs = [None, None]
        self.events = [None, None]
        self.turn = 0

    def take(self, nbytes):
        import torch
        i = self.turn
        self.turn ^= 1
        if self.events[i] is not None:
            self.events[i].synchronize()  # its previous upload has left
        if self.bufs[i] is None or self.bufs[i].numel() < nbytes:
            self.bufs[i] = torch.empty(max(nbytes, 1 << 20) * 5 // 4, dtype=torch.uint8,
                                       pin_memory=True)
        return i, self.bufs[i]

    def mark(self, i):
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.events[i] = ev


_STAGING = _Staging()


def _integral_coords(points):
    """Integer pixel coordinates below 2^24 (st_tri_tables' precondition)."""
    pts = np.asarray(points)
    return bool(pts.size == 0 or (np.all(np.floor(pts) == pts)
                                  and np.abs(pts).max() < float(1 << 24)))


class TriDevice:
    """A TriangulationPrior on the device: vertices, the Qhull walk tables
    `st_mu_raster` replays and the support list, packed into one pinned
    staging buffer and sent with a single asynchronous copy.  The two LAPACK
    tables -- planes (prior.py:351-357) and the barycentric transforms -- are
    recomputed on the device by st_tri_tables with the host libraries'
    operation order (host tables are only shipped for non-integer vertex
    coordinates, outside st_tri_tables' exactness precondition)."""

    def __init__(self, tri, slot=None):
        """slot (optional): an object with reusable `tri_stage` (pinned) and
        `tri_buf` (device) tensors -- a FramePipeline slot whose previous
        frame has finished -- instead of the shared staging ring and a fresh
        device allocation."""
        import torch
        from .device import dev
        dl = delaunay_of(tri)
        sp, sd = tri.support_points()
        sp = np.asarray(sp, dtype=np.float64).reshape(-1, 2)
        points = np.asarray(tri.points, dtype=np.float64).reshape(-1, 2)
        self.device_tables = _integral_coords(points)
        n_tri = int(np.asarray(tri.triangles).shape[0])
        disps = np.asarray(tri.disparities, dtype=np.float64).reshape(-1)
        sd = np.asarray(sd, dtype=np.float64).reshape(-1)
        # the support list is the leading rows of the vertex list (prior.py:312-315):
        # alias it on the device instead of sending it twice
        self.sup_alias = (sp.shape[0] <= points.shape[0] and sd.shape[0] == sp.shape[0]
                          and sp.ctypes.data == points.ctypes.data
                          and sp.strides == points.strides
                          and sd.ctypes.data == disps.ctypes.data
                          and sd.strides == disps.strides)
        parts = [
            ("points", points),
            ("disparities", disps),
            ("triangles", np.asarray(tri.triangles, dtype=np.int32).reshape(-1, 3)),
            ("neighbors", np.asarray(dl.neighbors, dtype=np.int32).reshape(-1, 3)),
            ("equations", np.asarray(dl.equations, dtype=np.float64).reshape(-1, 4)),
        ]
        if not self.sup_alias:
            parts += [("sup_uv", sp), ("sup_d", sd)]
        if not self.device_tables:
            parts += [("planes", np.asarray(tri.planes, dtype=np.float64).reshape(-1, 3)),
                      ("transform", np.asarray(dl.transform, dtype=np.float64).reshape(-1, 3, 2))]
        offs, total = [], 0
        for _, a in parts:
            offs.append(total)
            total += (a.nbytes + 255) & ~255
        dev_total = total
        if self.device_tables:  # device-only tail: planes, transform, flags
            t_planes = dev_total
            dev_total += (n_tri * 24 + 255) & ~255
            t_transform = dev_total
            dev_total += (n_tri * 48 + 255) & ~255
            t_flags = dev_total
            dev_total += 256
        if slot is None:
            i, stage = _STAGING.take(total)
        else:
            ev = getattr(slot, "tri_stage_event", None)
            if ev is not None:
                ev.synchronize()  # the slot's previous upload has left the staging buffer
            if getattr(slot, "tri_stage", None) is None or slot.tri_stage.numel() < total:
                slot.tri_stage = torch.empty(max(total, 1 << 20) * 5 // 4, dtype=torch.uint8,
                                             pin_memory=True)
            stage = slot.tri_stage
        # one native gather into the pinned staging block (the GIL is released
        # for it: a stream's other host thread keeps enqueueing meanwhile)
        arrs = [np.ascontiguousarray(a) for _, a in parts]
        srcs, goffs, sizes, n_parts = N.gather_args(arrs, offs)
        N.check(N.lib().st_host_gather(N.C.c_void_p(stage.data_ptr()), srcs, goffs, sizes,
                                       n_parts))
        if slot is None:
            self.buffer = torch.empty(max(dev_total, 1), dtype=torch.uint8, device=dev())
        else:
            if getattr(slot, "tri_buf", None) is None or slot.tri_buf.numel() < dev_total:
                slot.tri_buf = torch.empty(max(dev_total, 1 << 20) * 5 // 4, dtype=torch.uint8,
                                           device=dev())
            self.buffer = slot.tri_buf
        self.buffer[:total].copy_(stage[:total], non_blocking=True)
        if slot is None:
            _STAGING.mark(i)
        else:
            slot.tri_stage_event = torch.cuda.Event()
            slot.tri_stage_event.record(torch.cuda.current_stream())
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32}
        for (name, a), o in zip(parts, offs):
            view = self.buffer[o:o + a.nbytes].view(tdt[a.dtype]).reshape(a.shape)
            setattr(self, name, view if a.size else None)
        self.n_pts = points.shape[0]
        self.n_tri = n_tri
        self.n_sup = int(sp.shape[0])
        if self.sup_alias:
            self.sup_uv = self.points[:self.n_sup] if self.n_sup else None
            self.sup_d = self.disparities[:self.n_sup] if self.n_sup else None
        if self.device_tables:
            self.planes = self.buffer[t_planes:t_planes + n_tri * 24].view(torch.float64)
            self.transform = self.buffer[t_transform:t_transform + n_tri * 48].view(torch.float64)
            self.flags = self.buffer[t_flags:t_flags + 4].view(torch.int32)
            self.flags.zero_()
        else:
            self.flags = None
        s = N.StTri()
        s.points, s.disparities = self.points.data_ptr(), self.disparities.data_ptr()
        s.simplices, s.planes = self.triangles.data_ptr(), self.planes.data_ptr()
        s.neighbors, s.transform = self.neighbors.data_ptr(), self.transform.data_ptr()
        s.equations = self.equations.data_ptr()
        s.n_pts, s.n_tri = self.n_pts, self.n_tri
        s.paraboloid_scale = float(dl.paraboloid_scale)
        s.paraboloid_shift = float(dl.paraboloid_shift)
        # prior.py:290 `points.mean(axis=0)` (the off-hull nudge target).  With
        # integer vertex coordinates the column sums are exact in any order, so
        # k_mu_nudge computes it on the device when it is needed (NaN here);
        # otherwise numpy's value is shipped.
        cen = ((np.nan, np.nan) if self.device_tables
               else np.asarray(points, dtype=np.float64).mean(axis=0))
        for k in range(2):
            s.min_bound[k] = float(dl.min_bound[k])
            s.max_bound[k] = float(dl.max_bound[k])
            s.centroid[k] = float(cen[k])
        self.st = s
        if self.device_tables:
            N.invoke("st_tri_tables", s, self.planes, self.transform, self.flags)

    def check(self):
        """Raise the reference's triangulate error if a plane system was
        singular (numpy LinAlgError at prior.py:355-357).  Synchronises."""
        if self.flags is not None and int(self.flags.item()) & 1:
            raise ValueError("degenerate support set: zero-area triangle")

    @property
    def nbytes(self):
        return self.n_pts * 24 + self.n_tri * (12 + 12 + 32) + (
            0 if self.sup_alias else self.n_sup * 24) + (
            0 if self.device_tables else self.n_tri * 72)

    def tensors(self):
        return [self.buffer]


def mu_raster_device(tri, width, height, clip_dmax=0.0, tri_dev=None):
    """Dense surface raster on the device (torch CUDA float64 (h*w,))."""
    from .device import empty, require_cuda
    t = require_cuda()
    td = tri_dev or TriDevice(tri)
    mu = empty((height * width,), t.float64)
    ws = empty((int(N.lib().st_mu_raster_workspace(width, height, td.n_tri)),), t.uint8)
    N.invoke("st_mu_raster", td.st, width, height, float(clip_dmax), mu, ws, ws.numel())
    return mu


@dataclass
class TriangulationPrior:
    """Piecewise-linear disparity surface over the reference image (prior.py:265-315)."""

    points: np.ndarray
    disparities: np.ndarray
    triangles: np.ndarray
    planes: np.ndarray
    num_anchors: int
    _lookup: object = None

    def interpolate(self, u, v):
        """Surface value at arbitrary continuous points (host, scipy lookup)."""
        from scipy.spatial import Delaunay, cKDTree
        if self._lookup is None:
            self._lookup = Delaunay(self.points)
        u = np.atleast_1d(np.asarray(u, dtype=np.float64))
        v = np.atleast_1d(np.asarray(v, dtype=np.float64))
        q = np.stack([u, v], axis=1)
        simplex = self._lookup.find_simplex(q)
        miss = simplex < 0
        if miss.any():
            c = self.points.mean(axis=0)
            simplex[miss] = self._lookup.find_simplex(q[miss] + 1e-9 * (c - q[miss]))
            miss = simplex < 0
        out = np.empty(u.shape[0])
        ok = ~miss
        if ok.any():
            pl = self.planes[simplex[ok]]
            out[ok] = pl[:, 0] * u[ok] + pl[:, 1] * v[ok] + pl[:, 2]
        if miss.any():
            _, near = cKDTree(self.points).query(q[miss])
            out[miss] = self.disparities[near]
        return out

    def disparity_map(self, width, height):
        """Dense (h, w) float64 raster at pixel centres, computed on the GPU."""
        from .device import download
        return download(mu_raster_device(self, width, height)).reshape(height, width)

    def support_points(self):
        n = self.points.shape[0] - self.num_anchors
        return self.points[:n], self.disparities[:n]


def triangulate(points, width, height):
    """Delaunay surface over support points + corner anchors (prior.py:318-360).

    Upstream stage, host side (scipy Qhull), kept API-compatible.
    """
    if not points:
        raise ValueError("degenerate support set: no support points")
    return triangulate_arrays([p.u for p in points], [p.v for p in points],
                              [p.d for p in points], width, height)


def triangulate_arrays(u, v, d, width, height, planes=True):
    """triangulate over (u, v, d) arrays (same arithmetic as prior.py:318-360).

    planes=False skips the host plane solve (TriDevice recomputes the planes
    on the device; .planes is then None and a zero-area triangle surfaces
    through TriDevice.check)."""
    from scipy.spatial import Delaunay, QhullError, cKDTree
    if len(u) == 0:
        raise ValueError("degenerate support set: no support points")
    coords = np.stack([np.asarray(u, dtype=np.float64), np.asarray(v, dtype=np.float64)], axis=1)
    disps = np.asarray(d, dtype=np.float64).copy()
    corners = np.array([[0.0, 0.0], [width - 1.0, 0.0], [0.0, height - 1.0],
                        [width - 1.0, height - 1.0]])
    # prior.py:336-337 {(int(u), int(v))} membership, vectorised (int() truncates)
    ci = np.trunc(coords)
    missing = [c for c in corners
               if not np.any((ci[:, 0] == np.trunc(c[0])) & (ci[:, 1] == np.trunc(c[1])))]
    n_anchor = 0
    if missing:
        _, nearest = cKDTree(coords).query(np.array(missing))
        coords = np.concatenate([coords, np.array(missing)])
        disps = np.concatenate([disps, disps[nearest]])
        n_anchor = len(missing)
    try:
        dl = Delaunay(coords)
    except QhullError as exc:
        raise ValueError(f"degenerate support set: {exc}") from None
    tris = dl.simplices.astype(np.int32)
    if not planes:
        return TriangulationPrior(points=coords, disparities=disps, triangles=tris, planes=None,
                                  num_anchors=n_anchor, _lookup=dl)
    verts = coords[tris]
    mats = np.concatenate([verts, np.ones((verts.shape[0], 3, 1))], axis=2)
    try:
        planes = np.linalg.solve(mats, disps[tris][:, :, None])[:, :, 0]
    except np.linalg.LinAlgError:
        raise ValueError("degenerate support set: zero-area triangle") from None
    return TriangulationPrior(points=coords, disparities=disps, triangles=tris, planes=planes,
                              num_anchors=n_anchor, _lookup=dl)


# prior.py:25-30
SUPPORT_STRIDE = 5
MIN_TEXTURE = 25.0
UNIQUENESS_RATIO = 0.9
SECOND_BEST_EXCLUSION = 1.0
LEFT_RIGHT_TOL = 1.0


def _grid_len(d_max):
    """len(np.arange(0.5, d_max + 0.25, 0.5)) -- the scan grid (prior.py:114)."""
    return int(len(np.arange(0.5, float(d_max) + 0.25, 0.5)))


def harvest_device(frame, rig, params=None, threshold=0.7, stride=SUPPORT_STRIDE,
                   min_texture=MIN_TEXTURE):
    """collect_support up to deduplicate, on the GPU (st_harvest).

    Returns host arrays (u int32, v int32, d float64, source_view int32) of
    the collected points in the reference's collection order (views in
    order, each view's matches in raster order, prior.py:245-259).
    """
    from .device import download, empty, require_cuda
    from .frame import device_frame
    t = require_cuda()
    params = params or PriorParams()
    d = device_frame(frame)
    K, H, W = d.K, d.H, d.W
    if len(rig) != K:
        raise ValueError("frame view count does not match the rig")
    cams = N.make_cams(rig, W, H)
    lib = N.lib()
    cap = max(int(lib.st_harvest_capacity(K, W, H, int(stride))), 1)
    ws = empty((max(int(lib.st_harvest_workspace(K, W, H, int(stride))), 1),), t.uint8)
    ou = empty((cap,), t.int32)
    ov = empty((cap,), t.int32)
    od = empty((cap,), t.float64)
    osrc = empty((cap,), t.int32)
    cnt = empty((1,), t.int64)
    N.invoke("st_harvest", d.desc, d.priors, cams, float(params.d_max), _grid_len(params.d_max),
             float(threshold), int(stride), float(min_texture), ou, ov, od, osrc, cnt, None, ws,
             ws.numel())
    n = int(cnt.item())
    return download(ou[:n]), download(ov[:n]), download(od[:n]), download(osrc[:n])


def deduplicate_arrays(u, v, d, src, ref_index, width=None, height=None):
    """deduplicate (prior.py:183-212) over arrays; returns the kept indices
    in the final raster order (native host code, st_support_dedup)."""
    import ctypes as C
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.float64)
    src = np.ascontiguousarray(src, dtype=np.int32)
    n = u.shape[0]
    if n and (u.min() < 0 or v.min() < 0):
        raise ValueError("support points must have non-negative pixel coordinates")
    w = int(width) if width is not None else (int(u.max()) + 1 if n else 1)
    h = int(height) if height is not None else (int(v.max()) + 1 if n else 1)
    keep = np.empty(max(n, 1), dtype=np.int64)
    nk = C.c_int64(0)
    vp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    N.check(N.lib().st_support_dedup(vp(u), vp(v), vp(d), vp(src), n, int(ref_index), w, h,
                                     vp(keep), C.byref(nk)))
    return keep[:nk.value]


def deduplicate(points, ref_index):
    """prior.py:183-212 on SupportPoint lists."""
    if not points:
        return []
    keep = deduplicate_arrays([p.u for p in points], [p.v for p in points],
                              [p.d for p in points], [p.source_view for p in points], ref_index)
    return [points[i] for i in keep]


def collect_support(frame, rig, params, threshold, stride=SUPPORT_STRIDE,
                    min_texture=MIN_TEXTURE):
    """Full support-point harvest for one frame (prior.py:233-260): detection,
    matching, left-right check and reprojection on the GPU, deduplication in
    native host code.  Returns the reference's SupportPoint list."""
    u, v, d, src = harvest_device(frame, rig, params, threshold, stride, min_texture)
    h, w = frame.shape if hasattr(frame, "shape") else frame.images[0].shape[:2]
    keep = deduplicate_arrays(u, v, d, src, rig.ref_index, w, h)
    return [SupportPoint(u=int(u[i]), v=int(v[i]), d=float(d[i]), source_view=int(src[i]))
            for i in keep]


def prior_log_density(d, mu, params):
    """log(gamma + exp(-(d - mu)^2 / (2 sigma^2))) (prior.py:365-370)."""
    z = (np.asarray(d, dtype=np.float64) - np.asarray(mu, dtype=np.float64)) / params.sigma
    return np.log(params.gamma + np.exp(-0.5 * z * z))


def candidate_disparities(mu, neighbor_disparities, params):
    """Band + neighbours + coarse sweep, clipped to (0, d_max], unique (prior.py:373-386)."""
    jm = int(np.floor(2.0 * params.sigma / 0.5 + 1e-12))
    band = mu + 0.5 * np.arange(-jm, jm + 1)
    coarse = np.arange(1.0, params.d_max + 1e-9, 4.0)
    vals = np.concatenate([band, np.asarray(neighbor_disparities, dtype=np.float64).ravel(),
                           coarse])
    return np.unique(vals[(vals > 0.0) & (vals <= params.d_max)])


def dump_support_csv(points, path):
    with open(path, "w", encoding="ascii") as fh:
        fh.write("u,v,d,source_view\n")
        for p in points:
            fh.write(f"{p.u},{p.v},{p.d!r},{p.source_view}\n")


def dump_triangulation_obj(tri, path):
    with open(path, "w", encoding="ascii") as fh:
        for (u, v), d in zip(tri.points, tri.disparities):
            fh.write(f"v {u!r} {v!r} {d!r}\n")
        for t in tri.triangles:
            fh.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")
