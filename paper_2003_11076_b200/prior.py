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


class TriDevice:
    """A TriangulationPrior on the device: vertices, planes, the Qhull walk
    tables `st_mu_raster` replays, and the support list."""

    def __init__(self, tri):
        from .device import upload
        dl = delaunay_of(tri)
        f64 = lambda a, *s: upload(np.ascontiguousarray(a, dtype=np.float64).reshape(*s))  # noqa
        pts = np.asarray(tri.points, dtype=np.float64).reshape(-1, 2)
        self.n_pts = pts.shape[0]
        self.points = f64(pts, -1, 2)
        self.disparities = f64(tri.disparities, -1)
        self.triangles = upload(np.ascontiguousarray(tri.triangles, dtype=np.int32).reshape(-1, 3))
        self.n_tri = int(self.triangles.shape[0])
        self.planes = f64(tri.planes, -1, 3)
        self.neighbors = upload(np.ascontiguousarray(dl.neighbors, dtype=np.int32))
        self.transform = f64(dl.transform, -1, 3, 2)
        self.equations = f64(dl.equations, -1, 4)
        sp, sd = tri.support_points()
        sp = np.asarray(sp, dtype=np.float64).reshape(-1, 2)
        self.n_sup = int(sp.shape[0])
        self.sup_uv = f64(sp, -1, 2) if self.n_sup else None
        self.sup_d = f64(sd, -1) if self.n_sup else None
        s = N.StTri()
        s.points, s.disparities = self.points.data_ptr(), self.disparities.data_ptr()
        s.simplices, s.planes = self.triangles.data_ptr(), self.planes.data_ptr()
        s.neighbors, s.transform = self.neighbors.data_ptr(), self.transform.data_ptr()
        s.equations = self.equations.data_ptr()
        s.n_pts, s.n_tri = self.n_pts, self.n_tri
        s.paraboloid_scale = float(dl.paraboloid_scale)
        s.paraboloid_shift = float(dl.paraboloid_shift)
        for i in range(2):
            s.min_bound[i] = float(dl.min_bound[i])
            s.max_bound[i] = float(dl.max_bound[i])
        self.st = s

    @property
    def nbytes(self):
        return self.n_pts * 24 + self.n_tri * (12 + 24 + 12 + 48 + 32) + self.n_sup * 24


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
    from scipy.spatial import Delaunay, QhullError, cKDTree
    if not points:
        raise ValueError("degenerate support set: no support points")
    coords = np.array([[p.u, p.v] for p in points], dtype=np.float64)
    disps = np.array([p.d for p in points], dtype=np.float64)
    corners = np.array([[0.0, 0.0], [width - 1.0, 0.0], [0.0, height - 1.0],
                        [width - 1.0, height - 1.0]])
    taken = {(int(c[0]), int(c[1])) for c in coords}
    missing = [c for c in corners if (int(c[0]), int(c[1])) not in taken]
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
    verts = coords[tris]
    mats = np.concatenate([verts, np.ones((verts.shape[0], 3, 1))], axis=2)
    try:
        planes = np.linalg.solve(mats, disps[tris][:, :, None])[:, :, 0]
    except np.linalg.LinAlgError:
        raise ValueError("degenerate support set: zero-area triangle") from None
    return TriangulationPrior(points=coords, disparities=disps, triangles=tris, planes=planes,
                              num_anchors=n_anchor, _lookup=dl)


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
