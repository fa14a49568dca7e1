"""numpy restatement of the reference EM background-reconstruction hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import this).

Reference files (relative to /root/reference/pkg/src/seethrough/):
  sampling.py  -- bilinear gather (fp32 tap difference, fp64 lerp)
  features.py  -- gray, biased Sobel, 16-byte ring descriptors
  geometry.py  -- disparity-parameterised homography warp
  solver.py    -- candidate-set M-step, 2^K mask E-step, EM loop
  refocus.py   -- Eq. 2 static-ray average, provenance, clipped median
  prior.py     -- log prior density, candidate sets, mu raster

The arithmetic order of every floating-point expression follows the
reference (left-to-right evaluation, separate roundings, numpy's pairwise
16-channel sum in the M-step energy, sequential sums in the E-step), so the
oracle reproduces the reference bit for bit on the golden fixtures.
"""

from dataclasses import dataclass

import numpy as np

DESC_LEN = 16                    # features.py:19
DESC_MARGIN = 3                  # features.py:20
# features.py:24 -- (du, dv) ring; entry 2i = gx, 2i+1 = gy at offset i
RING = ((0, -2), (1, -1), (2, 0), (1, 1), (0, 2), (-1, 1), (-2, 0), (-1, -1))
VARIANCE_CEILING = float(DESC_LEN) * 127.5 ** 2   # solver.py:44
MAX_VIEWS = 12                   # solver.py:46
STATUS_VALID, STATUS_LOW_TEXTURE, STATUS_NO_STATIC_EVIDENCE = 0, 1, 2  # solver.py:48-50
PROV_FALLBACK, PROV_COPIED, PROV_REFOCUSED = 0, 128, 255                # refocus.py:19-21

_ROWS = 1 << 17          # pixels per vectorised energy batch
_ESTEP_ROWS = 1 << 14    # pixels per vectorised E-step batch


@dataclass
class OracleParams:
    """SolverParams (solver.py:56-62) + PriorParams (prior.py:33-40)."""
    beta: float = 1.0 / (DESC_LEN * 20.0 ** 2)
    threshold: float = 0.7
    max_iters: int = 5
    min_static_rays: int = 2
    epsilon_prior: float = 0.01
    sigma: float = 2.0
    gamma: float = 0.05
    d_max: float = 64.0
    neighborhood_radius: float = 20.0


# -- L1 primitives -----------------------------------------------------------

def numpy_sum_order(values):
    """np.add.reduce of a contiguous float64 array, restated: 0.0 plus
    numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) -- blocks
    of n <= 128 with eight strided accumulators combined as
    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail in order (n < 8: a
    running sum from 0.0), larger blocks split at n/2 rounded down to a
    multiple of 8.  This is the order solver.py:466/471 `finite.mean()` sums
    in; the device statistics (st_mean.cu) replay it.  Pure Python: small n."""
    a = [float(x) for x in np.asarray(values, dtype=np.float64).ravel()]

    def pw(lo, n):
        if n < 8:
            r = 0.0
            for i in range(n):
                r += a[lo + i]
            return r
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)

    return 0.0 + pw(0, len(a))


def warp(A, b, u, v, d):
    """geometry.py:204-219: h = A (u, v, 1) + d b, evaluated left to right."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    hx = A[0][0] * u + A[0][1] * v + A[0][2] + d * b[0]
    hy = A[1][0] * u + A[1][1] * v + A[1][2] + d * b[1]
    hz = A[2][0] * u + A[2][1] * v + A[2][2] + d * b[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        return hx / hz, hy / hz, hz > 0


def bilinear(plane, u, v):
    """sampling.py:21-55 on an (h, w, c) plane of any real dtype.

    Tap differences are taken in float32 (the reference samples float32
    planes), the lerp weights and accumulation in float64.  The reference's
    axis-aligned shortcuts are bit-identical to this general form (a zero
    weight multiplies a finite difference), so only the general form is kept.
    """
    plane = np.asarray(plane)
    if plane.ndim == 2:
        plane = plane[:, :, None]
    h, w, c = plane.shape
    flat = plane.reshape(h * w, c).astype(np.float32)
    u = np.clip(np.nan_to_num(np.asarray(u, np.float64), nan=0.0, posinf=0.0, neginf=0.0), 0.0, w - 1.0)
    v = np.clip(np.nan_to_num(np.asarray(v, np.float64), nan=0.0, posinf=0.0, neginf=0.0), 0.0, h - 1.0)
    iu = np.minimum(np.floor(u), w - 2.0) if w > 1 else np.zeros_like(u)
    iv = np.minimum(np.floor(v), h - 2.0) if h > 1 else np.zeros_like(v)
    fu = (u - iu)[:, None]
    fv = (v - iv)[:, None]
    base = iv.astype(np.int64) * w + iu.astype(np.int64)
    du = 1 if w > 1 else 0
    dv = w if h > 1 else 0
    t0 = flat[base]
    t1 = flat[base + du]
    b0 = flat[base + dv]
    b1 = flat[base + du + dv]
    top = t0 + fu * (t1 - t0)
    bot = b0 + fu * (b1 - b0)
    return top + fv * (bot - top)


def gray_of(img):
    """features.py:29-36: ITU-601 weights in fp64, rint half-even."""
    img = np.asarray(img)
    if img.ndim == 2:
        return img.astype(np.uint8, copy=False)
    g = img[..., 0] * 0.299 + img[..., 1] * 0.587 + img[..., 2] * 0.114
    return np.rint(g).astype(np.uint8)


def sobel_of(gray):
    """features.py:39-58: edge-replicated 3x3 Sobel, clip(rint(128 + g/4))."""
    g = np.pad(np.asarray(gray, dtype=np.int32), 1, mode="edge")
    h, w = g.shape[0] - 2, g.shape[1] - 2
    sx = g[0:h, :] + 2 * g[1:h + 1, :] + g[2:h + 2, :]       # vertical smoothing
    gx = sx[:, 2:] - sx[:, :-2]
    sy = g[:, 0:w] + 2 * g[:, 1:w + 1] + g[:, 2:w + 2]       # horizontal smoothing
    gy = sy[2:, :] - sy[:-2, :]
    enc = lambda r: np.clip(np.rint(128.0 + r / 4.0), 0, 255).astype(np.uint8)  # noqa: E731
    return enc(gx), enc(gy)


def descriptors_of(image):
    """features.py:81-104: (h, w, 16) uint8 ring descriptors, 128 off-image."""
    gray = gray_of(image)
    h, w = gray.shape
    if h < 2 * DESC_MARGIN + 1 or w < 2 * DESC_MARGIN + 1:
        raise ValueError("image too small for descriptors")
    gx, gy = sobel_of(gray)
    out = np.full((h, w, DESC_LEN), 128, dtype=np.uint8)
    for i, (ou, ov) in enumerate(RING):
        ys = slice(max(-ov, 0), h - max(ov, 0))
        xs = slice(max(-ou, 0), w - max(ou, 0))
        ys_src = slice(max(ov, 0), h + min(ov, 0))
        xs_src = slice(max(ou, 0), w + min(ou, 0))
        out[ys, xs, 2 * i] = gx[ys_src, xs_src]
        out[ys, xs, 2 * i + 1] = gy[ys_src, xs_src]
    return out


def log_prior(d, mu, sigma, gamma):
    """prior.py:365-370: log(gamma + exp(-z^2/2)), z = (d - mu)/sigma."""
    z = (np.asarray(d, np.float64) - np.asarray(mu, np.float64)) / sigma
    return np.log(gamma + np.exp(-0.5 * z * z))


# -- E-step ------------------------------------------------------------------

def mask_order(k):
    """solver.py:110-112: larger popcount first, then smaller encoding."""
    return sorted(range(1 << k), key=lambda m: (-bin(m).count("1"), m))


def e_step_scores(desc, valid, q, p):
    """All 2^K mask scores in mask_order (solver.py:115-157), (n, M) float64."""
    f = np.asarray(desc, dtype=np.float64)
    n, k, _ = f.shape
    if k > MAX_VIEWS:
        raise ValueError(f"mask enumeration is exponential; refusing {k} views "
                         f"(limit {MAX_VIEWS})")
    order = np.array(mask_order(k), dtype=np.uint32)
    sel = ((order[:, None] >> np.arange(k)[None, :]) & 1).astype(np.float64)  # (M, K)
    npop = sel.sum(axis=1)
    short = npop < p.min_static_rays
    nsafe = np.maximum(npop, 1.0)
    qc = np.clip(np.asarray(q, dtype=np.float64), p.epsilon_prior, 1.0 - p.epsilon_prior)
    l1 = np.log(qc)
    l0 = np.log(1.0 - qc)
    bad = ~np.asarray(valid, dtype=bool)
    out = np.empty((n, order.size))
    for lo in range(0, n, _ESTEP_ROWS):
        hi = min(lo + _ESTEP_ROWS, n)
        fb = f[lo:hi]
        # sums over the selected views run in view order (BLAS dgemm with a 0/1 operand)
        a1 = np.tensordot(fb, sel, axes=([1], [1]))
        a2 = np.tensordot(fb * fb, sel, axes=([1], [1]))
        var = np.clip((a2 - a1 * a1 / nsafe).sum(axis=1) / nsafe, 0.0, None)
        var[:, short] = VARIANCE_CEILING
        s = l1[lo:hi] @ sel.T + l0[lo:hi] @ (1.0 - sel.T) - p.beta * var
        s[bad[lo:hi].astype(np.float64) @ sel.T > 0] = -np.inf
        out[lo:hi] = s
    return out, order


def e_step(desc, valid, q, p):
    """solver.py:115-157: hard argmax over masks in mask_order."""
    s, order = e_step_scores(desc, valid, q, p)
    return order[np.argmax(s, axis=1)] if s.shape[0] else np.zeros(0, np.uint32)


# -- mu raster ---------------------------------------------------------------

def mu_raster(points, disparities, triangles, planes, width, height):
    """prior.py:276-310: containing-triangle plane at pixel centres.

    Rebuilds the scipy Delaunay lookup from the same vertices (deterministic,
    asserted to reproduce `triangles`), nudges off-hull queries by 1e-9 toward
    the centroid, and falls back to the nearest vertex.
    """
    from scipy.spatial import Delaunay, cKDTree
    pts = np.asarray(points, dtype=np.float64)
    lookup = Delaunay(pts)
    if not np.array_equal(lookup.simplices.astype(np.int32), np.asarray(triangles, np.int32)):
        raise AssertionError("Delaunay rebuild does not reproduce the triangulation")
    uu, vv = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
    u = uu.ravel()
    v = vv.ravel()
    qpts = np.stack([u, v], axis=1)
    simplex = lookup.find_simplex(qpts)
    miss = simplex < 0
    if miss.any():
        c = pts.mean(axis=0)
        simplex[miss] = lookup.find_simplex(qpts[miss] + 1e-9 * (c - qpts[miss]))
        miss = simplex < 0
    out = np.empty(u.size)
    ok = ~miss
    pl = np.asarray(planes)[simplex[ok]]
    out[ok] = pl[:, 0] * u[ok] + pl[:, 1] * v[ok] + pl[:, 2]
    if miss.any():
        _, near = cKDTree(pts).query(qpts[miss])
        out[miss] = np.asarray(disparities)[near]
    return out.reshape(height, width)


# -- dense solver ------------------------------------------------------------

class OracleSolver:
    """Restates DisparitySolver (solver.py:162-502).

    images: K x (h, w, 3) uint8; priors: K x (h, w) float32;
    warp_a (K, 3, 3), warp_b (K, 3) float64 (geometry.py:156-172);
    mu: (h, w) surface raster BEFORE clipping (prior.py:306-310);
    support_uv (n, 2), support_d (n,) -- TriangulationPrior.support_points().
    """

    def __init__(self, images, priors, warp_a, warp_b, ref_index, mu,
                 support_uv, support_d, params=None, descriptors=None):
        self.p = params or OracleParams()
        self.K = len(images)
        if self.K > MAX_VIEWS:
            raise ValueError(f"mask enumeration is exponential; refusing {self.K} views "
                             f"(limit {MAX_VIEWS})")
        self.h, self.w = images[0].shape[:2]
        self.images = [np.asarray(im) for im in images]
        self.priors = [np.asarray(pr, dtype=np.float32) for pr in priors]
        self.A = np.asarray(warp_a, dtype=np.float64)
        self.b = np.asarray(warp_b, dtype=np.float64)
        self.ref = int(ref_index)
        self.desc = descriptors if descriptors is not None else [descriptors_of(im) for im in self.images]
        # flat float32 planes, as DescriptorMap.flat32 / flatten_channels hold them
        self._dflat = [d.reshape(-1, DESC_LEN).astype(np.float32) for d in self.desc]
        self._pflat = [pr.reshape(-1).astype(np.float32) for pr in self.priors]
        self.mu = np.clip(np.asarray(mu, np.float64), 1e-6, self.p.d_max).ravel()  # solver.py:185-186
        jm = int(np.floor(2.0 * self.p.sigma / 0.5 + 1e-12))                      # solver.py:187
        band = 0.5 * np.arange(-jm, jm + 1)
        self.band = band[np.lexsort((band, np.abs(band)))]                         # nearest first
        self.coarse = np.arange(1.0, self.p.d_max + 1e-9, 4.0)                     # solver.py:192
        self.support_uv = np.asarray(support_uv, dtype=np.float64).reshape(-1, 2)
        self.support_d = np.asarray(support_d, dtype=np.float64).ravel()

    # -- sampling -----------------------------------------------------------

    def _lerp_rows(self, flat, c, pu, pv):
        """bilinear() on a flat float32 (h*w, c) plane; pu/pv already in range."""
        w, h = self.w, self.h
        u = np.clip(pu, 0.0, w - 1.0)
        v = np.clip(pv, 0.0, h - 1.0)
        iu = np.minimum(np.floor(u), w - 2.0)
        iv = np.minimum(np.floor(v), h - 2.0)
        fu = (u - iu)[:, None]
        fv = (v - iv)[:, None]
        base = iv.astype(np.int64) * w + iu.astype(np.int64)
        f2 = flat.reshape(-1, c)
        # zero-weight taps contribute exactly nothing, so (like sampling.py:40-55)
        # skip their gathers when a whole batch sits on integer columns / rows
        lerp_u = bool(fu.any())
        t0 = f2[base]
        top = t0 + fu * (f2[base + 1] - t0) if lerp_u else t0.astype(np.float64)
        if not fv.any():
            return top
        b0 = f2[base + w]
        bot = b0 + fu * (f2[base + w + 1] - b0) if lerp_u else b0.astype(np.float64)
        return top + fv * (bot - top)

    def ray(self, pix, d, k):
        """solver.py:197-204: warp + descriptor-support margin test."""
        u = (pix % self.w).astype(np.float64)
        v = (pix // self.w).astype(np.float64)
        pu, pv, ok = warp(self.A[k], self.b[k], u, v, d)
        m = DESC_MARGIN
        ok = ok & (pu >= m) & (pu <= self.w - m - 1) & (pv >= m) & (pv <= self.h - m - 1)
        return pu, pv, ok

    def gather_rays(self, pix, d):
        """solver.py:206-227: invalid rays carry desc 0 and q 0.5."""
        n = pix.shape[0]
        desc = np.zeros((n, self.K, DESC_LEN))
        valid = np.zeros((n, self.K), dtype=bool)
        q = np.full((n, self.K), 0.5)
        for k in range(self.K):
            pu, pv, ok = self.ray(pix, d, k)
            i = np.flatnonzero(ok)
            if i.size:
                desc[i, k] = self._lerp_rows(self._dflat[k], DESC_LEN, pu[i], pv[i])
                q[i, k] = self._lerp_rows(self._pflat[k], 1, pu[i], pv[i])[:, 0]
                valid[i, k] = True
        return desc, valid, q

    def energy(self, pix, d, bits):
        """solver.py:229-260 (+ prior.py:365-370): returns (energy, real)."""
        n = pix.shape[0]
        s1 = np.zeros((n, DESC_LEN))
        s2 = np.zeros((n, DESC_LEN))
        cnt = np.zeros(n, dtype=np.int32)
        for k in range(self.K):
            on = ((bits >> np.uint32(k)) & np.uint32(1)).astype(bool)
            if not on.any():
                continue
            pu, pv, ok = self.ray(pix, d, k)
            i = np.flatnonzero(on & ok)
            if i.size == 0:
                continue
            f = self._lerp_rows(self._dflat[k], DESC_LEN, pu[i], pv[i])
            s1[i] += f
            s2[i] += f * f
            cnt[i] += 1
        real = cnt >= self.p.min_static_rays
        nn = np.maximum(cnt, 1).astype(np.float64)
        # numpy's contiguous 16-wide sum is pairwise: (a_j + a_{j+8}) tree
        var = np.clip((s2 - s1 * s1 / nn[:, None]).sum(axis=1) / nn, 0.0, None)
        var = np.where(real, var, VARIANCE_CEILING)
        e = self.p.beta * var - log_prior(d, self.mu[pix], self.p.sigma, self.p.gamma)
        return e, real

    # -- candidates -----------------------------------------------------------

    def support_pairs(self, is_active):
        """solver.py:286-321: unique (pixel, float32 disparity) within radius."""
        r = self.p.neighborhood_radius
        ir = int(np.floor(r))
        span = np.arange(-ir, ir + 1)
        du, dv = np.meshgrid(span, span)
        disk = du * du + dv * dv <= r * r
        du = du[disk].astype(np.int64)
        dv = dv[disk].astype(np.int64)
        if self.support_d.size == 0:
            return np.zeros(0, np.int64), np.zeros(0, np.float32)
        pu = self.support_uv[:, 0].astype(np.int64)[:, None] + du[None, :]
        pv = self.support_uv[:, 1].astype(np.int64)[:, None] + dv[None, :]
        inside = (pu >= 0) & (pu < self.w) & (pv >= 0) & (pv < self.h)
        pix = (pv * self.w + pu)[inside]
        val = np.broadcast_to(self.support_d.astype(np.float32)[:, None], pu.shape)[inside]
        keep = is_active[pix]
        pix, val = pix[keep], val[keep]
        o = np.lexsort((val, pix))
        pix, val = pix[o], val[o]
        first = np.ones(pix.size, dtype=bool)
        first[1:] = (pix[1:] != pix[:-1]) | (val[1:] != val[:-1])
        return pix[first], val[first]

    def candidates(self, pixel):
        """Every candidate the M-step examines at one pixel (unsorted, may repeat)."""
        mu = self.mu[pixel]
        band = mu + self.band
        band = band[(band > 0.0) & (band <= self.p.d_max)]
        is_act = np.zeros(self.h * self.w, bool)
        is_act[pixel] = True
        _, sv = self.support_pairs(is_act)
        sv = sv.astype(np.float64)
        sv = sv[(sv > 0.0) & (sv <= self.p.d_max)]
        return np.concatenate([band, self.coarse, sv])

    # -- the two steps -------------------------------------------------------------

    def m_step(self, active, static_all, pairs=None):
        """solver.py:325-407: lexicographic (energy, d) argmin over candidates.

        Lower-bound pruning (-log prior <= incumbent) is the reference's exact
        shortcut (solver.py:341-347), kept so the CPU timing is honest.
        """
        n = active.shape[0]
        be = np.full(n, np.inf)
        bd = np.full(n, np.inf)
        br = np.zeros(n, dtype=bool)
        bits = static_all[active]
        mu = self.mu[active]
        p = self.p

        def offer(rows, dv):
            live = -log_prior(dv, mu[rows], p.sigma, p.gamma) <= be[rows]
            rows, dv = rows[live], dv[live]
            for lo in range(0, rows.size, _ROWS):
                r = rows[lo:lo + _ROWS]
                d = dv[lo:lo + _ROWS]
                e, real = self.energy(active[r], d, bits[r])
                win = (e < be[r]) | ((e == be[r]) & (d < bd[r]))
                be[r[win]] = e[win]
                bd[r[win]] = d[win]
                br[r[win]] = real[win]

        rows_all = np.arange(n)
        for off in self.band:
            d = mu + off
            ok = (d > 0.0) & (d <= p.d_max)
            offer(rows_all[ok], d[ok])
        for c in self.coarse:
            offer(rows_all, np.full(n, c))

        if pairs is None:
            is_act = np.zeros(self.h * self.w, dtype=bool)
            is_act[active] = True
            ppix, pval = self.support_pairs(is_act)
            pairs = (np.searchsorted(active, ppix), pval)
        prow, pval = pairs
        for lo in range(0, prow.size, _ROWS):
            r = prow[lo:lo + _ROWS]
            d = pval[lo:lo + _ROWS].astype(np.float64)
            keep = (d > 0.0) & (d <= p.d_max)
            keep &= -log_prior(d, mu[r], p.sigma, p.gamma) <= be[r]
            r, d = r[keep], d[keep]
            if r.size == 0:
                continue
            e, real = self.energy(active[r], d, bits[r])
            o = np.lexsort((d, e, r))          # per pixel: best (e, d) first
            r, e, d, real = r[o], e[o], d[o], real[o]
            lead = np.ones(r.size, dtype=bool)
            lead[1:] = r[1:] != r[:-1]
            r, e, d, real = r[lead], e[lead], d[lead], real[lead]
            win = (e < be[r]) | ((e == be[r]) & (d < bd[r]))
            be[r[win]] = e[win]
            bd[r[win]] = d[win]
            br[r[win]] = real[win]

        status = np.full(n, STATUS_VALID, dtype=np.uint8)
        empty = ~np.isfinite(be)
        status[empty] = STATUS_LOW_TEXTURE
        status[~empty & ~br] = STATUS_NO_STATIC_EVIDENCE
        bd[empty] = np.nan
        return bd, be, status, pairs

    def e_step_at(self, pix, d):
        """solver.py:409-419."""
        static = np.empty(pix.shape[0], dtype=np.uint32)
        vbits = np.empty(pix.shape[0], dtype=np.uint32)
        wts = np.arange(self.K, dtype=np.uint32)
        for lo in range(0, pix.shape[0], _ESTEP_ROWS):
            hi = min(lo + _ESTEP_ROWS, pix.shape[0])
            desc, valid, q = self.gather_rays(pix[lo:hi], d[lo:hi])
            static[lo:hi] = e_step(desc, valid, q, self.p)
            vbits[lo:hi] = (valid.astype(np.uint32) << wts).sum(axis=1)
        return static, vbits

    def initial_masks(self, pix):
        """solver.py:421-432: valid & q >= threshold at the surface disparity."""
        static = np.empty(pix.shape[0], dtype=np.uint32)
        vbits = np.empty(pix.shape[0], dtype=np.uint32)
        wts = np.arange(self.K, dtype=np.uint32)
        for lo in range(0, pix.shape[0], _ESTEP_ROWS):
            hi = min(lo + _ESTEP_ROWS, pix.shape[0])
            _, valid, q = self.gather_rays(pix[lo:hi], self.mu[pix[lo:hi]])
            static[lo:hi] = ((valid & (q >= self.p.threshold)).astype(np.uint32) << wts).sum(axis=1)
            vbits[lo:hi] = (valid.astype(np.uint32) << wts).sum(axis=1)
        return static, vbits

    def active_set(self, dynamic_only):
        allp = np.arange(self.h * self.w, dtype=np.int64)
        if dynamic_only:
            return allp[self.priors[self.ref].ravel() < self.p.threshold]
        return allp

    def solve(self, dynamic_only=False, forced_iters=None, active=None, trace=None):
        """solver.py:436-502.

        forced_iters (non-reference bench mode): run exactly that many
        M/E alternations, ignoring the convergence break.
        active: explicit sorted pixel subset (used for bounded CPU samples).
        trace: optional list receiving (static_before_m, d, e, status) per iteration.
        Returns dict with values/status/static/valid (flat) and stats.
        """
        npx = self.h * self.w
        allp = np.arange(npx, dtype=np.int64)
        if active is None:
            active = self.active_set(dynamic_only)
            static, vbits = self.initial_masks(allp)        # solver.py:455
        else:
            # bounded-sample mode: only the sampled pixels are initialised
            static = np.zeros(npx, dtype=np.uint32)
            vbits = np.zeros(npx, dtype=np.uint32)
            static[active], vbits[active] = self.initial_masks(active)
        stats = dict(iterations_run=0, converged_after=None, mean_energy=[],
                     prev_energy=[], changed_fraction=[])
        d_prev = None
        d_act = None
        st_act = None
        pairs = None
        iters = forced_iters if forced_iters is not None else self.p.max_iters
        for it in range(1, iters + 1):
            if active.size == 0:
                stats["converged_after"] = 0
                break
            stats["iterations_run"] = it
            static_before = static
            d_act, e_act, st_act, pairs = self.m_step(active, static, pairs)
            fin = e_act[np.isfinite(e_act)]
            stats["mean_energy"].append(float(fin.mean()) if fin.size else float("nan"))
            changed = None
            if d_prev is not None:
                pe, _ = self.energy(active, d_prev, static[active])
                pf = pe[np.isfinite(pe)]
                stats["prev_energy"].append(float(pf.mean()) if pf.size else float("nan"))
                with np.errstate(invalid="ignore"):
                    changed = float(np.mean(np.abs(d_act - d_prev) > 0.5))
                stats["changed_fraction"].append(changed)
            solved = st_act != STATUS_LOW_TEXTURE
            upd = active[solved]
            s_new, v_new = self.e_step_at(upd, d_act[solved])
            static = static.copy()
            vbits = vbits.copy()
            static[upd] = s_new
            vbits[upd] = v_new
            if trace is not None:
                trace.append((static_before, d_act, e_act, st_act))
            if forced_iters is None and changed is not None and changed < 1e-3:
                stats["converged_after"] = it - 1
                break
            d_prev = d_act
        values = self.mu.astype(np.float32).copy()
        status = np.full(npx, STATUS_VALID, dtype=np.uint8)
        if active.size and d_act is not None:
            ok = np.isfinite(d_act)
            values[active[ok]] = d_act[ok].astype(np.float32)
            values[active[~ok]] = 0.0
            status[active] = st_act
        return dict(values=values.reshape(self.h, self.w), status=status.reshape(self.h, self.w),
                    static_bits=static.reshape(self.h, self.w), valid_bits=vbits.reshape(self.h, self.w),
                    stats=stats, active=active)

    # -- decision margins (parity harness) -------------------------------------

    def m_margins(self, active, static_all):
        """Best minus second-best energy over candidates with |d - d_best| > 1e-9.

        Evaluates every candidate without pruning (SURVEY.md §8a recipe
        evidence 1).  Returns (d_best, e_best, margin) per active pixel.
        """
        n = active.shape[0]
        bits = static_all[active]
        mu = self.mu[active]
        cand_rows, cand_d = [], []
        rows_all = np.arange(n)
        for off in self.band:
            d = mu + off
            ok = (d > 0.0) & (d <= self.p.d_max)
            cand_rows.append(rows_all[ok])
            cand_d.append(d[ok])
        for c in self.coarse:
            cand_rows.append(rows_all)
            cand_d.append(np.full(n, c))
        is_act = np.zeros(self.h * self.w, dtype=bool)
        is_act[active] = True
        ppix, pval = self.support_pairs(is_act)
        prow = np.searchsorted(active, ppix)
        pv = pval.astype(np.float64)
        ok = (pv > 0.0) & (pv <= self.p.d_max)
        cand_rows.append(prow[ok])
        cand_d.append(pv[ok])
        rows = np.concatenate(cand_rows)
        ds = np.concatenate(cand_d)
        es = np.empty(rows.size)
        for lo in range(0, rows.size, _ROWS):
            r = rows[lo:lo + _ROWS]
            es[lo:lo + _ROWS], _ = self.energy(active[r], ds[lo:lo + _ROWS], bits[r])
        o = np.lexsort((ds, es, rows))
        rows, ds, es = rows[o], ds[o], es[o]
        lead = np.ones(rows.size, dtype=bool)
        lead[1:] = rows[1:] != rows[:-1]
        first = np.flatnonzero(lead)
        d_best = np.full(n, np.nan)
        e_best = np.full(n, np.inf)
        d_best[rows[first]] = ds[first]
        e_best[rows[first]] = es[first]
        far = np.abs(ds - d_best[rows]) > 1e-9
        second = np.full(n, np.inf)
        np.minimum.at(second, rows[far], es[far])
        return d_best, e_best, second - e_best

    def e_margins(self, pix, d):
        """Top-1 minus top-2 E-step score at disparity d (inf if one admissible mask)."""
        desc, valid, q = self.gather_rays(pix, d)
        s, _ = e_step_scores(desc, valid, q, self.p)
        top2 = -np.partition(-s, 1, axis=1)[:, :2]
        with np.errstate(invalid="ignore"):
            m = top2[:, 0] - top2[:, 1]
        m[~np.isfinite(top2[:, 1])] = np.inf
        return m


# -- refocus -----------------------------------------------------------------

def median_filter(image, radius):
    """refocus.py:68-106: per-channel median over the clipped window."""
    if radius <= 0:
        return image.copy()
    h, w = image.shape[:2]
    ch = image.shape[2] if image.ndim == 3 else 1
    src = image.reshape(h, w, ch).astype(np.float32)
    n = 2 * radius + 1
    pad = np.full((h + 2 * radius, w + 2 * radius, ch), np.inf, dtype=np.float32)
    pad[radius:radius + h, radius:radius + w] = src
    win = np.stack([pad[dy:dy + h, dx:dx + w] for dy in range(n) for dx in range(n)], axis=2)
    cy = np.minimum(np.arange(h) + radius, h - 1) - np.maximum(np.arange(h) - radius, 0) + 1
    cx = np.minimum(np.arange(w) + radius, w - 1) - np.maximum(np.arange(w) - radius, 0) + 1
    cnt = cy[:, None] * cx[None, :]
    win.sort(axis=2)
    lo = np.take_along_axis(win, ((cnt - 1) // 2)[:, :, None, None], axis=2)[:, :, 0]
    hi = np.take_along_axis(win, (cnt // 2)[:, :, None, None], axis=2)[:, :, 0]
    med = np.float32(0.5) * (lo + hi)
    return np.clip(np.rint(med), 0, 255).astype(image.dtype).reshape(image.shape)


def synthesize(images, warp_a, warp_b, ref_index, values, status, static_bits,
               min_static_rays=2, median_radius=1, copy_mask=None):
    """refocus.py:24-49 + 109-148: Eq. 2 average of static in-bounds rays."""
    ref = np.asarray(images[ref_index])
    h, w = ref.shape[:2]
    out = ref.copy()
    prov = np.full((h, w), PROV_FALLBACK, dtype=np.uint8)
    n_rays = np.zeros((h, w), dtype=np.uint8)
    copy = np.zeros((h, w), bool) if copy_mask is None else np.asarray(copy_mask, bool)
    prov[copy] = PROV_COPIED
    pix = np.flatnonzero(((~copy) & (status == STATUS_VALID)).ravel())
    if pix.size:
        d = values.ravel()[pix].astype(np.float64)
        bits = static_bits.ravel()[pix]
        u = (pix % w).astype(np.float64)
        v = (pix // w).astype(np.float64)
        tot = np.zeros((pix.size, 3))
        cnt = np.zeros(pix.size, dtype=np.int32)
        for k in range(len(images)):
            on = ((bits >> np.uint32(k)) & np.uint32(1)).astype(bool)
            if not on.any():
                continue
            pu, pv, ok = warp(warp_a[k], warp_b[k], u, v, d)
            kh, kw = images[k].shape[:2]
            ok = ok & (pu >= 0.0) & (pu <= kw - 1.0) & (pv >= 0.0) & (pv <= kh - 1.0)
            i = np.flatnonzero(on & ok)
            if i.size:
                tot[i] += bilinear(images[k], pu[i], pv[i])
                cnt[i] += 1
        n_rays.ravel()[pix] = np.clip(cnt, 0, 255).astype(np.uint8)
        good = cnt >= min_static_rays
        rgb = np.clip(np.rint(tot[good] / cnt[good, None]), 0, 255).astype(np.uint8)
        out.reshape(-1, 3)[pix[good]] = rgb
        prov.ravel()[pix[good]] = PROV_REFOCUSED
    if median_radius > 0:
        filt = median_filter(out, median_radius)
        rw = prov != PROV_COPIED
        out[rw] = filt[rw]
    return out, prov, n_rays
