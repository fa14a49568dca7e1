"""numpy restatement of the reference support-point harvest.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may import this).

Reference: /root/reference/pkg/src/seethrough/prior.py
  detect_support_candidates :51-66   texture + validity on a stride grid
  _scan_costs               :69-82   descriptor SAD along the warped locus
  _best_with_ratio          :85-98   first argmin + 0.9 uniqueness ratio
  match_support_points      :101-138 forward scan + left-right check
  reproject_occluded_support:146-180 lift through the source view
  deduplicate               :183-212 greedy priority-order resolution
  ring_min_prior            :215-230 prior erosion over the ring
  collect_support           :233-260 the whole harvest
and features.py:114-133 (texture_energy, sample_descriptors),
geometry.py:191-252 (nearest_neighbor, pair warps).

Cameras are plain arrays here: per view (fx, fy, cx, cy), rotation (3, 3),
translation (3,), plus unit_baseline and ref_index.  Every floating-point
expression keeps the reference's evaluation order.
"""

import numpy as np

from .em import DESC_MARGIN, RING

SUPPORT_STRIDE = 5            # prior.py:25
MIN_TEXTURE = 25.0            # prior.py:26
UNIQUENESS_RATIO = 0.9        # prior.py:27
SECOND_BEST_EXCLUSION = 1.0   # prior.py:29
LEFT_RIGHT_TOL = 1.0          # prior.py:30


class Cameras:
    """The rig quantities the harvest reads (geometry.py:128-252)."""

    def __init__(self, fx, fy, cx, cy, rotation, translation, unit_baseline, ref_index,
                 width, height):
        self.fx = [float(x) for x in fx]
        self.fy = [float(x) for x in fy]
        self.cx = [float(x) for x in cx]
        self.cy = [float(x) for x in cy]
        self.rot = [np.asarray(r, dtype=np.float64) for r in rotation]
        self.trans = [np.asarray(t, dtype=np.float64) for t in translation]
        self.unit_baseline = float(unit_baseline)
        self.ref_index = int(ref_index)
        self.width = int(width)
        self.height = int(height)
        self.centers = np.array([-r.T @ t for r, t in zip(self.rot, self.trans)])

    def __len__(self):
        return len(self.fx)

    def kmat(self, k):
        return np.array([[self.fx[k], 0.0, self.cx[k]], [0.0, self.fy[k], self.cy[k]],
                         [0.0, 0.0, 1.0]])

    def kinv(self, k):
        # geometry.py CameraIntrinsics.inverse_matrix: closed form
        fx, fy, cx, cy = self.fx[k], self.fy[k], self.cx[k], self.cy[k]
        return np.array([[1.0 / fx, 0.0, -cx / fx], [0.0, 1.0 / fy, -cy / fy],
                         [0.0, 0.0, 1.0]])

    def nearest_neighbor(self, k):
        """geometry.py:191-196 (ties -> lower index)."""
        d = np.linalg.norm(self.centers - self.centers[k], axis=1)
        d[k] = np.inf
        return int(np.argmin(d))

    def ref_warp(self, k):
        """geometry.py:156-172."""
        if k == self.ref_index:
            return np.eye(3), np.zeros(3)
        scale = self.fx[self.ref_index] * self.unit_baseline
        km = self.kmat(k)
        return km @ self.rot[k] @ self.kinv(self.ref_index), km @ self.trans[k] / scale

    def pair_warp(self, src, dst):
        """geometry.py:221-240."""
        if src == self.ref_index:
            return self.ref_warp(dst)
        rel_r = self.rot[dst] @ self.rot[src].T
        rel_t = self.trans[dst] - rel_r @ self.trans[src]
        km = self.kmat(dst)
        a = km @ rel_r @ self.kinv(src)
        b = km @ rel_t / (self.fx[src] * self.unit_baseline)
        if src == dst:
            a = np.eye(3)
            b = np.zeros(3)
        return a, b


def texture_energy(desc):
    """features.py:114-117: per-pixel sum of |entry - 128| (int32)."""
    return np.abs(desc.astype(np.int32) - 128).sum(axis=2)


def ring_min_prior(prob):
    """prior.py:215-230: min of the prior over the ring offsets (clipped)."""
    h, w = prob.shape
    out = prob.copy()
    ys = np.arange(h)
    xs = np.arange(w)
    for du, dv in RING:
        sy = np.clip(ys + dv, 0, h - 1)
        sx = np.clip(xs + du, 0, w - 1)
        np.minimum(out, prob[sy][:, sx], out)
    return out


def detect(desc, stride=SUPPORT_STRIDE, min_texture=MIN_TEXTURE):
    """prior.py:51-66 (descriptor-valid interior = margin 3, features.py:102-103)."""
    h, w = desc.shape[:2]
    energy = texture_energy(desc)
    vs = np.arange(0, h, stride)
    us = np.arange(0, w, stride)
    uu, vv = np.meshgrid(us, vs)
    uu = uu.ravel()
    vv = vv.ravel()
    valid = ((uu >= DESC_MARGIN) & (uu < w - DESC_MARGIN) & (vv >= DESC_MARGIN)
             & (vv < h - DESC_MARGIN))
    keep = valid & (energy[vv, uu] >= min_texture)
    return np.stack([uu[keep], vv[keep]], axis=1)


def _sample(flat, h, w, u, v):
    """features.py:120-133 over a cached float32 (h*w, 16) plane: sampling.py
    bilinear (fp32 tap difference, fp64 lerp) plus the margin validity."""
    valid = ((u >= DESC_MARGIN) & (u <= w - DESC_MARGIN - 1)
             & (v >= DESC_MARGIN) & (v <= h - DESC_MARGIN - 1))
    uc = np.clip(np.nan_to_num(u, nan=0.0, posinf=0.0, neginf=0.0), 0.0, w - 1.0)
    vc = np.clip(np.nan_to_num(v, nan=0.0, posinf=0.0, neginf=0.0), 0.0, h - 1.0)
    iu = np.minimum(np.floor(uc), w - 2.0)
    iv = np.minimum(np.floor(vc), h - 2.0)
    fu = (uc - iu)[:, None]
    fv = (vc - iv)[:, None]
    base = iv.astype(np.int64) * w + iu.astype(np.int64)
    t0 = flat[base]
    t1 = flat[base + 1]
    b0 = flat[base + w]
    b1 = flat[base + w + 1]
    top = t0 + fu * (t1 - t0)
    bot = b0 + fu * (b1 - b0)
    return top + fv * (bot - top), valid


def _warp(a, b, u, v, d):
    """geometry.py:242-252, left to right."""
    hx = a[0, 0] * u + a[0, 1] * v + a[0, 2] + d * b[0]
    hy = a[1, 0] * u + a[1, 1] * v + a[1, 2] + d * b[1]
    hz = a[2, 0] * u + a[2, 1] * v + a[2, 2] + d * b[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        return hx / hz, hy / hz, hz > 0


def scan_costs(a, b, u, v, d_grid, flat_src, flat_dst, h, w):
    """prior.py:69-82: (n, n_d) SAD, inf where the ray or a sample is invalid.
    The 16-term sum is numpy's contiguous reduction (8 lanes + pairwise)."""
    ref_desc, ref_ok = _sample(flat_src, h, w, u, v)
    n = u.shape[0]
    costs = np.full((n, d_grid.size), np.inf, dtype=np.float64)
    for j, d in enumerate(d_grid):
        pu, pv, front = _warp(a, b, u, v, np.full(n, d))
        tgt, tgt_ok = _sample(flat_dst, h, w, pu, pv)
        ok = ref_ok & tgt_ok & front
        if not ok.any():
            continue
        costs[ok, j] = np.abs(ref_desc[ok] - tgt[ok]).sum(axis=1)
    return costs


def best_with_ratio(costs, d_grid):
    """prior.py:85-98."""
    best_j = np.argmin(costs, axis=1)
    rows = np.arange(costs.shape[0])
    best_cost = costs[rows, best_j]
    best_d = d_grid[best_j]
    masked = costs.copy()
    masked[np.abs(d_grid[None, :] - best_d[:, None]) <= SECOND_BEST_EXCLUSION] = np.inf
    second = masked.min(axis=1)
    ok = np.isfinite(best_cost)
    with np.errstate(invalid="ignore"):
        ok &= ~(np.isfinite(second) & (best_cost > UNIQUENESS_RATIO * second))
    return np.where(ok, best_d, np.nan), best_cost


def match(cams, src, dst, cands, flats, d_max):
    """prior.py:101-138 -> list of (u, v, d, src)."""
    if cands.shape[0] == 0:
        return []
    h, w = cams.height, cams.width
    d_grid = np.arange(0.5, d_max + 0.25, 0.5)
    u = cands[:, 0].astype(np.float64)
    v = cands[:, 1].astype(np.float64)
    a, b = cams.pair_warp(src, dst)
    best_d, _ = best_with_ratio(scan_costs(a, b, u, v, d_grid, flats[src], flats[dst], h, w),
                                d_grid)
    have = np.isfinite(best_d)
    if not have.any():
        return []
    iu = np.flatnonzero(have)
    pu, pv, _ = _warp(a, b, u[iu], v[iu], best_d[iu])
    ru = np.rint(pu)
    rv = np.rint(pv)
    ra, rb = cams.pair_warp(dst, src)
    rbest, _ = best_with_ratio(scan_costs(ra, rb, ru, rv, d_grid, flats[dst], flats[src], h, w),
                               d_grid)
    scale = cams.fx[src] / cams.fx[dst]
    agree = np.isfinite(rbest) & (np.abs(rbest * scale - best_d[iu]) <= LEFT_RIGHT_TOL)
    return [(int(cands[r, 0]), int(cands[r, 1]), float(best_d[r]), src) for r in iu[agree]]


def reproject(points, cams, ref_prior, d_max, threshold):
    """prior.py:146-180 (scalar per point, like the reference)."""
    out = []
    ref = cams.ref_index
    fxr, fyr, cxr, cyr = cams.fx[ref], cams.fy[ref], cams.cx[ref], cams.cy[ref]
    h, w = cams.height, cams.width
    for (u, v, d, src) in points:
        if src == ref:
            continue
        depth = cams.fx[src] * cams.unit_baseline / d
        xc = (u - cams.cx[src]) / cams.fx[src] * depth
        yc = (v - cams.cy[src]) / cams.fy[src] * depth
        cam = np.array([xc, yc, depth])
        world = cams.rot[src].T @ (cam - cams.trans[src])
        if world[2] <= 0:
            continue
        ur = fxr * world[0] / world[2] + cxr
        vr = fyr * world[1] / world[2] + cyr
        iu = int(np.rint(ur))
        iv = int(np.rint(vr))
        if not (0 <= iu < w and 0 <= iv < h):
            continue
        if ref_prior[iv, iu] >= threshold:
            continue
        d_ref = fxr * cams.unit_baseline / world[2]
        if not 0.0 < d_ref <= d_max:
            continue
        out.append((iu, iv, float(d_ref), src))
    return out


def deduplicate(points, ref_index):
    """prior.py:183-212: stable priority sort, greedy acceptance, raster sort."""
    ranked = sorted(points, key=lambda p: (p[3] != ref_index, p[2], p[1], p[0]))
    taken = {}
    accepted = []
    for p in ranked:
        key = (p[0], p[1])
        if key in taken:
            continue
        conflict = False
        for du in (-1, 0, 1):
            for dv in (-1, 0, 1):
                q = taken.get((p[0] + du, p[1] + dv))
                if q is not None and abs(q[2] - p[2]) > 2.0:
                    conflict = True
                    break
            if conflict:
                break
        if conflict:
            continue
        taken[key] = p
        accepted.append(p)
    accepted.sort(key=lambda p: (p[1], p[0], p[2]))
    return accepted


def collect_support(descs, priors, cams, d_max, threshold, stride=SUPPORT_STRIDE,
                    min_texture=MIN_TEXTURE, stages=None):
    """prior.py:233-260 -> list of (u, v, d, source_view), raster order.

    `stages` (optional dict) receives the per-view candidates and matches."""
    ref = cams.ref_index
    h, w = cams.height, cams.width
    flats = [np.asarray(dsc, dtype=np.float32).reshape(h * w, -1) for dsc in descs]
    thr = np.float32(threshold)  # NEP 50: a Python float compares as float32
    collected = []
    for view in range(len(cams)):
        cands = detect(descs[view], stride, min_texture)
        if cands.shape[0] == 0:
            continue
        eroded = ring_min_prior(priors[view])
        cands = cands[eroded[cands[:, 1], cands[:, 0]] >= thr]
        matched = match(cams, view, cams.nearest_neighbor(view), cands, flats, d_max)
        if stages is not None:
            stages[view] = (cands, matched)
        if view == ref:
            collected.extend(p for p in matched if p[2] <= d_max)
        else:
            collected.extend(reproject(matched, cams, priors[ref], d_max, thr))
    return deduplicate(collected, ref)
