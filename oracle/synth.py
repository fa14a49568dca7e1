"""The reference renderer restated in numpy -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's `pkg/src/seethrough/synth.py` (lattice
hash / value noise :25-56, surface_color :59-82, _trace :174-230, render
:244-309, box_blur and corrupt_prior :314-346), its structure and arithmetic
kept so its frames are bit-identical to the reference's (pinned by
tests/test_synth_port.py against the reference in the build container and
against the frame digests the reference recorded in tests/golden/bench_*).
It is the checker for the device renderer (paper_2003_11076_b200.renderer)
and the input generator of CPU-only tests and bench.py's reference arm; the
product package never imports it.
"""

import numpy as np

from paper_2003_11076_b200.frame import LightFieldFrame
from paper_2003_11076_b200.synth import GroundTruth

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def _lattice(ix, iy, seed):
    """Per-lattice-point hash in [0, 1) (synth.py:25-36, wrapping uint64)."""
    with np.errstate(over="ignore"):
        h = (ix.astype(np.uint64) * _M1 ^ iy.astype(np.uint64) * _M2
             ^ np.uint64(seed & 0xFFFFFFFF) * _M3)
        h ^= h >> np.uint64(30)
        h *= _M2
        h ^= h >> np.uint64(27)
        h *= _M3
        h ^= h >> np.uint64(31)
    return (h >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def _noise(x, y, seed):
    """Smoothstep-interpolated lattice noise in [-1, 1] (synth.py:39-56)."""
    x0 = np.floor(x)
    y0 = np.floor(y)
    tx = x - x0
    ty = y - y0
    i = x0.astype(np.int64)
    j = y0.astype(np.int64)
    wx = tx * tx * (3.0 - 2.0 * tx)
    wy = ty * ty * (3.0 - 2.0 * ty)
    a = _lattice(i, j, seed)
    b = _lattice(i + 1, j, seed)
    c = _lattice(i, j + 1, seed)
    d = _lattice(i + 1, j + 1, seed)
    upper = a + wx * (b - a)
    lower = c + wx * (d - c)
    return 2.0 * (upper + wy * (lower - upper)) - 1.0


def surface_color(x, y, seed, base, amplitude, frequency):
    """(n, 3) float64 texture in [0, 255] at world coordinates (synth.py:59-82)."""
    x = np.asarray(x, dtype=np.float64) * frequency
    y = np.asarray(y, dtype=np.float64) * frequency
    rng = np.random.default_rng(seed)
    ang = rng.uniform(0.0, np.pi, size=3)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(3, 3))
    rate = rng.uniform(0.6, 1.1, size=3)
    nw = rng.uniform(0.3, 0.5, size=3)
    nz = _noise(x + 13.7, y + 7.31, seed)
    out = np.empty(x.shape + (3,), dtype=np.float64)
    for c in range(3):
        acc = np.zeros_like(x)
        for i in range(3):
            acc += np.sin(2.0 * np.pi * rate[i] * (x * np.cos(ang[i]) + y * np.sin(ang[i]))
                          + ph[i, c])
        out[..., c] = base + amplitude * ((1.0 - nw[c]) * (acc / 3.0) + nw[c] * nz)
    return np.clip(out, 0.0, 255.0)


def _trace(spec, center, rotation, su, sv, with_occluders=True):
    """Nearest-surface ray cast from one camera (synth.py:174-230)."""
    intr = spec.intrinsics()
    dirs = np.stack([(su - intr.cx) / intr.fx, (sv - intr.cy) / intr.fy, np.ones_like(su)],
                    axis=-1) @ rotation
    n = su.size
    color = np.zeros((n, 3))
    hit_occ = np.zeros(n, dtype=bool)
    depth = np.full(n, np.inf)
    done = np.zeros(n, dtype=bool)
    order = []
    if with_occluders:
        order += [("occ", o) for o in sorted(spec.occluders, key=lambda o: o.depth)]
    order += [("plane", p) for p in sorted(spec.planes, key=lambda p: p.depth)]
    for kind, s in order:
        if done.all():
            break
        todo = ~done
        dz = dirs[todo, 2]
        fwd = dz > 0
        with np.errstate(invalid="ignore"):
            t = np.where(fwd, (s.depth - center[2]) / np.where(dz == 0, 1.0, dz), np.inf)
            px = center[0] + t * dirs[todo, 0]
            py = center[1] + t * dirs[todo, 1]
        if kind == "occ":
            hit = (fwd & (np.abs(px - s.center_x) <= s.width / 2.0)
                   & (np.abs(py - s.center_y) <= s.height / 2.0))
        else:
            hit = fwd.copy()
            if s.x_min is not None:
                hit &= px >= s.x_min
            if s.x_max is not None:
                hit &= px < s.x_max
        if not hit.any():
            continue
        idx = np.flatnonzero(todo)[hit]
        color[idx] = surface_color(px[hit], py[hit], s.seed, s.base, s.amplitude, s.frequency)
        depth[idx] = s.depth
        hit_occ[idx] = kind == "occ"
        done[idx] = True
    if not done.all():
        raise ValueError("scene constraint violated: some rays hit no surface "
                         "(deepest plane must be an unbounded backdrop)")
    return color, hit_occ, depth


def _billboard_rect(spec, occ, center):
    intr = spec.intrinsics()
    z = occ.depth - center[2]
    return (intr.cx + intr.fx * (occ.center_x - occ.width / 2.0 - center[0]) / z,
            intr.cx + intr.fx * (occ.center_x + occ.width / 2.0 - center[0]) / z,
            intr.cy + intr.fy * (occ.center_y - occ.height / 2.0 - center[1]) / z,
            intr.cy + intr.fy * (occ.center_y + occ.height / 2.0 - center[1]) / z)


def render(spec):
    """SceneSpec -> (LightFieldFrame, GroundTruth) (synth.py:244-309)."""
    spec.validate()
    rig = spec.rig()
    h, w = spec.height, spec.width
    uu, vv = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    su, sv = uu.ravel(), vv.ravel()
    images, masks = [], []
    gt_disp = gt_bg = None
    for k in range(spec.cameras):
        center = rig.camera_center(k)
        rot = rig.extrinsics(k).rotation
        color, occ, _ = _trace(spec, center, rot, su, sv)
        cover = occ.astype(np.float64)
        edge = np.zeros(h * w, dtype=bool)
        for o in spec.occluders:
            u0, u1, v0, v1 = _billboard_rect(spec, o, center)
            edge |= (((np.abs(su - u0) <= 0.5) | (np.abs(su - u1) <= 0.5))
                     & (sv >= v0 - 0.5) & (sv <= v1 + 0.5))
            edge |= (((np.abs(sv - v0) <= 0.5) | (np.abs(sv - v1) <= 0.5))
                     & (su >= u0 - 0.5) & (su <= u1 + 0.5))
        if edge.any():
            bu, bv = su[edge], sv[edge]
            csum = np.zeros((bu.size, 3))
            osum = np.zeros(bu.size)
            for du, dv in ((-0.25, -0.25), (0.25, -0.25), (-0.25, 0.25), (0.25, 0.25)):
                c, o, _ = _trace(spec, center, rot, bu + du, bv + dv)
                csum += c
                osum += o
            color[edge] = csum / 4.0
            cover[edge] = osum / 4.0
        images.append(np.clip(np.rint(color), 0, 255).astype(np.uint8).reshape(h, w, 3))
        masks.append((cover >= 0.5).reshape(h, w))
        if k == rig.ref_index:
            bgc, _, bgz = _trace(spec, center, rot, su, sv, with_occluders=False)
            gt_bg = np.clip(np.rint(bgc), 0, 255).astype(np.uint8).reshape(h, w, 3)
            gt_disp = (spec.focal * rig.unit_baseline / bgz).astype(np.float32).reshape(h, w)
    priors = [corrupt_prior(1.0 - masks[k].astype(np.float64), spec.p_flip, spec.blur_radius,
                            seed=[spec.seed, k, 17]) for k in range(spec.cameras)]
    return (LightFieldFrame(images=images, priors=priors),
            GroundTruth(disparity=gt_disp, background=gt_bg, masks=masks))


def box_blur(arr, radius):
    """Clipped-window mean via an integral image (synth.py:314-331)."""
    a = np.asarray(arr, dtype=np.float64)
    if radius <= 0:
        return a.copy()
    h, w = a.shape
    s = np.zeros((h + 1, w + 1))
    s[1:, 1:] = a.cumsum(axis=0).cumsum(axis=1)
    r0 = np.maximum(np.arange(h) - radius, 0)
    r1 = np.minimum(np.arange(h) + radius + 1, h)
    c0 = np.maximum(np.arange(w) - radius, 0)
    c1 = np.minimum(np.arange(w) + radius + 1, w)
    tot = (s[r1[:, None], c1[None, :]] - s[r0[:, None], c1[None, :]]
           - s[r1[:, None], c0[None, :]] + s[r0[:, None], c0[None, :]])
    return tot / ((r1 - r0)[:, None] * (c1 - c0)[None, :])


def corrupt_prior(static_prob, p_flip, blur_radius, seed):
    """Seeded label flips, box blur, clamp -> float32 (synth.py:334-346)."""
    exact = np.asarray(static_prob, dtype=np.float64)
    flips = np.random.default_rng(seed).random(exact.shape) < p_flip
    return np.clip(box_blur(np.where(flips, 1.0 - exact, exact), blur_radius),
                   0.0, 1.0).astype(np.float32)


