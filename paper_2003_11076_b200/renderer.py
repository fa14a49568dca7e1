"""Synthetic light fields rendered on the device.

`render(spec)` is the reference's `render` (synth.py:244-309): per view a
nearest-surface ray cast with the value-noise + sinusoid textures, the 4x
supersampled billboard edges, the reference view's background and
disparity ground truth, and the seeded, box-blurred priors
(`corrupt_prior`, synth.py:334-346) -- computed by st_render_view,
st_render_background and st_corrupt_prior (csrc/st_render.cu).

The host does what the reference does with numpy scalars: each surface's
texture constants are drawn from `np.random.default_rng(seed)` exactly as
`surface_color` draws them (synth.py:66-70), the angle cosines / sines and
2*pi*rate are evaluated with numpy, and the flip stream's PCG64 state comes
from `np.random.default_rng([seed, k, 17])`; the device advances that
stream itself.  The billboard rectangles (synth.py:233-241) are five scalar
operations per occluder, evaluated here in the reference's order.
"""

import ctypes as C

import numpy as np

from . import _native as N
from .device import download, empty, require_cuda, upload
from .frame import LightFieldFrame


def _surface(s, is_occluder):
    out = N.StSurface()
    out.is_occluder = 1 if is_occluder else 0
    seed32 = int(s.seed) & 0xFFFFFFFF  # the lattice hash uses the low 32 bits (synth.py:33)
    out.seed = seed32 - (1 << 32) if seed32 >= 1 << 31 else seed32
    out.depth, out.base = float(s.depth), float(s.base)
    out.amplitude, out.frequency = float(s.amplitude), float(s.frequency)
    if is_occluder:
        out.half_w, out.half_h = s.width / 2.0, s.height / 2.0
        out.center_x, out.center_y = float(s.center_x), float(s.center_y)
    else:
        out.has_x_min = int(s.x_min is not None)
        out.has_x_max = int(s.x_max is not None)
        out.x_min = float(s.x_min) if s.x_min is not None else 0.0
        out.x_max = float(s.x_max) if s.x_max is not None else 0.0
    # surface_color's draws, in its order (synth.py:66-70)
    rng = np.random.default_rng(s.seed)
    ang = rng.uniform(0.0, np.pi, size=3)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(3, 3))
    rate = rng.uniform(0.6, 1.1, size=3)
    nw = rng.uniform(0.3, 0.5, size=3)
    for i in range(3):
        out.c0[i] = float(2.0 * np.pi * rate[i])
        out.ca[i] = float(np.cos(ang[i]))
        out.sa[i] = float(np.sin(ang[i]))
        out.nw[i] = float(nw[i])
        for c in range(3):
            out.ph[i][c] = float(ph[i, c])
    return out


def _scene(spec):
    surfaces = ([(o, True) for o in sorted(spec.occluders, key=lambda o: o.depth)]
                + [(p, False) for p in sorted(spec.planes, key=lambda p: p.depth)])
    if len(surfaces) > N.MAX_SURFACES:
        raise ValueError(f"the device renderer holds at most {N.MAX_SURFACES} surfaces")
    intr = spec.intrinsics()
    sc = N.StScene()
    sc.width, sc.height = int(spec.width), int(spec.height)
    sc.n_surfaces = len(surfaces)
    sc.fx, sc.fy, sc.cx, sc.cy = intr.fx, intr.fy, intr.cx, intr.cy
    for i, (s, occ) in enumerate(surfaces):
        sc.surf[i] = _surface(s, occ)
    return sc


def _rects(spec, center):
    """The occluders' billboard rectangles from one camera (synth.py:233-241)."""
    intr = spec.intrinsics()
    out = []
    for o in spec.occluders:
        z = o.depth - center[2]
        out += [intr.cx + intr.fx * (o.center_x - o.width / 2.0 - center[0]) / z,
                intr.cx + intr.fx * (o.center_x + o.width / 2.0 - center[0]) / z,
                intr.cy + intr.fy * (o.center_y - o.height / 2.0 - center[1]) / z,
                intr.cy + intr.fy * (o.center_y + o.height / 2.0 - center[1]) / z]
    return np.asarray(out, dtype=np.float64)


def _pcg_state(seed):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m = (1 << 64) - 1
    s, inc = int(st["state"]), int(st["inc"])
    return (C.c_uint64 * 4)(s >> 64, s & m, inc >> 64, inc & m)


def _vec(x, n):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(n))
    return a, a.ctypes.data_as(C.c_void_p)


def render(spec):
    """SceneSpec -> (LightFieldFrame, GroundTruth) on the device (synth.py:244-309)."""
    from .synth import GroundTruth
    t = require_cuda()
    spec.validate()
    rig = spec.rig()
    h, w = spec.height, spec.width
    sc = _scene(spec)
    lib = N.lib()
    fail = t.zeros((1,), dtype=t.int32, device="cuda")
    ws = empty((int(lib.st_corrupt_prior_workspace(w, h)),), t.uint8)
    images, masks, priors = [], [], []
    gt_disp = gt_bg = None
    keep = []
    for k in range(spec.cameras):
        center = np.asarray(rig.camera_center(k), dtype=np.float64)
        rot = np.asarray(rig.extrinsics(k).rotation, dtype=np.float64)
        c_arr, c_ptr = _vec(center, 3)
        r_arr, r_ptr = _vec(rot, 9)
        rects = upload(_rects(spec, center)) if spec.occluders else None
        img = empty((h, w, 3), t.uint8)
        mask = empty((h, w), t.uint8)
        N.invoke("st_render_view", C.byref(sc), c_ptr, r_ptr, rects, len(spec.occluders), img,
                 mask, fail)
        prior = empty((h, w), t.float32)
        N.invoke("st_corrupt_prior", mask, w, h, _pcg_state([spec.seed, k, 17]),
                 float(spec.p_flip), int(spec.blur_radius), prior, ws, ws.numel())
        images.append(img)
        masks.append(mask)
        priors.append(prior)
        if k == rig.ref_index:
            gt_bg = empty((h, w, 3), t.uint8)
            gt_disp = empty((h, w), t.float32)
            N.invoke("st_render_background", C.byref(sc), c_ptr, r_ptr,
                     float(spec.focal * rig.unit_baseline), gt_bg, gt_disp, fail)
        keep.append((c_arr, r_arr, rects))
    if int(download(fail)[0]):
        raise ValueError("scene constraint violated: some rays hit no surface "
                         "(deepest plane must be an unbounded backdrop)")
    # plain (pageable) numpy arrays out, like the reference's
    t.cuda.current_stream().synchronize()
    frame = LightFieldFrame(images=[x.cpu().numpy() for x in images],
                            priors=[x.cpu().numpy() for x in priors])
    gt = GroundTruth(disparity=gt_disp.cpu().numpy(), background=gt_bg.cpu().numpy(),
                     masks=[m.cpu().numpy().astype(bool) for m in masks])
    return frame, gt
