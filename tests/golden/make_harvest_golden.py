"""Generate tests/golden/harvest_cases.npz by running the REFERENCE harvest.

Run in the build container only (the reference is not on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_harvest_golden.py

For each case it renders a seeded scene with the reference renderer
(synth.py:244-309), builds the rig (optionally tilted / with mixed focal
lengths), and records the inputs, the camera arrays, the points collected by
collect_support before deduplication (prior.py:245-259, replayed with the
reference's own stage functions) and the final support list
(prior.py:233-260).  Nothing here is product code.
"""

import os
import sys

import numpy as np

REF_SRC = os.environ.get("SEETHROUGH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
import seethrough as st  # noqa: E402
from seethrough import prior as sp  # noqa: E402
from seethrough.geometry import CameraExtrinsics, CameraIntrinsics, CameraRig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import tilted_rig  # noqa: E402


def mixed_focal_rig(rig, seed):
    """Per-view focal lengths / principal points perturbed (lr_scale != 1)."""
    rng = np.random.default_rng(seed)
    cams = []
    for i, (intr, extr) in enumerate(rig.cameras):
        if i != rig.ref_index:
            f = intr.fx * (1.0 + rng.uniform(-0.03, 0.03))
            intr = CameraIntrinsics(fx=f, fy=f * (1.0 + rng.uniform(-0.01, 0.01)),
                                    cx=intr.cx + rng.uniform(-2, 2),
                                    cy=intr.cy + rng.uniform(-2, 2),
                                    width=intr.width, height=intr.height)
        cams.append((intr, extr))
    return CameraRig(cams, ref_index=rig.ref_index, unit_baseline=rig.unit_baseline)


def collected(frame, rig, params, threshold, stride, min_texture):
    """collect_support's loop (prior.py:245-259) without the final dedup."""
    ref = rig.ref_index
    out = []
    for view in range(len(rig)):
        cands = sp.detect_support_candidates(frame.descriptors(view), stride, min_texture)
        if cands.shape[0] == 0:
            continue
        eroded = sp.ring_min_prior(frame.priors[view])
        cands = cands[eroded[cands[:, 1], cands[:, 0]] >= threshold]
        matched = sp.match_support_points(frame, rig, view, rig.nearest_neighbor(view), cands,
                                          params)
        if view == ref:
            out.extend(p for p in matched if p.d <= params.d_max)
        else:
            out.extend(sp.reproject_occluded_support(matched, rig, frame.priors[ref], params,
                                                     threshold))
    return out


def arrays(points):
    return (np.array([p.u for p in points], np.int32), np.array([p.v for p in points], np.int32),
            np.array([p.d for p in points], np.float64),
            np.array([p.source_view for p in points], np.int32))


def case(out, name, frame, rig, d_max=64.0, threshold=0.7, stride=5, min_texture=25.0):
    params = st.PriorParams(d_max=d_max)
    col = collected(frame, rig, params, threshold, stride, min_texture)
    fin = st.collect_support(frame, rig, params, threshold, stride=stride,
                             min_texture=min_texture)
    k = len(rig)
    cams = [rig.cameras[i] for i in range(k)]
    out.update({
        f"{name}_images": np.stack(frame.images), f"{name}_priors": np.stack(frame.priors),
        f"{name}_fx": np.array([c[0].fx for c in cams]), f"{name}_fy": np.array([c[0].fy for c in cams]),
        f"{name}_cx": np.array([c[0].cx for c in cams]), f"{name}_cy": np.array([c[0].cy for c in cams]),
        f"{name}_rot": np.stack([c[1].rotation for c in cams]),
        f"{name}_trans": np.stack([c[1].translation for c in cams]),
        f"{name}_scalars": np.array([rig.unit_baseline, rig.ref_index, d_max, threshold, stride,
                                     min_texture]),
        f"{name}_nn": np.array([rig.nearest_neighbor(i) for i in range(k)], np.int32),
    })
    for tag, pts in (("col", col), ("fin", fin)):
        u, v, d, s = arrays(pts)
        out.update({f"{name}_{tag}_u": u, f"{name}_{tag}_v": v, f"{name}_{tag}_d": d,
                    f"{name}_{tag}_src": s})
    print(f"{name}: {len(col)} collected, {len(fin)} kept "
          f"({sum(p.source_view != rig.ref_index for p in fin)} reprojected)", flush=True)


def main():
    out = {}
    spec = st.occluder_scene(width=160, height=120)
    frame, _ = st.render(spec)
    rig = spec.rig()
    case(out, "occ160", frame, rig)
    case(out, "occ160_tilt", frame, tilted_rig(rig, 5))
    case(out, "occ160_focal", frame, mixed_focal_rig(rig, 9))
    case(out, "occ160_s3", frame, rig, stride=3, min_texture=10.0, d_max=30.3)
    spec = st.occluder_scene(width=200, height=150, cameras=4, seed=5, p_flip=0.1,
                             blur_radius=2)
    frame, _ = st.render(spec)
    case(out, "occ200_k4", frame, spec.rig(), d_max=32.0)
    spec = st.occluder_scene(width=128, height=96, cameras=9, p_flip=0.1, blur_radius=1)
    frame, _ = st.render(spec)
    case(out, "occ128_k9", frame, spec.rig(), d_max=48.0)
    spec = st.low_texture_scene(width=160, height=120)
    frame, _ = st.render(spec)
    case(out, "low160", frame, spec.rig())
    path = os.path.join(HERE, "harvest_cases.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
