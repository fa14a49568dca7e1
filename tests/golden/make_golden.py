"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container only (the reference is not on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports `seethrough` from /root/reference/pkg/src, renders seeded scenes
with the reference renderer (synth.py:244-309), harvests support with the
reference (prior.py:233-260, 318-360), solves with the reference
(solver.py:505-508, refocus.py:109-148) and stores inputs + outputs as
compressed .npz.  Nothing here is product code.
"""

import json
import os
import sys

import numpy as np

REF_SRC = os.environ.get("SEETHROUGH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
import seethrough as st  # noqa: E402
from seethrough.geometry import CameraExtrinsics, CameraRig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _rot(axis, angle):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    kx, ky, kz = axis
    k = np.array([[0.0, -kz, ky], [kz, 0.0, -kx], [-ky, kx, 0.0]])
    return np.eye(3) + np.sin(angle) * k + (1.0 - np.cos(angle)) * (k @ k)


def rig_arrays(rig):
    k = len(rig)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    dims = np.array([[rig.intrinsics(i).height, rig.intrinsics(i).width] for i in range(k)])
    return a, b, dims


def stats_json(stats):
    return json.dumps(dict(iterations_run=stats.iterations_run,
                           converged_after=stats.converged_after,
                           mean_energy=stats.mean_energy,
                           prev_energy=stats.prev_energy,
                           changed_fraction=stats.changed_fraction))


def scene_fixture(name, frame, rig, tri, prior_params=None, solver_params=None):
    h, w = frame.shape
    pp = prior_params or st.PriorParams()
    sp = solver_params or st.SolverParams()
    a, b, dims = rig_arrays(rig)
    out = dict(
        images=np.stack(frame.images), priors=np.stack(frame.priors),
        warp_a=a, warp_b=b, dims=dims, ref_index=np.int64(rig.ref_index),
        tri_points=tri.points, tri_disp=tri.disparities, tri_triangles=tri.triangles,
        tri_planes=tri.planes, tri_num_anchors=np.int64(tri.num_anchors),
        mu_raw=tri.disparity_map(w, h),
        params=json.dumps(dict(beta=sp.beta, threshold=sp.threshold, max_iters=sp.max_iters,
                               min_static_rays=sp.min_static_rays,
                               epsilon_prior=sp.epsilon_prior, sigma=pp.sigma,
                               gamma=pp.gamma, d_max=pp.d_max,
                               neighborhood_radius=pp.neighborhood_radius)),
    )
    solver = st.DisparitySolver(frame, rig, tri, params=sp, prior_params=pp)
    allp = np.arange(h * w, dtype=np.int64)
    s0, v0 = solver.initial_masks(allp)
    out.update(init_static=s0, init_valid=v0)
    d1, e1, st1 = solver.m_step(allp, s0)
    out.update(m1_d=d1, m1_e=e1, m1_status=st1)
    upd = allp[st1 != st.STATUS_LOW_TEXTURE]
    s1, v1 = solver.e_step_at(upd, d1[st1 != st.STATUS_LOW_TEXTURE])
    out.update(e1_pix=upd, e1_static=s1, e1_valid=v1)
    for tag, dyn in (("full", False), ("dyn", True)):
        dmap, seg, stats = st.em_solve(frame, rig, tri, params=sp, prior_params=pp,
                                       dynamic_only=dyn)
        out[f"{tag}_values"] = dmap.values
        out[f"{tag}_status"] = dmap.status
        out[f"{tag}_static"] = seg.static_bits
        out[f"{tag}_valid"] = seg.valid_bits
        out[f"{tag}_stats"] = stats_json(stats)
        copy = (frame.priors[rig.ref_index] >= sp.threshold) if dyn else None
        for r in (0, 1):
            img, prov, nr = st.synthesize(frame, rig, dmap, seg,
                                          min_static_rays=sp.min_static_rays,
                                          median_radius=r, copy_mask=copy)
            out[f"{tag}_synth{r}_img"] = img
            out[f"{tag}_synth{r}_prov"] = prov
            out[f"{tag}_synth{r}_nrays"] = nr
    path = os.path.join(HERE, f"scene_{name}.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


def rendered(spec):
    frame, gt = st.render(spec)
    rig = spec.rig()
    support = st.collect_support(frame, rig, st.PriorParams(), threshold=0.7)
    tri = st.triangulate(support, spec.width, spec.height)
    return frame, gt, rig, tri


def tilted_rig(rig, seed):
    """Same intrinsics, small random rotations + off-axis translations."""
    rng = np.random.default_rng(seed)
    cams = []
    for i in range(len(rig)):
        intr, extr = rig.cameras[i]
        if i == rig.ref_index:
            cams.append((intr, CameraExtrinsics.identity()))
            continue
        r = _rot(rng.normal(size=3), np.deg2rad(rng.uniform(0.2, 1.5)))
        t = extr.translation + rng.uniform(-0.01, 0.01, size=3)
        cams.append((intr, CameraExtrinsics(r, t)))
    return CameraRig(cams, ref_index=rig.ref_index, unit_baseline=rig.unit_baseline)


def estep_fixture():
    """Acceptance-3 style instances (test_acceptance.py:228-249) + K=3,4,9."""
    params = st.SolverParams()
    out = {}
    rng = np.random.default_rng(303)
    n = 10_000
    desc = rng.integers(0, 256, size=(n, 5, 16)).astype(np.float64)
    valid = rng.random((n, 5)) < 0.85
    prob = rng.random((n, 5))
    hard = rng.random((n, 5)) < 0.08
    prob[hard] = rng.integers(0, 2, size=int(hard.sum())).astype(np.float64)
    desc[-500:, 1] = desc[-500:, 0]
    prob[-500:, 1] = prob[-500:, 0]
    valid[-500:, 1] = valid[-500:, 0]
    out.update(k5_desc=desc.astype(np.uint8), k5_valid=valid, k5_q=prob,
               k5_out=st.e_step(desc, valid, prob, params))
    # fractional descriptors (bilinear-like) at K = 3, 4, 9
    for k, cnt in ((3, 500), (4, 500), (9, 600)):
        r = np.random.default_rng(400 + k)
        d = np.round(r.uniform(0, 255, size=(cnt, k, 16)) * 64) / 64
        v = r.random((cnt, k)) < 0.85
        q = r.random((cnt, k)).astype(np.float32).astype(np.float64)
        d[-50:, 2] = d[-50:, 1]
        q[-50:, 2] = q[-50:, 1]
        v[-50:, 2] = v[-50:, 1]
        out.update({f"k{k}_desc": d, f"k{k}_valid": v, f"k{k}_q": q,
                    f"k{k}_out": st.e_step(d, v, q, params)})
    path = os.path.join(HERE, "estep_cases.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


def sampling_fixture():
    """bilinear (sampling.py:21-55) and descriptors (features.py:81-104)."""
    from seethrough.sampling import bilinear, flatten_channels
    rng = np.random.default_rng(21)
    out = {}
    for i, (h, w, c) in enumerate(((9, 13, 1), (17, 11, 3), (24, 40, 16), (1, 7, 2), (6, 1, 1))):
        img = rng.uniform(0, 255, size=(h, w, c)).astype(np.float32)
        if i == 2:
            img = np.rint(img).astype(np.float32)
        u = rng.uniform(-2, w + 2, size=300)
        v = rng.uniform(-2, h + 2, size=300)
        u[:40] = np.floor(u[:40])
        v[40:80] = np.floor(v[40:80])
        u[80:84] = [np.nan, np.inf, -np.inf, 0.0]
        flat, fh, fw = flatten_channels(img)
        out[f"b{i}_img"] = img
        out[f"b{i}_u"] = u
        out[f"b{i}_v"] = v
        out[f"b{i}_out"] = bilinear(flat, fh, fw, u, v)
    imgs = rng.integers(0, 256, size=(3, 37, 53, 3), dtype=np.uint8)
    imgs[2, :, :20] = 200
    out["desc_images"] = imgs
    out["desc_gray"] = np.stack([st.rgb_to_gray(im) for im in imgs])
    out["desc_out"] = np.stack([st.compute_descriptors(im).data for im in imgs])
    med = rng.integers(0, 256, size=(23, 31, 3), dtype=np.uint8)
    out["median_in"] = med
    out["median_r1"] = st.median_filter(med, 1)
    out["median_r2"] = st.median_filter(med, 2)
    path = os.path.join(HERE, "sampling_cases.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


def main():
    estep_fixture()
    sampling_fixture()
    frame, gt, rig, tri = rendered(st.occluder_scene(width=160, height=120))
    scene_fixture("occ160", frame, rig, tri)
    scene_fixture("occ160_tilt", frame, tilted_rig(rig, 5), tri)
    frame, gt, rig, tri = rendered(st.occluder_scene(width=160, height=120, p_flip=0.1,
                                                     blur_radius=2))
    scene_fixture("occ160_noisy", frame, rig, tri)
    frame, gt, rig, tri = rendered(st.two_plane_scene(width=160, height=120))
    scene_fixture("two160", frame, rig, tri)
    frame, gt, rig, tri = rendered(st.low_texture_scene(width=160, height=120))
    scene_fixture("low160", frame, rig, tri)
    frame, gt, rig, tri = rendered(st.occluder_scene(width=128, height=96, cameras=9,
                                                     p_flip=0.1, blur_radius=1))
    scene_fixture("occ128_k9", frame, rig, tri, prior_params=st.PriorParams(d_max=128.0),
                  solver_params=st.SolverParams(max_iters=10))
    frame, gt, rig, tri = rendered(st.occluder_scene(width=320, height=240, p_flip=0.1,
                                                     blur_radius=2))
    scene_fixture("occ320_noisy", frame, rig, tri)


if __name__ == "__main__":
    main()
