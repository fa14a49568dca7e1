"""Edge shapes through the whole device path, checked against the CPU oracle.

The golden scenes and the benchmark configs use 4:3 / 16:9 frames with 5
or 9 views; these cases cover the other rig sizes the reference accepts
(K = 2 ... 12, solver.py:46, 129-131), odd and tiny frame sizes (partial
descriptor, support and median tiles, 1-pixel margins), a short disparity
range and a dynamic-only solve.  Each case renders a scene with the
renderer port, runs the device pipeline from the raw frame
(reconstruct_frame: device harvest -> dedup -> Qhull -> solve -> refocus),
and compares the solve and refocus against the oracle on the same
triangulation (parity criterion of BASELINE.json: exact where the margin
allows, >= 99.9 % overall).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # (width, height, views, d_max, dynamic_only)
    (48, 32, 2, 64.0, False),
    (61, 37, 3, 64.0, False),
    (96, 64, 4, 32.0, False),
    (80, 48, 6, 64.0, False),
    (72, 40, 7, 40.5, True),
    (64, 48, 12, 64.0, False),
    (33, 129, 5, 64.0, False),
    (20, 14, 5, 64.0, False),
    (40, 30, 9, 24.0, True),
]


@pytest.fixture(scope="module")
def st():
    import paper_2003_11076_b200 as pkg
    pkg.device.require_cuda()
    return pkg


@pytest.mark.parametrize("w,h,k,dmax,dyn", CASES)
def test_edge_shapes_match_oracle(st, w, h, k, dmax, dyn):
    import oracle
    from paper_2003_11076_b200.synth import occluder_scene, render
    spec = occluder_scene(width=w, height=h, cameras=k, coverage=0.25, seed=11 + k, p_flip=0.1,
                          blur_radius=1)
    frame, _ = render(spec)
    rig = spec.rig()
    sp = st.SolverParams()
    pp = st.PriorParams(d_max=dmax)
    r, tri = st.reconstruct_frame(frame, rig, sp, pp, dynamic_only=dyn)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    sup_uv, sup_d = tri.support_points()
    planes = tri.planes
    if planes is None:  # solved on the device by reconstruct_frame: numpy's here (prior.py:351-357)
        pts, tris = np.asarray(tri.points), np.asarray(tri.triangles)
        mats = np.concatenate([pts[tris], np.ones(tris.shape + (1,))], axis=2)
        planes = np.linalg.solve(mats, np.asarray(tri.disparities)[tris][:, :, None])[:, :, 0]
    mu = oracle.mu_raster(tri.points, tri.disparities, tri.triangles, planes, w, h)
    o = oracle.OracleSolver(frame.images, frame.priors, a, b, rig.ref_index, mu, sup_uv, sup_d,
                            params=oracle.OracleParams(d_max=dmax))
    want = o.solve(dynamic_only=dyn)
    copy = frame.priors[rig.ref_index] >= np.float32(sp.threshold) if dyn else None
    img, prov, nr = oracle.synthesize(frame.images, a, b, rig.ref_index, want["values"],
                                      want["status"], want["static_bits"], copy_mask=copy)
    assert r.stats.iterations_run == want["stats"]["iterations_run"]
    for got, ref in ((r.disparity.values, want["values"]), (r.disparity.status, want["status"]),
                     (r.segmentation.static_bits, want["static_bits"]),
                     (r.segmentation.valid_bits, want["valid_bits"]), (r.provenance, prov),
                     (r.n_rays, nr)):
        assert got.shape == ref.shape
        assert (got == ref).mean() >= 0.999, (got != ref).sum()
    assert (r.image == img).all(axis=2).mean() >= 0.999
