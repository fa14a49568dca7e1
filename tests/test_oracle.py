"""Pin the CPU oracle to the reference: bit-exact on every golden fixture.

CPU-only (no GPU marker).  The fixtures were produced by the reference
itself (tests/golden/make_golden.py); when /root/reference is present the
oracle is also compared against it live on fresh seeds.
"""

import numpy as np
import pytest

import oracle
from golden_io import SCENES, cases, load, oracle_solver, support


def test_estep_cases_exact():
    z = cases("estep_cases")
    p = oracle.OracleParams()
    for k in (5, 3, 4, 9):
        got = oracle.e_step(z[f"k{k}_desc"].astype(np.float64), z[f"k{k}_valid"], z[f"k{k}_q"], p)
        assert np.array_equal(got, z[f"k{k}_out"]), k


def test_bilinear_cases_bit_exact():
    z = cases("sampling_cases")
    for i in range(5):
        got = oracle.bilinear(z[f"b{i}_img"], z[f"b{i}_u"], z[f"b{i}_v"])
        want = z[f"b{i}_out"]
        assert got.dtype == np.float64
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), i


def test_descriptors_and_median_exact():
    z = cases("sampling_cases")
    for im, g, d in zip(z["desc_images"], z["desc_gray"], z["desc_out"]):
        assert np.array_equal(oracle.gray_of(im), g)
        assert np.array_equal(oracle.descriptors_of(im), d)
    assert np.array_equal(oracle.median_filter(z["median_in"], 1), z["median_r1"])
    assert np.array_equal(oracle.median_filter(z["median_in"], 2), z["median_r2"])


@pytest.mark.parametrize("name", SCENES)
def test_scene_bit_exact(name):
    g = load(name)
    h, w = g["images"].shape[1:3]
    uv, _ = support(g)
    mu = oracle.mu_raster(g["tri_points"], g["tri_disp"], g["tri_triangles"], g["tri_planes"], w, h)
    assert np.array_equal(mu, g["mu_raw"])
    s = oracle_solver(g)
    allp = np.arange(h * w, dtype=np.int64)
    s0, v0 = s.initial_masks(allp)
    assert np.array_equal(s0, g["init_static"]) and np.array_equal(v0, g["init_valid"])
    d1, e1, st1, _ = s.m_step(allp, s0)
    assert np.array_equal(st1, g["m1_status"])
    assert np.array_equal(d1, g["m1_d"], equal_nan=True)
    assert np.array_equal(e1, g["m1_e"])
    s1, v1 = s.e_step_at(g["e1_pix"], d1[g["e1_pix"]])
    assert np.array_equal(s1, g["e1_static"]) and np.array_equal(v1, g["e1_valid"])
    for tag, dyn in (("full", False), ("dyn", True)):
        r = s.solve(dynamic_only=dyn)
        assert np.array_equal(r["values"], g[f"{tag}_values"])
        assert np.array_equal(r["status"], g[f"{tag}_status"])
        assert np.array_equal(r["static_bits"], g[f"{tag}_static"])
        assert np.array_equal(r["valid_bits"], g[f"{tag}_valid"])
        assert r["stats"] == g[f"{tag}_stats"]
        copy = (g["priors"][int(g["ref_index"])] >= s.p.threshold) if dyn else None
        for rad in (0, 1):
            img, prov, nr = oracle.synthesize(list(g["images"]), g["warp_a"], g["warp_b"],
                                              int(g["ref_index"]), r["values"], r["status"],
                                              r["static_bits"], s.p.min_static_rays, rad, copy)
            assert np.array_equal(img, g[f"{tag}_synth{rad}_img"])
            assert np.array_equal(prov, g[f"{tag}_synth{rad}_prov"])
            assert np.array_equal(nr, g[f"{tag}_synth{rad}_nrays"])


def test_margins_are_positive_and_consistent():
    g = load("occ160_noisy")
    s = oracle_solver(g)
    h, w = g["images"].shape[1:3]
    allp = np.arange(h * w, dtype=np.int64)
    s0, _ = s.initial_masks(allp)
    d, e, m = s.m_margins(allp, s0)
    # the margin harness picks the same winner as the pruned M-step
    assert np.array_equal(d, g["m1_d"], equal_nan=True)
    assert np.array_equal(e, g["m1_e"])
    assert (m >= 0).all()


def test_oracle_matches_live_reference(reference):
    st = reference
    spec = st.occluder_scene(width=96, height=72, seed=13, p_flip=0.1, blur_radius=1)
    frame, gt = st.render(spec)
    rig = spec.rig()
    sup = st.collect_support(frame, rig, st.PriorParams(), threshold=0.7)
    tri = st.triangulate(sup, spec.width, spec.height)
    dmap, seg, stats = st.em_solve(frame, rig, tri)
    pts, disps = tri.support_points()
    a = np.stack([rig.warp_coefficients(k)[0] for k in range(len(rig))])
    b = np.stack([rig.warp_coefficients(k)[1] for k in range(len(rig))])
    s = oracle.OracleSolver(frame.images, frame.priors, a, b, rig.ref_index,
                            tri.disparity_map(spec.width, spec.height), pts, disps)
    r = s.solve()
    assert np.array_equal(r["values"], dmap.values)
    assert np.array_equal(r["static_bits"], seg.static_bits)
    assert np.array_equal(r["valid_bits"], seg.valid_bits)
    assert r["stats"]["mean_energy"] == stats.mean_energy


def test_numpy_sum_order_is_numpys():
    """The summation order the device statistics replay (st_mean.cu) is
    numpy's own: identity start + pairwise blocks (discriminated against the
    first-element start on arrays where the two differ)."""
    import oracle
    rng = np.random.default_rng(7)
    for n in list(range(0, 40)) + [127, 128, 129, 255, 256, 257, 1000, 4097, 20011]:
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)
        assert oracle.numpy_sum_order(x) == np.add.reduce(x), n
        if n:
            assert oracle.numpy_sum_order(x) / n == x.mean(), n
    assert str(oracle.numpy_sum_order(np.array([-0.0]))) == str(np.add.reduce(np.array([-0.0])))
