"""Parity at BASELINE.json's sizes.

C1 (640x480, K=5, d_max 32): the GPU path against the CPU oracle on the
same reference-identical inputs (renderer port checked against recorded
digests; support recorded from the reference's harvest), whole frame.
C2 (1280x720, d_max 64): size-independent properties -- determinism, the
reference's dynamic_only == full-solve-on-active-pixels identity, banded ==
full, forced iterations extend the reference iterations.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    import paper_2003_11076_b200 as pkg
    pkg.device.require_cuda()
    return pkg


def bench_inputs(cfg):
    import bench
    return bench.load_inputs(cfg)


def _inputs(cfg):
    import bench
    frame, rig, tri, exact = bench.load_inputs(cfg)
    assert exact, "renderer port no longer reproduces the reference frame"
    sp, pp = bench.params_for(cfg)
    return frame, rig, tri, sp, pp


@pytest.mark.slow
def test_c1_full_frame_matches_oracle(st):
    import oracle
    frame, rig, tri, sp, pp = _inputs("C1")
    r = st.reconstruct(frame, rig, tri, sp, pp)
    k = len(rig)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    sup_uv, sup_d = tri.support_points()
    mu = oracle.mu_raster(tri.points, tri.disparities, tri.triangles, tri.planes, 640, 480)
    p = oracle.OracleParams(d_max=pp.d_max, max_iters=sp.max_iters)
    o = oracle.OracleSolver(frame.images, frame.priors, a, b, rig.ref_index, mu, sup_uv, sup_d,
                            params=p)
    want = o.solve()
    img, prov, nr = oracle.synthesize(frame.images, a, b, rig.ref_index, want["values"],
                                      want["status"], want["static_bits"])
    assert r.stats.iterations_run == want["stats"]["iterations_run"]
    assert r.stats.converged_after == want["stats"]["converged_after"]
    agree = (r.disparity.values == want["values"]).mean()
    assert agree >= 0.999, agree
    assert (r.disparity.status == want["status"]).mean() >= 0.999
    assert (r.segmentation.static_bits == want["static_bits"]).mean() >= 0.999
    assert (r.segmentation.valid_bits == want["valid_bits"]).mean() >= 0.999
    assert (r.image == img).all(axis=2).mean() >= 0.999
    assert (r.provenance == prov).mean() >= 0.999
    assert np.allclose(r.stats.mean_energy, want["stats"]["mean_energy"], rtol=1e-9)
    # report exact agreement for the record
    print(f"C1 parity: values {agree:.6f}, image {(r.image == img).all(axis=2).mean():.6f}")


def test_c2_properties(st):
    frame, rig, tri, sp, pp = _inputs("C2")
    a = st.reconstruct(frame, rig, tri, sp, pp)
    b = st.reconstruct(frame, rig, tri, sp, pp)
    # byte-identical artefacts run to run (test_acceptance.py:310-332)
    for x, y in ((a.disparity.values, b.disparity.values), (a.image, b.image),
                 (a.segmentation.static_bits, b.segmentation.static_bits)):
        assert np.array_equal(x, y)
    assert a.stats.mean_energy == b.stats.mean_energy
    # dynamic_only solves exactly the full solve's values on the active
    # pixels (test_solver.py:323-337)
    dyn = st.reconstruct(frame, rig, tri, sp, pp, dynamic_only=True)
    active = frame.priors[rig.ref_index] < np.float32(sp.threshold)
    assert active.any()
    assert np.array_equal(dyn.disparity.values[active], a.disparity.values[active])
    assert np.array_equal(dyn.segmentation.static_bits[active],
                          a.segmentation.static_bits[active])
    assert (dyn.provenance[~active] == st.PROV_COPIED).all()
    # static rays are a subset of valid rays
    assert not (a.segmentation.static_bits & ~a.segmentation.valid_bits).any()
    # forcing more iterations keeps the reference iterations' statistics
    f = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=5)
    assert f.stats.iterations_run == 5
    assert np.allclose(f.stats.mean_energy[:a.stats.iterations_run], a.stats.mean_energy,
                       rtol=1e-12)
    # energy descent (test_solver.py:305-320)
    for i, prev in enumerate(f.stats.prev_energy):
        assert f.stats.mean_energy[i + 1] <= prev + 1e-9


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_screened_em_equals_exhaustive(st, monkeypatch, cfg):
    """The fp32-screened E-step and the pruned M-step decide exactly what
    evaluating every mask / every candidate in fp64 decides (st_em.cu
    estep_small; k_m_step's prior-bound and hopeless-pixel radii), whole
    frame."""
    frame, rig, tri, sp, pp = _inputs(cfg)
    a = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=5)
    monkeypatch.setenv("ST_ESTEP_EXHAUSTIVE", "1")
    monkeypatch.setenv("ST_MSTEP_EXHAUSTIVE", "1")
    b = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=5)
    assert np.array_equal(a.segmentation.static_bits, b.segmentation.static_bits)
    assert np.array_equal(a.segmentation.valid_bits, b.segmentation.valid_bits)
    assert np.array_equal(a.disparity.values, b.disparity.values)
    assert np.array_equal(a.image, b.image)
    assert list(a.stats.mean_energy) == list(b.stats.mean_energy)


@pytest.mark.parametrize("forced", [0, 5])
def test_async_solve_equals_sync(st, forced):
    """st_solve_async (device-side convergence test and statistics, no host
    round trip) == st_solve, outputs and EMStats."""
    from paper_2003_11076_b200.prior import TriDevice
    from paper_2003_11076_b200.reconstruct import AsyncStats, FramePipeline, _outputs_of
    frame, rig, tri, sp, pp = _inputs("C2")
    h, w = frame.shape
    pipe = FramePipeline(rig, w, h, sp, pp)
    td = TriDevice(tri)
    res = []
    for timing in (True, False):
        pipe.load(frame.images, frame.priors)
        stats = pipe.run(td, forced_iters=forced, timing=timing)
        assert isinstance(stats, AsyncStats) == (not timing)
        res.append(_outputs_of(pipe, stats, pipe.fetch()))
    a, b = res
    for x, y in ((a.disparity.values, b.disparity.values), (a.disparity.status, b.disparity.status),
                 (a.segmentation.static_bits, b.segmentation.static_bits),
                 (a.segmentation.valid_bits, b.segmentation.valid_bits), (a.image, b.image)):
        assert np.array_equal(x, y)
    for f in ("iterations_run", "converged_after", "changed_fraction", "candidates_total",
              "energy_evals", "msteps", "esteps", "prev_evals", "active_pixels"):
        assert getattr(a.stats, f) == getattr(b.stats, f), f
    # the synchronous path sums the energies in a fixed order, the
    # asynchronous one replays numpy's pairwise order (st_mean.cu)
    for f in ("mean_energy", "prev_energy"):
        np.testing.assert_allclose(getattr(a.stats, f), getattr(b.stats, f), rtol=1e-12)


@pytest.mark.slow
def test_c4_mu_raster_bit_exact_incl_off_hull_pixels(st):
    """C4 (3840x2160, 296k support points): the raster walk leaves a few
    interior pixels near the top edge outside the triangulation, exactly as
    scipy's find_simplex does; the reference then re-queries them nudged
    1e-9 toward the centroid (prior.py:287-293).  The device raster
    (k_mu_nudge) must reproduce the reference's surface bit for bit."""
    import oracle
    frame, rig, tri, exact = bench_inputs("C4")
    h, w = frame.shape
    got = st.TriangulationPrior(tri.points, tri.disparities, tri.triangles, tri.planes,
                                tri.num_anchors).disparity_map(w, h)
    want = oracle.mu_raster(tri.points, tri.disparities, tri.triangles, tri.planes, w, h)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), int((got != want).sum())


@pytest.mark.parametrize("cfg,forced,max_iters,dyn", [
    ("C2", 0, None, False), ("C2", 9, None, False), ("C3", 0, None, False),
    ("C2", 0, 200, False), ("C2", 0, None, True), ("C2", 6, None, True)])
def test_graph_tail_equals_launch_loop(st, monkeypatch, cfg, forced, max_iters, dyn):
    """Iterations >= 3 as a CUDA-graph WHILE loop (st_api.cu run_tail_graph,
    the statistics kernel sets the condition) == the plain launch loop
    (ST_NO_GRAPH), outputs and EMStats bit for bit, with the reference's
    convergence test, forced iterations, a long cap and dynamic_only (the
    row-band driver, one shard: the active count stays on the device and
    k_band_control sets the condition)."""
    import dataclasses
    from paper_2003_11076_b200 import _native as N
    frame, rig, tri, sp, pp = _inputs(cfg)
    if max_iters:
        sp = dataclasses.replace(sp, max_iters=max_iters)
    lib = N.lib()
    l0 = lib.st_tail_graph_count(1)
    a = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=forced, dynamic_only=dyn)
    b0 = lib.st_tail_graph_count(0)
    a2 = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=forced, dynamic_only=dyn)
    assert lib.st_tail_graph_count(0) == b0, "the second solve did not reuse the cached graph"
    l1 = lib.st_tail_graph_count(1)
    assert l1 == l0 + 2, "the graph loop did not run"
    monkeypatch.setenv("ST_NO_GRAPH", "1")
    b = st.reconstruct(frame, rig, tri, sp, pp, forced_iters=forced, dynamic_only=dyn)
    assert lib.st_tail_graph_count(1) == l1
    for r in (a, a2):
        for x, y in ((r.disparity.values, b.disparity.values),
                     (r.disparity.status, b.disparity.status),
                     (r.segmentation.static_bits, b.segmentation.static_bits),
                     (r.segmentation.valid_bits, b.segmentation.valid_bits), (r.image, b.image)):
            assert np.array_equal(x, y)
        assert repr(r.stats) == repr(b.stats)
    if forced:
        assert a.stats.iterations_run == forced


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_dynamic_only_device_count_equals_readback(st, monkeypatch, cfg):
    """dynamic_only with the active count kept on the device (one shard, no
    host read-back, st_solve_rows) == the read-back path
    (ST_DYNAMIC_READBACK), outputs and EMStats bit for bit."""
    frame, rig, tri, sp, pp = _inputs(cfg)
    a = st.reconstruct(frame, rig, tri, sp, pp, dynamic_only=True)
    monkeypatch.setenv("ST_DYNAMIC_READBACK", "1")
    monkeypatch.setenv("ST_NO_GRAPH", "1")
    b = st.reconstruct(frame, rig, tri, sp, pp, dynamic_only=True)
    for x, y in ((a.disparity.values, b.disparity.values),
                 (a.disparity.status, b.disparity.status),
                 (a.segmentation.static_bits, b.segmentation.static_bits),
                 (a.segmentation.valid_bits, b.segmentation.valid_bits), (a.image, b.image),
                 (a.provenance, b.provenance)):
        assert np.array_equal(x, y)
    assert repr(a.stats) == repr(b.stats)
