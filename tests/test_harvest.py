"""Support harvest (prior.py:51-260): oracle pinned to the reference's
fixtures on CPU; the device harvest (st_harvest) + native dedup
(st_support_dedup) bit-exact against the same fixtures and, at BASELINE.json's
sizes, against the support lists the reference harvested for C1-C4."""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["occ160", "occ160_tilt", "occ160_focal", "occ160_s3", "occ200_k4", "occ128_k9",
         "low160"]


@pytest.fixture(scope="module")
def fx():
    return np.load(os.path.join(HERE, "golden", "harvest_cases.npz"))


def _scal(fx, name):
    ub, ref, d_max, thr, stride, mt = fx[f"{name}_scalars"]
    return float(ub), int(ref), float(d_max), float(thr), int(stride), float(mt)


def _points(fx, name, tag):
    return list(zip(fx[f"{name}_{tag}_u"].tolist(), fx[f"{name}_{tag}_v"].tolist(),
                    fx[f"{name}_{tag}_d"].tolist(), fx[f"{name}_{tag}_src"].tolist()))


def _oracle_cams(fx, name):
    from oracle.harvest import Cameras
    ub, ref, *_ = _scal(fx, name)
    h, w = fx[f"{name}_priors"].shape[1:]
    return Cameras(fx[f"{name}_fx"], fx[f"{name}_fy"], fx[f"{name}_cx"], fx[f"{name}_cy"],
                   fx[f"{name}_rot"], fx[f"{name}_trans"], ub, ref, w, h)


def _rig(fx, name):
    from paper_2003_11076_b200.geometry import CameraExtrinsics, CameraIntrinsics, CameraRig
    ub, ref, *_ = _scal(fx, name)
    h, w = fx[f"{name}_priors"].shape[1:]
    cams = []
    for i in range(fx[f"{name}_fx"].shape[0]):
        intr = CameraIntrinsics(fx=float(fx[f"{name}_fx"][i]), fy=float(fx[f"{name}_fy"][i]),
                                cx=float(fx[f"{name}_cx"][i]), cy=float(fx[f"{name}_cy"][i]),
                                width=int(w), height=int(h))
        cams.append((intr, CameraExtrinsics(fx[f"{name}_rot"][i], fx[f"{name}_trans"][i])))
    return CameraRig(cams, ref_index=ref, unit_baseline=ub)


# -- CPU: the oracle against the reference's fixtures --------------------------

@pytest.mark.parametrize("name", CASES)
def test_oracle_harvest_matches_reference(fx, name):
    import oracle
    from oracle import harvest as H
    ub, ref, d_max, thr, stride, mt = _scal(fx, name)
    cams = _oracle_cams(fx, name)
    assert [cams.nearest_neighbor(i) for i in range(len(cams))] == fx[f"{name}_nn"].tolist()
    descs = [oracle.descriptors_of(im) for im in fx[f"{name}_images"]]
    got = H.collect_support(descs, list(fx[f"{name}_priors"]), cams, d_max, thr, stride, mt)
    assert got == _points(fx, name, "fin")


@pytest.mark.parametrize("name", CASES)
def test_oracle_dedup_matches_reference(fx, name):
    from oracle import harvest as H
    _, ref, *_ = _scal(fx, name)
    assert H.deduplicate(_points(fx, name, "col"), ref) == _points(fx, name, "fin")


def _native_dedup(points, ref, w, h):
    from paper_2003_11076_b200.prior import deduplicate_arrays
    u, v, d, s = (np.array(x) for x in zip(*points)) if points else ([], [], [], [])
    return [points[i] for i in deduplicate_arrays(u, v, d, s, ref, w, h)]


@pytest.mark.parametrize("name", CASES)
def test_native_dedup_matches_reference(fx, name):
    """st_support_dedup is host code in the library (no device needed)."""
    _, ref, *_ = _scal(fx, name)
    h, w = fx[f"{name}_priors"].shape[1:]
    assert _native_dedup(_points(fx, name, "col"), ref, w, h) == _points(fx, name, "fin")


def test_native_dedup_random_conflicts():
    """Dense colliding / conflicting points, duplicate keys (stable order)."""
    from oracle import harvest as H
    rng = np.random.default_rng(7)
    for trial in range(20):
        n = int(rng.integers(1, 400))
        pts = [(int(rng.integers(0, 12)), int(rng.integers(0, 9)),
                float(rng.choice([1.0, 2.0, 2.5, 3.0, 4.5, 7.0, 9.25])), int(rng.integers(0, 4)))
               for _ in range(n)]
        ref = int(rng.integers(0, 4))
        assert _native_dedup(pts, ref, 12, 9) == H.deduplicate(pts, ref), trial


# -- GPU: device harvest against the fixtures ----------------------------------

@pytest.fixture(scope="module")
def st():
    import paper_2003_11076_b200 as pkg
    pkg.device.require_cuda()
    return pkg


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_harvest_matches_reference(st, fx, name):
    from paper_2003_11076_b200.prior import harvest_device
    ub, ref, d_max, thr, stride, mt = _scal(fx, name)
    rig = _rig(fx, name)
    assert [rig.nearest_neighbor(i) for i in range(len(rig))] == fx[f"{name}_nn"].tolist()
    frame = st.LightFieldFrame(images=list(fx[f"{name}_images"]),
                               priors=list(fx[f"{name}_priors"]))
    pp = st.PriorParams(d_max=d_max)
    u, v, d, s = harvest_device(frame, rig, pp, thr, stride, mt)
    got = list(zip(u.tolist(), v.tolist(), d.tolist(), s.tolist()))
    assert got == _points(fx, name, "col")
    fin = st.collect_support(frame, rig, pp, thr, stride=stride, min_texture=mt)
    assert [(p.u, p.v, p.d, p.source_view) for p in fin] == _points(fx, name, "fin")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", pytest.param("C4", marks=pytest.mark.slow)])
def test_device_harvest_full_size(st, cfg):
    """The reference's own support lists at BASELINE.json's sizes."""
    import bench
    frame, rig, _, exact = bench.load_inputs(cfg)
    assert exact
    _, pp = bench.params_for(cfg)
    z = np.load(os.path.join(HERE, "golden", f"bench_{cfg}.npz"))
    fin = st.collect_support(frame, rig, pp, 0.7)
    assert len(fin) == z["support_d"].shape[0]
    assert np.array_equal(np.array([[p.u, p.v] for p in fin]), z["support_uv"])
    assert np.array_equal(np.array([p.d for p in fin]), z["support_d"])
    assert np.array_equal(np.array([p.source_view for p in fin]), z["support_src"])


@pytest.mark.gpu
def test_frame_in_path_matches_reference_inputs(st):
    """reconstruct_frame (device harvest -> native dedup -> host Qhull ->
    device planes/transforms -> solve -> refocus) reproduces the
    triangulation built from the reference's own support list and the
    outputs of reconstruct() on it; reconstruct_frames streams the same."""
    import bench
    frame, rig, tri_ref, exact = bench.load_inputs("C1")
    assert exact
    sp, pp = bench.params_for("C1")
    rec, tri = st.reconstruct_frame(frame, rig, sp, pp)
    assert np.array_equal(tri.points, tri_ref.points)
    assert np.array_equal(tri.disparities, tri_ref.disparities)
    assert np.array_equal(tri.triangles, tri_ref.triangles)
    ref = st.reconstruct(frame, rig, tri_ref, sp, pp)
    for a, b in ((rec.disparity.values, ref.disparity.values), (rec.image, ref.image),
                 (rec.segmentation.static_bits, ref.segmentation.static_bits),
                 (rec.provenance, ref.provenance), (rec.n_rays, ref.n_rays)):
        assert np.array_equal(a, b)
    assert rec.stats.mean_energy == ref.stats.mean_energy
    outs = list(st.reconstruct_frames([frame] * 3, rig, sp, pp, workers=2))
    assert len(outs) == 3
    for o in outs:
        assert np.array_equal(o.disparity.values, ref.disparity.values)
        assert np.array_equal(o.image, ref.image)


@pytest.mark.gpu
def test_stream_equals_single_calls(st):
    """reconstruct_stream (native st_frame_run path, and the Python path for
    dynamic_only) == reconstruct() frame by frame."""
    import bench
    frame, rig, tri, _ = bench.load_inputs("C1")
    sp, pp = bench.params_for("C1")
    for dyn in (False, True):
        ref = st.reconstruct(frame, rig, tri, sp, pp, dynamic_only=dyn)
        outs = list(st.reconstruct_stream([(frame, tri)] * 4, rig, sp, pp, dynamic_only=dyn))
        assert len(outs) == 4
        for o in outs:
            for a, b in ((o.disparity.values, ref.disparity.values), (o.image, ref.image),
                         (o.segmentation.static_bits, ref.segmentation.static_bits),
                         (o.segmentation.valid_bits, ref.segmentation.valid_bits),
                         (o.provenance, ref.provenance)):
                assert np.array_equal(a, b)
            assert o.stats.iterations_run == ref.stats.iterations_run
            assert o.stats.mean_energy == ref.stats.mean_energy
