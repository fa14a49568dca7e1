"""st_tri_tables: the planes (np.linalg.solve, prior.py:351-357) and scipy's
barycentric transforms recomputed on the device -- bit-exact against the
host libraries on every golden triangulation, NaN rows for flat triangles,
numpy's singular-system error surfaced through TriDevice.check."""

import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def st():
    import paper_2003_11076_b200 as pkg
    pkg.device.require_cuda()
    return pkg


def _same(a, b):
    return np.array_equal(a, b) or bool(np.all((a == b) | (np.isnan(a) & np.isnan(b))))


def _check(tri):
    from paper_2003_11076_b200.prior import TriDevice, delaunay_of
    td = TriDevice(tri)
    assert td.device_tables
    planes = td.planes.cpu().numpy().reshape(-1, 3)
    transform = td.transform.cpu().numpy().reshape(-1, 3, 2)
    assert _same(planes, np.asarray(tri.planes)), "planes differ from np.linalg.solve"
    assert _same(transform, delaunay_of(tri).transform), "transforms differ from scipy"
    td.check()


def _scene_tris():
    from paper_2003_11076_b200.prior import triangulate, SupportPoint
    for path in sorted(glob.glob(os.path.join(HERE, "golden", "scene_*.npz"))):
        z = np.load(path)
        n = z["tri_points"].shape[0] - int(z["tri_num_anchors"])
        h, w = z["priors"].shape[1:]
        pts = [SupportPoint(int(u), int(v), float(d), 0)
               for (u, v), d in zip(z["tri_points"][:n], z["tri_disp"][:n])]
        yield os.path.basename(path), triangulate(pts, w, h)


def test_tables_match_host_on_golden_scenes(st):
    for name, tri in _scene_tris():
        _check(tri)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_tables_match_host_at_full_size(st, cfg):
    import bench
    _, _, tri, _ = bench.load_inputs(cfg)
    _check(tri)


def test_flat_triangles_and_random_grids(st):
    """Dense integer grids (many cocircular sets -> Qhull's flat simplices)
    and random integer clouds, against numpy / scipy."""
    from paper_2003_11076_b200.prior import SupportPoint, triangulate
    rng = np.random.default_rng(5)
    for trial in range(6):
        if trial < 3:
            xs, ys = np.meshgrid(np.arange(0, 60, 5 + trial), np.arange(0, 40, 4 + trial))
            uv = np.stack([xs.ravel(), ys.ravel()], 1)
        else:
            uv = np.unique(rng.integers(0, 300, size=(400, 2)), axis=0)
        d = rng.uniform(0.5, 60, size=uv.shape[0])
        pts = [SupportPoint(int(a), int(b), float(c), 0) for (a, b), c in zip(uv, d)]
        _check(triangulate(pts, 300, 200))


def test_singular_plane_raises(st):
    """A system whose LU hits an exact zero pivot: numpy raises LinAlgError
    (triangulate -> ValueError); the device path reports the same error."""
    import types
    from paper_2003_11076_b200.prior import TriDevice
    from scipy.spatial import Delaunay
    pts = np.array([[0.0, 0.0], [10.0, 0.0], [0.0, 10.0], [10.0, 10.0], [5.0, 5.0]])
    dl = Delaunay(pts)
    tris = dl.simplices.astype(np.int32).copy()
    tris[0] = [0, 4, 3]  # collinear vertices (0,0), (5,5), (10,10)
    mats = np.concatenate([pts[tris], np.ones((tris.shape[0], 3, 1))], axis=2)
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.solve(mats, np.ones((tris.shape[0], 3, 1)))
    fake = types.SimpleNamespace(points=pts, disparities=np.ones(5), triangles=tris,
                                 planes=None, num_anchors=0, _lookup=dl,
                                 support_points=lambda: (pts, np.ones(5)))
    td = TriDevice(fake)
    with pytest.raises(ValueError, match="zero-area triangle"):
        td.check()
    assert np.isnan(td.transform.cpu().numpy().reshape(-1, 6)[0]).all()
