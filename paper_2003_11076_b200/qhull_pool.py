"""Host Delaunay stage of the frame-in pipeline, in worker processes.

triangulate (prior.py:318-360) is scipy Qhull -- sequential, ~0.2 s per
1280x720 frame -- so a stream of frames runs it in a pool of spawn-started
processes (they import numpy/scipy only) while the device harvests the next
frames and solves the previous ones.  Workers return only the tables the
device needs: vertices, disparities, simplices and the walk tables of
scipy's find_simplex; the planes and barycentric transforms are recomputed on
the device (st_tri_tables).
"""

import numpy as np


class WalkTables:
    """The attributes of a scipy Delaunay object that TriDevice reads."""

    def __init__(self, neighbors, equations, paraboloid_scale, paraboloid_shift, min_bound,
                 max_bound):
        self.neighbors = neighbors
        self.equations = equations
        self.paraboloid_scale = paraboloid_scale
        self.paraboloid_shift = paraboloid_shift
        self.min_bound = min_bound
        self.max_bound = max_bound


def delaunay_tables(u, v, d, width, height):
    """Worker: triangulate_arrays without the host plane solve."""
    from .prior import triangulate_arrays
    tri = triangulate_arrays(u, v, d, width, height, planes=False)
    dl = tri._lookup
    return dict(points=tri.points, disparities=tri.disparities, triangles=tri.triangles,
                num_anchors=int(tri.num_anchors),
                neighbors=np.ascontiguousarray(dl.neighbors, dtype=np.int32),
                equations=np.ascontiguousarray(dl.equations, dtype=np.float64),
                paraboloid_scale=float(dl.paraboloid_scale),
                paraboloid_shift=float(dl.paraboloid_shift),
                min_bound=np.array(dl.min_bound, dtype=np.float64),
                max_bound=np.array(dl.max_bound, dtype=np.float64))


def prior_of(tables):
    """TriangulationPrior (planes left to the device) from a worker result."""
    from .prior import TriangulationPrior
    look = WalkTables(tables["neighbors"], tables["equations"], tables["paraboloid_scale"],
                      tables["paraboloid_shift"], tables["min_bound"], tables["max_bound"])
    return TriangulationPrior(points=tables["points"], disparities=tables["disparities"],
                              triangles=tables["triangles"], planes=None,
                              num_anchors=tables["num_anchors"], _lookup=look)


def _ping():
    import scipy.spatial  # noqa: F401 -- import once per worker
    return 0


_POOLS = {}


def make_pool(workers=None):
    """A persistent pool of spawn-started workers (created and warmed once
    per process: every worker has imported scipy before the first frame)."""
    import atexit
    import multiprocessing as mp
    import os
    from concurrent.futures import ProcessPoolExecutor
    n = workers or max(1, min(len(os.sched_getaffinity(0)) - 2, 32))
    pool = _POOLS.get(n)
    if pool is None:
        pool = ProcessPoolExecutor(max_workers=n, mp_context=mp.get_context("spawn"))
        for f in [pool.submit(_ping) for _ in range(4 * n)]:
            f.result()
        _POOLS[n] = pool
        atexit.register(pool.shutdown, wait=False, cancel_futures=True)
    return pool, n
