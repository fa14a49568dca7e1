"""Where TriDevice(tri, slot) spends host time per frame (GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2003_11076_b200 import _native as N
from paper_2003_11076_b200.prior import TriDevice, delaunay_of, _integral_coords
from paper_2003_11076_b200.reconstruct import FramePipeline

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
h, w = frame.shape
pipe = FramePipeline(rig, w, h, sp, pp)
for _ in range(5):
    TriDevice(tri, slot=pipe)
torch.cuda.synchronize()


def timeit(name, fn, n=50):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:32s} {(time.perf_counter() - t0) / n * 1e3:.3f} ms", flush=True)


timeit("TriDevice(tri, slot)", lambda: TriDevice(tri, slot=pipe))
dl = delaunay_of(tri)
timeit("delaunay_of", lambda: delaunay_of(tri))
pts = np.asarray(tri.points, dtype=np.float64).reshape(-1, 2)
timeit("_integral_coords", lambda: _integral_coords(pts))
parts = [pts, np.asarray(tri.disparities, dtype=np.float64), np.asarray(tri.triangles, dtype=np.int32),
         np.asarray(dl.neighbors, dtype=np.int32), np.asarray(dl.equations, dtype=np.float64)]
timeit("asarray parts", lambda: [np.asarray(tri.triangles, dtype=np.int32), np.asarray(dl.neighbors, dtype=np.int32), np.asarray(dl.equations, dtype=np.float64)])
offs, tot = [], 0
for a in parts:
    offs.append(tot)
    tot += (a.nbytes + 255) & ~255
print("total bytes", tot)
stage = torch.empty(tot, dtype=torch.uint8, pin_memory=True)
arrs = [np.ascontiguousarray(a) for a in parts]
srcs, goffs, sizes, n = N.gather_args(arrs, offs)
timeit("st_host_gather", lambda: N.lib().st_host_gather(N.C.c_void_p(stage.data_ptr()), srcs, goffs, sizes, n))
timeit("support_points", lambda: tri.support_points())
