"""Section timings of TriDevice construction (GPU box diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2003_11076_b200 import prior as P
frame, rig, tri, _ = bench.load_inputs("C2")
P.TriDevice(tri); torch.cuda.synchronize()
T = {}
def t(name, f):
    t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
for _ in range(5):
    dl = t("delaunay_of", lambda: P.delaunay_of(tri))
    sp = t("support_points", lambda: tri.support_points())
    arrs = t("asarray", lambda: [np.asarray(dl.transform, dtype=np.float64), np.asarray(dl.equations, dtype=np.float64), np.asarray(dl.neighbors, dtype=np.int32)])
    t("full TriDevice", lambda: P.TriDevice(tri))
for k, v in T.items(): print(f"{k:16s} {v/5*1e3:.3f} ms")
print(type(dl.neighbors), dl.neighbors.dtype, dl.neighbors.flags['C_CONTIGUOUS'], type(dl.transform))
