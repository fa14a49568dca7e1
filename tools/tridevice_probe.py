"""Host cost of TriDevice (the per-frame Qhull table upload), single thread."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402

frame, rig, tri, _ = bench.load_inputs("C2")


class Slot:
    pass


slot = Slot()
for _ in range(5):
    TriDevice(tri, slot)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    TriDevice(tri, slot)
torch.cuda.synchronize()
print("TriDevice(slot) ms", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    TriDevice(tri, slot)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
