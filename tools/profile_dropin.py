"""cProfile of the drop-in path (em_solve + synthesize on pageable numpy, C2)."""
import cProfile
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402
import torch  # noqa: E402

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
imgs = [np.array(x) for x in frame.images]
pris = [np.array(x) for x in frame.priors]


def one():
    f = st.LightFieldFrame(images=imgs, priors=pris)
    dmap, seg, _ = st.em_solve(f, rig, tri, sp, pp)
    st.synthesize(f, rig, dmap, seg)


for _ in range(3):
    one()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    one()
torch.cuda.synchronize()
print("dropin ms/frame", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    one()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
