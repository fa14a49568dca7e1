"""e2e stream throughput probe (run on the GPU box): reconstruct_stream over
pinned host frames, like bench.py's e2e leg, median of 3 streams of 60."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pin_i + pin_p, list(frame.images) + list(frame.priors)):
    d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
for _ in st.reconstruct_stream([(hf, tri)] * 4, rig, sp, pp):
    pass
reps = []
for _ in range(3):
    t0 = time.perf_counter()
    for _ in st.reconstruct_stream([(hf, tri)] * 60, rig, sp, pp):
        pass
    torch.cuda.synchronize()
    reps.append((time.perf_counter() - t0) * 1e3 / 60)
print("e2e ms/frame", sorted(reps), "fps", 1e3 / sorted(reps)[1], os.environ.get("TAG", ""))
