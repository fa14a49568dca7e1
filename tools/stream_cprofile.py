"""cProfile of reconstruct_stream's consumer thread (GPU box)."""
import cProfile
import os
import pstats
import sys

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
for _ in st.reconstruct_stream([(hf, tri)] * 8, rig, sp, pp):
    pass
pr = cProfile.Profile()
pr.enable()
for _ in st.reconstruct_stream([(hf, tri)] * 100, rig, sp, pp):
    pass
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
