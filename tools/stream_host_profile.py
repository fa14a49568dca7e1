"""Host-side phases of reconstruct_stream (ST_STREAM_PROFILE) over a long
stream of pinned C2 frames, with the GPU-side frame time for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2003_11076_b200 as st

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pin_i + pin_p, list(frame.images) + list(frame.priors)):
    d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
for _ in st.reconstruct_stream([(hf, tri)] * 10, rig, sp, pp):
    pass
n = 200
os.environ["ST_STREAM_PROFILE"] = "1"
t0 = time.perf_counter()
for _ in st.reconstruct_stream([(hf, tri)] * n, rig, sp, pp):
    pass
torch.cuda.synchronize()
print(f"{n} frames: {(time.perf_counter() - t0) / n * 1e3:.3f} ms/frame", flush=True)
