"""e2e stream variants (GPU box): pinned host frames vs device-resident
frames through reconstruct_stream, and stream slot counts."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402
import importlib  # noqa: E402
R = importlib.import_module("paper_2003_11076_b200.reconstruct")

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pin_i + pin_p, list(frame.images) + list(frame.priors)):
    d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
dimg = torch.from_numpy(np.stack(frame.images)).cuda()
dpri = torch.from_numpy(np.stack(frame.priors)).cuda()


class DevFrame:
    images, priors = dimg, dpri
    num_views = len(frame.images)
    shape = frame.shape


def run(src, n=60):
    for _ in st.reconstruct_stream([(src, tri)] * 8, rig, sp, pp):
        pass
    reps = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in st.reconstruct_stream([(src, tri)] * n, rig, sp, pp):
            pass
        torch.cuda.synchronize()
        reps.append((time.perf_counter() - t0) * 1e3 / n)
    return sorted(reps)[1]


print("pinned host frames ms/frame", run(hf))
print("device frames ms/frame", run(DevFrame()))
R.STREAM_SLOTS = 4
R._STREAM_PIPES.clear()
print("pinned, 4 slots ms/frame", run(hf))
