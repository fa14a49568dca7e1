"""Experiment: is reconstruct_stream's e2e bound by its preparation thread?
Times the stream normally, then with TriDevice replaced by a per-slot cache
(the tables not re-packed / re-uploaded: NOT a valid e2e, a bound probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2003_11076_b200 as st
R = sys.modules["paper_2003_11076_b200.reconstruct"]

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pin_i + pin_p, list(frame.images) + list(frame.priors)):
    d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)


def run(n=120):
    for _ in st.reconstruct_stream([(hf, tri)] * 10, rig, sp, pp):
        pass
    torch.cuda.synchronize()
    r = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in st.reconstruct_stream([(hf, tri)] * n, rig, sp, pp):
            pass
        torch.cuda.synchronize()
        r.append(n / (time.perf_counter() - t0))
    return np.median(r)


print("normal fps", run(), flush=True)
orig = R.TriDevice
cache = {}


def cached(tri_, slot=None):
    k = id(slot)
    if k not in cache:
        cache[k] = orig(tri_, slot=slot)
    return cache[k]


R.TriDevice = cached
print("tables cached per slot (probe only) fps", run(), flush=True)
