"""reconstruct_stream throughput vs compute-stream mode (experiment):
ST_STREAM_COMPUTE=main (every slot's EM on the caller's stream), k (k slot
streams), slot (one per slot); full and dynamic_only, pinned C2 frames."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2003_11076_b200 as st

frame, rig, tri, exact = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(im.shape, np.uint8) for im in frame.images]
pin_p = [st.device.pinned_empty(p.shape, np.float32) for p in frame.priors]
for d, s in zip(pin_i, frame.images):
    d[...] = s
for d, s in zip(pin_p, frame.priors):
    d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)


def stream(n, dyn):
    for _ in st.reconstruct_stream([(hf, tri)] * 8, rig, sp, pp, dynamic_only=dyn):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in st.reconstruct_stream([(hf, tri)] * n, rig, sp, pp, dynamic_only=dyn):
        pass
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t0)


CASES = os.environ.get("MODE_CASES", "main:1,main:2,main:4,slot:4,2:4,slot:2,main:1").split(",")
for case in CASES:
    mode, depth = case.split(":")
    os.environ["ST_STREAM_COMPUTE"] = mode
    os.environ["ST_STREAM_DEPTH"] = depth
    for dyn in (False, True):
        r = [stream(60, dyn) for _ in range(3)]
        print(f"mode {mode:5s} depth {depth} dyn {int(dyn)}: fps {np.median(r):.1f} "
              f"({min(r):.1f}-{max(r):.1f})", flush=True)
