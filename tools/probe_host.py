"""Host-side cost of the per-frame calls (GPU box): enqueue time of
FramePipeline.run (async path), TriDevice construction and fetch_async."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402
from paper_2003_11076_b200.reconstruct import FramePipeline  # noqa: E402


def main():
    frame, rig, tri, _ = bench.load_inputs("C2")
    sp, pp = bench.params_for("C2")
    h, w = frame.shape
    pipe = FramePipeline(rig, w, h, sp, pp)
    pipe.load(frame.images, frame.priors)
    td = TriDevice(tri)
    for _ in range(3):
        pipe.run(td)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    res = {}
    for name, fn in (("TriDevice", lambda: TriDevice(tri)),
                     ("run (enqueue)", lambda: pipe.run(td)),
                     ("fetch_async (enqueue)", lambda: pipe.fetch_async(s)),
                     ("load (enqueue, pageable)", lambda: pipe.load(frame.images, frame.priors))):
        ts = []
        for _ in range(20):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        res[name] = 1e3 * float(np.median(ts))
    print({k: round(v, 3) for k, v in res.items()})


if __name__ == "__main__":
    main()
