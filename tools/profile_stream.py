"""Where does reconstruct_stream spend host time? (run on the GPU box)"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402


def main():
    frame, rig, tri, _ = bench.load_inputs("C2")
    sp, pp = bench.params_for("C2")
    pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
    pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
    for d, s in zip(pin_i, frame.images):
        d[...] = s
    for d, s in zip(pin_p, frame.priors):
        d[...] = s
    hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
    # isolated pieces
    s = torch.cuda.Stream()
    for name, fn in [("TriDevice (pageable)", lambda: TriDevice(tri)),
                     ("delaunay tables", lambda: (tri._lookup.transform, tri._lookup.equations))]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            with torch.cuda.stream(s):
                fn()
        torch.cuda.synchronize()
        print(f"{name:24s} {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
    os.environ["ST_STREAM_PROFILE"] = "1"
    for n in (10, 30):
        t0 = time.perf_counter()
        for _ in st.reconstruct_stream([(hf, tri)] * n, rig, sp, pp):
            pass
        torch.cuda.synchronize()
        print(f"stream x{n}: {(time.perf_counter() - t0) / n * 1e3:.3f} ms/frame")
    del os.environ["ST_STREAM_PROFILE"]
    # frame-in stream: harvest + dedup + pooled Qhull + solve per frame
    ref = st.reconstruct(hf, rig, tri, sp, pp)
    from paper_2003_11076_b200.qhull_pool import make_pool
    t0 = time.perf_counter()
    make_pool()
    print(f"pool start + warm: {time.perf_counter() - t0:.2f} s")
    for n in (8, 64):
        t0 = time.perf_counter()
        outs = list(st.reconstruct_frames([hf] * n, rig, sp, pp))
        dt = (time.perf_counter() - t0) / n
        ok = all(np.array_equal(o.disparity.values, ref.disparity.values)
                 and np.array_equal(o.image, ref.image) for o in outs)
        print(f"reconstruct_frames x{n}: {dt * 1e3:.2f} ms/frame ({1 / dt:.1f} fps), "
              f"outputs == reconstruct(): {ok}")


if __name__ == "__main__":
    main()
