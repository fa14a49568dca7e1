"""Host-side breakdown of one reconstruct() call (run on the GPU box)."""

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
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402


def main(cfg="C2", n=10):
    frame, rig, tri, _ = bench.load_inputs(cfg)
    sp, pp = bench.params_for(cfg)
    pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
    pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
    for d, s in zip(pin_i, frame.images):
        d[...] = s
    for d, s in zip(pin_p, frame.priors):
        d[...] = s
    hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
    for _ in range(3):
        st.reconstruct(hf, rig, tri, sp, pp)
    torch.cuda.synchronize()
    acc = {}

    def tick(name, t0):
        torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    for _ in range(n):
        t0 = time.perf_counter()
        pipe = R._pipeline_for(rig, frame.shape[1], frame.shape[0], sp, pp)
        t0 = tick("pipeline_lookup", t0)
        pipe.load(hf.images, hf.priors)
        t0 = tick("h2d_frame", t0)
        td = TriDevice(tri)
        t0 = tick("tri_device", t0)
        stats = pipe.run(td)
        t0 = tick("run", t0)
        out = pipe.fetch()
        t0 = tick("d2h", t0)
    for k, v in acc.items():
        print(f"{k:16s} {v / n * 1e3:8.3f} ms")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C2"]))


def fetch_detail(cfg="C2"):
    frame, rig, tri, _ = bench.load_inputs(cfg)
    sp, pp = bench.params_for(cfg)
    pipe = R.FramePipeline(rig, frame.shape[1], frame.shape[0], sp, pp)
    pipe.load(frame.images, frame.priors)
    td = TriDevice(tri)
    for _ in range(3):
        pipe.run(td)
        out = pipe.fetch()
    torch.cuda.synchronize()
    for it in range(3):
        pipe.run(td)
        torch.cuda.synchronize()
        t = time.perf_counter()
        hosts = []
        for d in (pipe.values, pipe.status, pipe.sbits, pipe.vbits, pipe.image, pipe.prov, pipe.n_rays):
            t1 = time.perf_counter()
            h = torch.empty(d.shape, dtype=d.dtype, pin_memory=True)
            t2 = time.perf_counter()
            h.copy_(d, non_blocking=True)
            t3 = time.perf_counter()
            hosts.append(h)
            print(f"  alloc {1e3*(t2-t1):.3f} copy-issue {1e3*(t3-t2):.3f}")
        torch.cuda.current_stream().synchronize()
        print("total fetch", 1e3 * (time.perf_counter() - t), "ms")
        out = hosts


if __name__ == "__main__" and os.environ.get("FETCH_DETAIL"):
    fetch_detail()
