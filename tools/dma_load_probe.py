"""Host->device DMA throughput alone and while the resident four-slot stream
runs (run on the GPU box): is reconstruct_stream's e2e DMA-bound?"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402
from paper_2003_11076_b200.reconstruct import FramePipeline  # noqa: E402

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
h, w = frame.shape
NB = 36 << 20
src = [torch.empty(NB // 2, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
dst = [torch.empty(NB // 2, dtype=torch.uint8, device="cuda") for _ in range(2)]
cs = [torch.cuda.Stream() for _ in range(2)]


def dma(n, streams):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(cs[0])
    for s in cs[1:streams]:
        s.wait_event(e0)
    for i in range(n):
        for j in range(2):
            s = cs[j % streams]
            with torch.cuda.stream(s):
                dst[j].copy_(src[j], non_blocking=True)
    for s in cs[1:streams]:
        cs[0].wait_stream(s)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(cs[0])
    e1.synchronize()
    return n * NB / (e0.elapsed_time(e1) / 1e3) / 1e9


slots = []
for _ in range(4):
    p = FramePipeline(rig, w, h, sp, pp)
    p.load(frame.images, frame.priors)
    slots.append((p, TriDevice(tri)))


def resident(n):
    done = [None] * 4
    for j in range(n):
        p, td = slots[j % 4]
        c = p.compute
        if done[j % 4] is not None:
            c.wait_event(done[j % 4])
        ready = torch.cuda.Event()
        ready.record(c)
        with torch.cuda.stream(c):
            p.run(td, ready=ready)
        ev = torch.cuda.Event()
        ev.record(c)
        done[j % 4] = ev
    torch.cuda.synchronize()


dma(5, 1)
resident(8)
for streams in (1, 2):
    print(f"H2D alone, {streams} copy stream(s): {dma(40, streams):.1f} GB/s", flush=True)
for streams in (1, 2):
    stop = [False]
    out = []

    def bg():
        while not stop[0]:
            resident(8)
    th = threading.Thread(target=bg)
    th.start()
    time.sleep(0.3)
    rates = [dma(20, streams) for _ in range(5)]
    stop[0] = True
    th.join()
    print(f"H2D under the resident stream, {streams} copy stream(s): "
          f"{np.median(rates):.1f} GB/s ({min(rates):.1f}-{max(rates):.1f})", flush=True)
