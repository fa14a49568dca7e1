"""Does host-link DMA traffic slow the resident pipelined stream (L2 / HBM
interference), and does an L2 persistence window on the descriptor maps help?"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2003_11076_b200 import _native as N  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice  # noqa: E402
from paper_2003_11076_b200.reconstruct import FramePipeline  # noqa: E402

frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
w, h = 1280, 720
slots = []
for _ in range(2):
    p = FramePipeline(rig, w, h, sp, pp)
    p.load(frame.images, frame.priors)
    slots.append((p, TriDevice(tri)))
stream = torch.cuda.current_stream()
done = [None, None]


def pipelined(n):
    for j in range(n):
        p, td = slots[j % 2]
        ready = done[j % 2]
        if ready is None:
            ready = torch.cuda.Event()
            ready.record(stream)
        p.run(td, ready=ready)
        ev = torch.cuda.Event()
        ev.record(stream)
        done[j % 2] = ev


def timed(n=60):
    pipelined(8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipelined(n)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


h_in = torch.empty(37_111_088, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty(16_588_800, dtype=torch.uint8, device="cuda")
h_out = torch.empty_like(d_out, device="cpu").pin_memory()
cs1, cs2 = torch.cuda.Stream(), torch.cuda.Stream()
stop = threading.Event()


def copier():
    while not stop.is_set():
        with torch.cuda.stream(cs1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(cs2):
            h_out.copy_(d_out, non_blocking=True)
        cs1.synchronize()
        cs2.synchronize()


def native_copier():
    # 64 H2D copies of 37 MB per ctypes call: the GIL is held only between calls
    import numpy as np
    src = h_in.numpy()
    arrs = [src] * 64
    srcs, offs, sizes, n = N.gather_args(arrs, [0] * 64)
    while not stop.is_set():
        N.check(N.lib().st_h2d_gather(N.C.c_void_p(d_in.data_ptr()), srcs, offs, sizes, n,
                                      N.C.c_void_p(cs1.cuda_stream)))
        cs1.synchronize()


out = {"alone_ms": timed()}
th = threading.Thread(target=native_copier)
th.start()
out["with_native_h2d_copies_ms"] = timed()
stop.set()
th.join()
stop.clear()
th = threading.Thread(target=copier)
th.start()
out["with_copies_ms"] = timed()
for mb in (48, 80):
    N.check(N.lib().st_l2_set_aside(mb << 20))
    for p, _ in slots:
        for s in (stream, p.side, p.side2):
            N.check(N.lib().st_stream_l2_window(N.C.c_void_p(s.cuda_stream),
                                                N.C.c_void_p(p.desc.data_ptr()),
                                                p.desc.numel(), 0.6))
    out[f"with_copies_l2persist_{mb}MB_ms"] = timed()
stop.set()
th.join()
out["alone_l2persist_ms"] = timed()
print(out)
