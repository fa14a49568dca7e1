"""Resident-frame throughput vs frame slots and EM streams (experiment).

slots S frame pipelines rotate; with `streams` = S each slot's EM runs on its
own stream (frames in flight concurrently), with 1 they share the caller's
stream (EM serialised, pre-solve overlapped: bench.py's `value` loop)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2003_11076_b200.prior import TriDevice
from paper_2003_11076_b200.reconstruct import FramePipeline

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
w, h, k, dmax, iters = bench.CONFIGS[cfg]
sp, pp = bench.params_for(cfg)
frame, rig, tri, exact = bench.load_inputs(cfg)
pipes = []
for _ in range(int(os.environ.get('SLOTS_MAX', '4'))):
    p = FramePipeline(rig, w, h, sp, pp)
    p.load(frame.images, frame.priors)
    pipes.append((p, TriDevice(tri)))
main = torch.cuda.current_stream()


def run(n_slots, n_streams, steps, prio=0):
    streams = [torch.cuda.Stream(priority=prio) for _ in range(n_streams)]
    done = [None] * n_slots
    start = torch.cuda.Event(enable_timing=True)
    start.record(main)
    for s in streams:
        s.wait_event(start)
    for j in range(steps):
        slot = j % n_slots
        s = streams[j % n_streams]
        p, td = pipes[slot]
        with torch.cuda.stream(s):
            if done[slot] is not None:
                s.wait_event(done[slot])
            ready = torch.cuda.Event()
            ready.record(s)
            p.run(td, ready=ready)
            ev = torch.cuda.Event()
            ev.record(s)
            done[slot] = ev
    for s in streams:
        main.wait_stream(s)
    end = torch.cuda.Event(enable_timing=True)
    end.record(main)
    torch.cuda.synchronize()
    return steps / (start.elapsed_time(end) / 1e3)


out = {}
CASES = [tuple(int(v) for v in c.split(',')) for c in os.environ['SLOT_CASES'].split(';')] if os.environ.get('SLOT_CASES') else ((2, 1, 0), (2, 2, 0), (3, 3, 0), (4, 4, 0), (4, 2, 0), (2, 2, -1), (3, 3, -1))
for slots, streams, prio in CASES:
    run(slots, streams, 8, prio)
    fps = [run(slots, streams, steps, prio) for _ in range(5)]
    out[f"slots{slots}_streams{streams}_prio{prio}"] = [round(float(np.median(fps)), 1), round(min(fps), 1), round(max(fps), 1)]
    print(cfg, slots, streams, prio, out[f"slots{slots}_streams{streams}_prio{prio}"], flush=True)
print(json.dumps({"config": cfg, "fps_median_min_max": out}))
