"""Host link bandwidth on the GPU box: the per-frame C2 transfer sizes
(37.1 MB H2D, 16.6 MB D2H) from/to pinned memory, alone and concurrently
on two streams (the e2e stream's situation)."""
import json
import time

import torch

H2D, D2H, REPS = 37_111_088, 16_588_800, 50
h_in = torch.empty(H2D, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(H2D, dtype=torch.uint8, device="cuda")
d_out = torch.empty(D2H, dtype=torch.uint8, device="cuda")
h_out = torch.empty(D2H, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(REPS):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / REPS


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t_h, t_d, t_b = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_gbs": H2D / t_h / 1e9, "d2h_gbs": D2H / t_d / 1e9,
                  "concurrent_ms_per_frame": t_b * 1e3,
                  "concurrent_fps_bound": 1.0 / t_b,
                  "concurrent_h2d_gbs": H2D / t_b / 1e9}))
