"""Row-band sharding host logic across 2 processes (gloo, CPU): band split,
the st_solve reduce callback, and band gathering."""

import os
import socket

import numpy as np
import pytest

from paper_2003_11076_b200.sharding import band_mask, band_rows


def test_band_rows_partition():
    for h in (1, 7, 120, 720, 1081):
        for world in (1, 2, 3, 4, 8):
            got = [band_rows(h, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    m = sum(band_mask(10, 4, 3, r).astype(int) for r in range(3))
    assert (m == 1).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import ctypes
    import torch.distributed as dist
    from paper_2003_11076_b200.sharding import CollectiveReduce, gather_bands
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the callback sums per-iteration statistics in place, like st_solve calls it
        red = CollectiveReduce()
        vals = (ctypes.c_double * 7)(*[rank + 1.0 + i for i in range(7)])
        rc = red(vals, 7, None)
        summed = [vals[i] for i in range(7)]
        # every rank fills only its band rows; the gather rebuilds the frame
        h, w = 13, 5
        full = (np.arange(h * w * 3, dtype=np.float32).reshape(h, w, 3) * 0.5)
        local = np.full_like(full, -1.0)
        r0, r1 = band_rows(h, world, rank)
        local[r0:r1] = full[r0:r1]
        got = gather_bands(local, h, world, rank)
        bits = np.arange(h * w, dtype=np.uint32).reshape(h, w) * 7919
        lb = np.zeros_like(bits)
        lb[r0:r1] = bits[r0:r1]
        gb = gather_bands(lb, h, world, rank)
        q.put((rank, rc, summed, bool(np.array_equal(got, full)), bool(np.array_equal(gb, bits))))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(1.0 + i) + (2.0 + i) for i in range(7)]
    for rank, rc, summed, ok_f, ok_b in res:
        assert rc == 0
        assert summed == want
        assert ok_f and ok_b


@pytest.mark.gpu
def test_banded_solve_matches_full_solve():
    """Two bands solved concurrently (two host threads, two streams, one
    GPU; they only meet in the host-side statistics reduction) reproduce
    the single-device solve bit for bit."""
    import threading

    import torch

    import paper_2003_11076_b200 as st
    from golden_io import load
    from test_gpu_parity import _Rig, _Tri, _frame, _params

    g = load("occ160_noisy")
    sp, pp = _params(st, g)
    frame = _frame(st, g)
    full_d, full_s, full_stats = st.DisparitySolver(frame, _Rig(g), _Tri(g), sp, pp).solve()
    h, w = frame.shape
    world = 2
    barrier = threading.Barrier(world)
    slots = [None] * world

    def make_reduce(rank):
        def red(values, n, user):
            slots[rank] = [values[i] for i in range(n)]
            barrier.wait()
            tot = [sum(slots[r][i] for r in range(world)) for i in range(n)]
            barrier.wait()
            for i in range(n):
                values[i] = tot[i]
            return 0
        return red

    out = [None] * world

    def run(rank):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            s = st.DisparitySolver(frame, _Rig(g), _Tri(g), sp, pp)
            (v, status, sb, vb), stats = s.solve_device(active_mask=band_mask(h, w, world, rank),
                                                        reduce=make_reduce(rank))
            stream.synchronize()
            out[rank] = ([x.cpu().numpy() for x in (v, status, sb, vb)], stats)

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    values = np.empty((h, w), np.float32)
    status = np.empty((h, w), np.uint8)
    sbits = np.empty((h, w), np.int32)
    for r in range(world):
        r0, r1 = band_rows(h, world, r)
        values[r0:r1] = out[r][0][0][r0:r1]
        status[r0:r1] = out[r][0][1][r0:r1]
        sbits[r0:r1] = out[r][0][2][r0:r1]
    assert np.array_equal(values, full_d.values)
    assert np.array_equal(status, full_d.status)
    assert np.array_equal(sbits.view(np.uint32), full_s.static_bits)
    for r in range(world):
        stats = out[r][1]
        assert stats.iterations_run == full_stats.iterations_run
        assert stats.converged_after == full_stats.converged_after
        assert np.allclose(stats.mean_energy, full_stats.mean_energy, rtol=1e-12)
