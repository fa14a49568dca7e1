"""Row-band sharding (sharding.py): band split and halos, the per-iteration
record exchange and the band gather across 2-3 processes (gloo, CPU), and on
the GPU the banded reconstruction against the single-device one."""

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


def test_band_extents_cover_the_frame_with_halos():
    from paper_2003_11076_b200.sharding import DESC_HALO, band_extents
    for h in (5, 120, 1080):
        for world in (1, 2, 3, 8):
            for mr in (0, 1, 2):
                own = []
                for r in range(world):
                    e = band_extents(h, world, r, mr, rectified=True)
                    r0, r1 = e["rows"]
                    own.append((r0, r1))
                    e0, e1 = e["solve"]
                    assert e0 == max(0, r0 - mr) and e1 == min(h, r1 + mr)
                    d0, d1 = e["desc"]
                    assert d0 <= e0 and d1 >= e1
                    i0, i1 = e["images"]
                    assert i0 == max(0, d0 - DESC_HALO) and i1 == min(h, d1 + DESC_HALO)
                    assert e["priors"] == e["desc"]
                    g = band_extents(h, world, r, mr, rectified=False)
                    assert g["images"] == (0, h) and g["priors"] == (0, h)
                assert own[0][0] == 0 and own[-1][1] == h
                assert all(a[1] == b[0] for a, b in zip(own, own[1:]))


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2003_11076_b200.sharding import RecordExchange, gather_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the per-iteration record exchange st_solve_rows calls (rank order)
        rec = 96
        send = torch.arange(rec, dtype=torch.uint8) + rank
        recv = torch.zeros(world * rec, dtype=torch.uint8)
        ex = RecordExchange(send, recv, None)
        rc = ex._call(None, None)
        gathered = recv.numpy().reshape(world, rec)
        ok_x = rc == 0 and all(np.array_equal(gathered[r], np.arange(rec) + r)
                               for r in range(world))
        # every rank fills only its band rows; rank 0 gathers the frame
        h, w = 13, 5
        full = np.arange(h * w * 3, dtype=np.float32).reshape(h, w, 3) * 0.5
        bits = (np.arange(h * w, dtype=np.int64).reshape(h, w) * 7919).astype(np.int32)
        a = torch.full((h, w, 3), -1.0)
        b = torch.zeros((h, w), dtype=torch.int32)
        r0, r1 = band_rows(h, world, rank)
        a[r0:r1] = torch.from_numpy(full[r0:r1])
        b[r0:r1] = torch.from_numpy(bits[r0:r1])
        gather_rows([a, b], h, world, rank, dst=0)
        ok_g = rank != 0 or (np.array_equal(a.numpy(), full) and np.array_equal(b.numpy(), bits))
        q.put((rank, bool(ok_x), bool(ok_g)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_exchange_and_gather(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_x, ok_g in res:
        assert ok_x and ok_g, rank


def _band_gpu_worker(rank, world, port, q, dynamic_only, force_retry=False):
    import torch
    import torch.distributed as dist
    if force_retry:
        os.environ["ST_MU_FORCE_UNSAFE"] = "1"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2003_11076_b200 as st
        from paper_2003_11076_b200.sharding import reconstruct_band, solve_band
        from golden_io import load
        from test_gpu_parity import _Rig, _Tri, _frame, _params
        g = load("occ320_noisy")
        sp, pp = _params(st, g)
        frame, rig, tri = _frame(st, g), _Rig(g), _Tri(g)
        r = reconstruct_band(frame, rig, tri, sp, pp, dynamic_only=dynamic_only)
        from paper_2003_11076_b200.sharding import _BANDS
        retries = sum(b.retries for b in _BANDS.values())
        assert (retries > 0) == force_retry, retries
        out = None
        if r is not None:
            out = dict(values=r.disparity.values, status=r.disparity.status,
                       static=r.segmentation.static_bits, valid=r.segmentation.valid_bits,
                       image=r.image, prov=r.provenance, n_rays=r.n_rays,
                       stats=(r.stats.iterations_run, r.stats.converged_after,
                              list(r.stats.mean_energy), list(r.stats.prev_energy),
                              list(r.stats.changed_fraction), r.stats.active_pixels))
        solver = st.DisparitySolver(frame, rig, tri, sp, pp)
        d, s, stats = solve_band(solver, dynamic_only=dynamic_only)
        q.put((rank, out, (d.values, s.static_bits, stats.iterations_run)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,dynamic_only,force_retry",
                         [(2, False, False), (3, False, False), (2, True, False),
                          (3, False, True)])
def test_row_bands_match_single_device(world, dynamic_only, force_retry):
    """`reconstruct_band` over 2-3 processes (gloo collectives, one GPU; no
    kernel waits on another process) reproduces the single-device
    `reconstruct` bit for bit: disparity, status, bits, refocused image
    (median halo rows included), provenance, n_rays; EMStats iterations,
    changed fractions exact, energies to 1e-12 (a different summation
    order).  solve_band likewise.  force_retry: every shard's row-window
    surface raster is flagged inexact, so every shard redoes the frame with
    the whole-frame raster (ST_EAGAIN) -- same results."""
    import torch.multiprocessing as mp

    import paper_2003_11076_b200 as st
    from golden_io import load
    from test_gpu_parity import _Rig, _Tri, _frame, _params
    g = load("occ320_noisy")
    sp, pp = _params(st, g)
    ref = st.reconstruct(_frame(st, g), _Rig(g), _Tri(g), sp, pp, dynamic_only=dynamic_only)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_gpu_worker,
                         args=(r, world, port, q, dynamic_only, force_retry))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = res[0][1]
    assert all(x[1] is None for x in res[1:])
    for key, want in (("values", ref.disparity.values), ("status", ref.disparity.status),
                      ("static", ref.segmentation.static_bits),
                      ("valid", ref.segmentation.valid_bits), ("image", ref.image),
                      ("prov", ref.provenance), ("n_rays", ref.n_rays)):
        assert np.array_equal(out[key], want), key
    it, conv, me, pe, cf, act = out["stats"]
    assert (it, conv) == (ref.stats.iterations_run, ref.stats.converged_after)
    assert cf == list(ref.stats.changed_fraction)
    assert act == ref.stats.active_pixels
    np.testing.assert_allclose(me, ref.stats.mean_energy, rtol=1e-12)
    np.testing.assert_allclose(pe, ref.stats.prev_energy, rtol=1e-12)
    for rank, _, (vals, sbits, iters) in res:
        assert np.array_equal(vals, ref.disparity.values), rank
        assert np.array_equal(sbits, ref.segmentation.static_bits), rank
        assert iters == ref.stats.iterations_run


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


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_row_window_mu_raster_equals_whole_frame(cfg):
    """st_mu_raster_rows (a band's rows + 2 halo rows of Qhull-walk replay)
    gives the whole-frame raster's mu bit for bit on the band's rows, for
    the bands of 2, 3, 5 and 8 shards (a window it cannot make exact must
    say so)."""
    import torch

    import bench
    from paper_2003_11076_b200 import _native as N
    from paper_2003_11076_b200.prior import TriDevice
    from paper_2003_11076_b200.sharding import band_extents
    frame, rig, tri, _ = bench.load_inputs(cfg)
    sp, pp = bench.params_for(cfg)
    h, w = frame.shape
    td = TriDevice(tri)
    ws = torch.empty(int(N.lib().st_mu_raster_workspace(w, h, td.n_tri)), dtype=torch.uint8,
                     device="cuda")
    full = torch.empty(h * w, dtype=torch.float64, device="cuda")
    N.invoke("st_mu_raster", td.st, w, h, float(pp.d_max), full, ws, ws.numel())
    want = full.cpu().numpy().reshape(h, w)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    unsafe = checked = 0
    for world in ((2, 8) if cfg == "C4" else (2, 3, 5, 8)):
        for rank in range(world):
            e0, e1 = band_extents(h, world, rank, 1, True)["solve"]
            mu = torch.full((h * w,), float("nan"), dtype=torch.float64, device="cuda")
            N.invoke("st_mu_raster_rows", td.st, w, h, float(pp.d_max), mu, ws, ws.numel(), e0,
                     e1, flag)
            if int(flag.item()):
                unsafe += 1
                continue
            got = mu.cpu().numpy().reshape(h, w)[e0:e1]
            assert np.array_equal(got.view(np.uint64), want[e0:e1].view(np.uint64)), \
                (world, rank, int((got != want[e0:e1]).sum()))
            checked += 1
    print(f"{cfg}: {checked} band windows exact, {unsafe} flagged for the whole-frame raster")
    assert checked > 0
