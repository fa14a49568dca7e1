#!/usr/bin/env python
"""Benchmark: refocused static frames/s of the EM background reconstruction.

One step = one synthetic light-field frame through the whole hot path
(descriptors, surface raster, support candidate lists, initial masks, EM with
the reference's convergence rule (max 5 iterations at C2), Eq. 2 refocus,
median) -- `FramePipeline.run` on frames already resident in HBM (`value`),
and the public `reconstruct()` call from pinned host memory with the
artefacts copied back (`e2e`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

N > 1 is launched by torchrun: one rank per GPU, each rank reconstructs its
own frames (frame-parallel, BASELINE C5; no data-path collective), time =
max over ranks.  `--impl reference` times the CPU oracle (the numpy
restatement of the reference) on a bounded pixel sample of the same frame.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "refocused static frames/sec (and Gpix·plane/s) at 1/2/4/8 B200 vs CPU ref"
CONFIGS = {  # name: (width, height, cameras, d_max, max_iters)
    "C1": (640, 480, 5, 32.0, 5),
    "C2": (1280, 720, 5, 64.0, 5),
    "C3": (1920, 1080, 5, 128.0, 10),
    "C4": (3840, 2160, 9, 128.0, 10),
}
SCENE = dict(coverage=0.25, seed=11, p_flip=0.1, blur_radius=2)
L2_FLUSH_BYTES = 256 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# -- inputs -----------------------------------------------------------------------

def load_inputs(cfg, host=None):
    """Render the config's frame (bit-identical to the reference renderer:
    checked against the digests the reference recorded) and triangulate the
    support the reference harvested for it.  The device renderer
    (paper_2003_11076_b200.renderer) when CUDA is up; `host` (the reference
    arm, CPU-only tests) takes the numpy restatement in oracle/synth.py."""
    import hashlib
    import torch
    from paper_2003_11076_b200 import synth
    from paper_2003_11076_b200.prior import SupportPoint, triangulate
    if host is None:
        host = not torch.cuda.is_available()
    w, h, k, dmax, iters = CONFIGS[cfg]
    spec = synth.occluder_scene(width=w, height=h, cameras=k, **SCENE)
    if host:
        from oracle.synth import render
    else:
        render = synth.render
    frame, _ = render(spec)
    rig = spec.rig()
    path = os.path.join(ROOT, "tests", "golden", f"bench_{cfg}.npz")
    z = np.load(path)

    def digest(arrs):
        hh = hashlib.sha256()
        for a in arrs:
            hh.update(np.ascontiguousarray(a).tobytes())
        return hh.hexdigest()

    exact = (digest(frame.images) == str(z["image_digest"])
             and digest(frame.priors) == str(z["prior_digest"]))
    pts = [SupportPoint(int(u), int(v), float(d), int(s))
           for (u, v), d, s in zip(z["support_uv"], z["support_d"], z["support_src"])]
    tri = triangulate(pts, w, h)
    return frame, rig, tri, exact


def params_for(cfg):
    import paper_2003_11076_b200 as st
    w, h, k, dmax, iters = CONFIGS[cfg]
    return st.SolverParams(max_iters=iters), st.PriorParams(d_max=dmax)


# -- clocks ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML
    polled every 2 ms from a thread (plus one synchronous sample when the
    region opens and one when it closes); nvidia-smi -lms as the fallback."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.samples = []          # (sm_mhz, max_mhz, reason bits)
        self.nvml = None
        self.stop = threading.Event()
        self.proc = None
        self.lines = []

    def _handle(self, nv):
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return nv.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        self.samples.append((float(sm), float(mx), int(get(h))))

    def _poll(self):
        while not self.stop.wait(0.002):
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                return

    def __enter__(self):
        # preferred: the library's native NVML thread (never takes the GIL
        # from the thread that enqueues the frames)
        try:
            from paper_2003_11076_b200 import _native as N
            if N.lib().st_clocks_start(2000) == 0:
                self.native = N
                return self
        except Exception:  # noqa: BLE001
            pass
        self.native = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, self._handle(nv))
            self._sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                bits = sum(b for (_, b), v in zip(self.REASONS, parts[2:6])
                           if v.lower() == "active")
                self.samples.append((float(parts[0]), float(parts[1]), bits))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *exc):
        if getattr(self, "native", None) is not None:
            cap = 65536
            sm = np.zeros(cap, np.uint32)
            mx = np.zeros(cap, np.uint32)
            rs = np.zeros(cap, np.uint64)
            n = int(self.native.lib().st_clocks_stop(sm.ctypes.data, mx.ctypes.data,
                                                     rs.ctypes.data, cap))
            for i in range(max(0, min(n, cap))):
                self.samples.append((float(sm[i]), float(mx[i]), int(rs[i])))
            return False
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [x[0] for x in self.samples]
        bits = 0
        for x in self.samples:
            bits |= x[2]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.samples[-1][1],
                "reasons": sorted(n for n, b in self.REASONS if bits & b),
                "samples": len(sm),
                "source": ("nvml (native sampler thread)" if getattr(self, "native", None)
                           else "nvml" if self.nvml else "nvidia-smi")}


# -- CPU oracle sample ------------------------------------------------------------------

def next_rows(frame, rig, cfg, pipe, host_frame, peak, cpu_leg=True):
    """SURVEY 8(f) rows widened this round, measured like the hot path:
    (f)1 the device support harvest (st_harvest + native dedup) with its
    roofline and a CPU-port baseline, (f)2 host Qhull + device planes /
    transforms, the frame-in stream (reconstruct_frames) and (f)3 frame
    directories -> artefact directories (run_reconstruct_sequence)."""
    import torch
    import paper_2003_11076_b200 as st
    from paper_2003_11076_b200 import _native as N
    from paper_2003_11076_b200.prior import TriDevice, deduplicate_arrays, triangulate_arrays, _grid_len
    w, h, k, dmax, iters = CONFIGS[cfg]
    sp, pp = params_for(cfg)
    pipe.load(frame.images, frame.priors)
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    for _ in range(3):
        pipe.harvest()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        pipe.harvest(counters=ctr)
    e1.record()
    e1.synchronize()
    hv_ms = e0.elapsed_time(e1) / reps
    n_cand, n_rev = (int(x) for x in ctr.cpu())
    nd = _grid_len(dmax)
    samples = (n_cand + n_rev) * nd          # descriptor samples, 16 B each (SURVEY 8d unit)
    t0 = time.perf_counter()
    u, v, d, src = pipe.harvest_host()
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    tri = triangulate_arrays(u, v, d, w, h, planes=False)
    t_qhull = time.perf_counter() - t0
    td = TriDevice(tri)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        N.invoke("st_tri_tables", td.st, td.planes, td.transform, td.flags)
    e1.record()
    e1.synchronize()
    tt_ms = e0.elapsed_time(e1) / reps
    # frame-in stream: raw frames -> harvest -> dedup -> pooled Qhull -> solve -> refocus
    from paper_2003_11076_b200.qhull_pool import make_pool
    pool, n_workers = make_pool()
    for _ in st.reconstruct_frames([host_frame] * 4, rig, sp, pp):
        pass
    n_fi = 48
    t0 = time.perf_counter()
    for _ in st.reconstruct_frames([host_frame] * n_fi, rig, sp, pp):
        pass
    torch.cuda.synchronize()
    fi_fps = n_fi / (time.perf_counter() - t0)
    # (f)3 frame directories on disk -> artefact sets on disk (run_reconstruct_sequence)
    import shutil
    import tempfile
    from paper_2003_11076_b200 import pipeline as PL
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    io_dir = tempfile.mkdtemp(prefix="st_bench_io_", dir=base)
    try:
        fdir = os.path.join(io_dir, "frames")
        PL.write_frame_dir(fdir, host_frame, rig)
        calib = os.path.join(fdir, "calib.txt")
        PL.run_reconstruct_sequence(calib, [fdir] * 2, [os.path.join(io_dir, f"w{i}")
                                                         for i in range(2)])
        n_io = 24
        outs = [os.path.join(io_dir, f"o{i}") for i in range(n_io)]
        t0 = time.perf_counter()
        PL.run_reconstruct_sequence(calib, [fdir] * n_io, outs)
        io_fps = n_io / (time.perf_counter() - t0)
        art = sum(os.path.getsize(os.path.join(outs[0], f)) for f in os.listdir(outs[0]))
        inp = sum(os.path.getsize(os.path.join(fdir, f)) for f in os.listdir(fdir))
        t0 = time.perf_counter()
        res = PL.run_reconstruct(calib, fdir, os.path.join(io_dir, "single"))
        single_s = time.perf_counter() - t0
    finally:
        shutil.rmtree(io_dir, ignore_errors=True)
    # (f)4 the device renderer (st_render.cu): one whole synthetic frame
    # (K views + priors + ground truth) to host numpy arrays
    from paper_2003_11076_b200 import synth
    spec = synth.occluder_scene(width=w, height=h, cameras=k, **SCENE)
    synth.render(spec)
    torch.cuda.synchronize()
    n_r = 5
    t0 = time.perf_counter()
    for _ in range(n_r):
        synth.render(spec)
    torch.cuda.synchronize()
    render_ms = (time.perf_counter() - t0) * 1e3 / n_r
    out = {
        "renderer": {"device_frame_ms": render_ms, "config": cfg,
                     "api": "synth.render (device: st_render_view / st_render_background / "
                            "st_corrupt_prior), host numpy frame + ground truth out",
                     "parity": "bit-identical to the reference renderer "
                               "(tests/test_gpu_render.py, bench digests C1-C4)"},
        "harvest": {"device_ms": hv_ms, "includes": "descriptors + st_harvest",
                    "candidates": n_cand, "reverse_scans": n_rev, "grid": nd,
                    "host_d2h_dedup_ms": t_host * 1e3, "points_kept": int(len(u)),
                    "roofline": {"bound": "hbm", "kernel": "k_hv_match (+ k_hv_detect)",
                                 "unit": "GB/s", "achieved": samples * 16 / (hv_ms / 1e3) / 1e9,
                                 "peak": peak, "frac": samples * 16 / (hv_ms / 1e3) / 1e9 / peak,
                                 "algorithmic_bytes": samples * 16,
                                 "unit_note": "16 B per (candidate, disparity) descriptor "
                                              "sample, forward + reverse scans"}},
        "triangulation": {"qhull_host_ms": t_qhull * 1e3, "device_tables_ms": tt_ms,
                          "triangles": int(td.n_tri)},
        "frame_in_stream": {"value": fi_fps, "unit": "frames/s", "frames": n_fi,
                            "qhull_workers": n_workers,
                            "api": "reconstruct_frames (raw frames in, artefacts out)"},
        "frame_io_stream": {"value": io_fps, "unit": "frames/s", "frames": n_io,
                            "input_bytes_per_frame": inp, "artefact_bytes_per_frame": art,
                            "storage": base or "tempdir",
                            "api": "pipeline.run_reconstruct_sequence (frame directories "
                                   "in, artefact directories out)",
                            "single_run_reconstruct_s": single_s,
                            "single_stage_s": res["timings"]},
    }
    if cpu_leg:
        import oracle
        from oracle import harvest as OH
        cams = OH.Cameras([c[0].fx for c in rig.cameras], [c[0].fy for c in rig.cameras],
                          [c[0].cx for c in rig.cameras], [c[0].cy for c in rig.cameras],
                          [c[1].rotation for c in rig.cameras],
                          [c[1].translation for c in rig.cameras], rig.unit_baseline,
                          rig.ref_index, w, h)
        descs = [x.cpu().numpy() for x in pipe.desc]
        flats = [x.reshape(h * w, 16).astype(np.float32) for x in descs]
        view = rig.ref_index
        t0 = time.perf_counter()
        cands = OH.detect(descs[view])
        eroded = OH.ring_min_prior(frame.priors[view])
        cands = cands[eroded[cands[:, 1], cands[:, 0]] >= np.float32(0.7)]
        OH.match(cams, view, cams.nearest_neighbor(view), cands, flats, dmax)
        t_view = time.perf_counter() - t0
        out["harvest"]["cpu_baseline"] = {
            "value": 1.0 / (t_view * k), "unit": "frames/s", "cores": cpu_cores(),
            "kind": "port",
            "sample": f"reference view's detection + SAD match + left-right check through the "
                      f"numpy oracle ({t_view:.2f} s), x{k} views; descriptors from the device"}
        from oracle.synth import render as host_render
        t0 = time.perf_counter()
        host_render(spec)
        t_r = time.perf_counter() - t0
        out["renderer"]["cpu_baseline"] = {
            "value": 1.0 / t_r, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"one whole {cfg} frame through the numpy restatement of the reference "
                      f"renderer (oracle/synth.py, {t_r:.2f} s)"}
    return out


def oracle_sample(frame, rig, tri, cfg, rows):
    """Time the CPU oracle (numpy restatement of the reference) on a band of
    `rows` reference rows; extrapolate to a full frame.

    Full-frame per-frame parts (descriptors, mu raster) are timed in full;
    the per-pixel parts (initial masks, EM, refocus, median) on the band.
    """
    import oracle
    w, h, k, dmax, iters = CONFIGS[cfg]
    sp, pp = params_for(cfg)
    p = oracle.OracleParams(beta=sp.beta, threshold=sp.threshold, max_iters=sp.max_iters,
                            min_static_rays=sp.min_static_rays, epsilon_prior=sp.epsilon_prior,
                            sigma=pp.sigma, gamma=pp.gamma, d_max=pp.d_max,
                            neighborhood_radius=pp.neighborhood_radius)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    sup_uv, sup_d = tri.support_points()
    t0 = time.perf_counter()
    desc = [oracle.descriptors_of(im) for im in frame.images]
    mu = oracle.mu_raster(tri.points, tri.disparities, tri.triangles, tri.planes, w, h)
    t_full = time.perf_counter() - t0
    # evenly strided rows: a representative sample of the frame
    row_ids = np.unique(np.linspace(0, h - 1, rows).round().astype(np.int64))
    rows = row_ids.size
    active = (row_ids[:, None] * w + np.arange(w)[None, :]).ravel()
    s = oracle.OracleSolver(frame.images, frame.priors, a, b, rig.ref_index, mu, sup_uv, sup_d,
                            params=p, descriptors=desc)
    t1 = time.perf_counter()
    res = s.solve(active=active)
    # refocus on the sampled rows, median on a row-proportional slab
    st_band = np.full((h, w), oracle.STATUS_LOW_TEXTURE, np.uint8)
    st_band[row_ids] = res["status"][row_ids]
    img, prov, nr = oracle.synthesize(frame.images, a, b, rig.ref_index, res["values"], st_band,
                                      res["static_bits"], sp.min_static_rays, 0)
    oracle.median_filter(img[:rows], 1)
    t_band = time.perf_counter() - t1
    frac = rows / h
    t_frame = t_full + t_band / frac
    return {"t_frame": t_frame, "t_full": t_full, "t_band": t_band, "rows": rows, "frac": frac,
            "iterations": res["stats"]["iterations_run"]}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def oracle_frame(frame, rig, tri, cfg):
    """One WHOLE frame through the CPU oracle (the numpy restatement of the
    reference): descriptors, surface raster, initial masks, EM with the
    reference's convergence rule, refocus + median -- the timed unit of
    SURVEY.md §8(d) (solver.py:436-502 + refocus.py:109-148), descriptors
    included as for a fresh LightFieldFrame.  Returns seconds."""
    import oracle
    w, h, k, dmax, iters = CONFIGS[cfg]
    sp, pp = params_for(cfg)
    p = oracle.OracleParams(beta=sp.beta, threshold=sp.threshold, max_iters=sp.max_iters,
                            min_static_rays=sp.min_static_rays, epsilon_prior=sp.epsilon_prior,
                            sigma=pp.sigma, gamma=pp.gamma, d_max=pp.d_max,
                            neighborhood_radius=pp.neighborhood_radius)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    sup_uv, sup_d = tri.support_points()
    t0 = time.perf_counter()
    desc = [oracle.descriptors_of(im) for im in frame.images]
    mu = oracle.mu_raster(tri.points, tri.disparities, tri.triangles, tri.planes, w, h)
    s = oracle.OracleSolver(frame.images, frame.priors, a, b, rig.ref_index, mu, sup_uv, sup_d,
                            params=p, descriptors=desc)
    res = s.solve()
    oracle.synthesize(frame.images, a, b, rig.ref_index, res["values"], res["status"],
                      res["static_bits"], sp.min_static_rays, 1)
    return time.perf_counter() - t0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def blas_threads(n):
    """Context manager limiting BLAS (OpenBLAS) threads to n (None = all)."""
    import contextlib
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(n if n is not None else cpu_cores(), user_api="blas")
    except Exception:  # noqa: BLE001
        return contextlib.nullcontext()


def cpu_baseline_block(frame, rig, tri, cfg):
    """cpu_baseline of the GPU arm (rank 0, N = 1): whole frames through the
    oracle on the box's host cores -- the bench config once with all cores
    (`value`), and C1 (the configuration the CPU reference runs,
    BASELINE configs[0]) with one BLAS thread and with all cores."""
    with blas_threads(None):
        t_cfg = oracle_frame(frame, rig, tri, cfg)
    f1, r1, t1, _ = load_inputs("C1")
    with blas_threads(1):
        t_c1_one = oracle_frame(f1, r1, t1, "C1")
    with blas_threads(None):
        t_c1_all = oracle_frame(f1, r1, t1, "C1")
    return {"value": 1.0 / t_cfg, "unit": "frames/s", "cores": cpu_cores(), "kind": "port",
            "sample": f"one whole {cfg} frame (descriptors, surface raster, EM with the "
                      f"reference convergence rule, refocus + median) through the numpy "
                      f"oracle, all cores for BLAS ({t_cfg:.1f} s)",
            "cpu_model": cpu_model(),
            "c1_whole_frame": {"one_thread_s": t_c1_one, "all_cores_s": t_c1_all,
                               "one_thread_fps": 1.0 / t_c1_one,
                               "all_cores_fps": 1.0 / t_c1_all,
                               "note": "C1 = 640x480, K=5, d_max 32 (BASELINE configs[0]); "
                                       "OPENBLAS threads 1 vs all (threadpoolctl)"}}


def run_reference(args):
    """--impl reference: the CPU oracle (numpy restatement of the reference,
    which is pure Python and cannot travel to the GPU box) on WHOLE frames of
    the same config, rank 0 only, all host cores available to BLAS.  Warm-up
    steps run on a 1/16 row band (import and cache warm-up only); every timed
    step is one whole frame."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = args.config
    w, h, k, dmax, iters = CONFIGS[cfg]
    frame, rig, tri, exact = load_inputs(cfg, host=True)  # (none of this repo's kernels)
    with blas_threads(None):
        for _ in range(args.warmup):
            oracle_sample(frame, rig, tri, cfg, rows=max(8, h // 16))
        times = [oracle_frame(frame, rig, tri, cfg) for _ in range(args.steps)]
    t = float(np.mean(times))
    fps = 1.0 / t
    sample = (f"whole {w}x{h} frames, one per step: descriptors, surface raster, EM "
              f"(reference convergence rule), refocus + median through the numpy oracle; "
              f"{cpu_cores()} host cores available to BLAS")
    out = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_block(cfg, args, exact), l2="CPU arm: not applicable"),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cpu_cores(),
                         "kind": "port", "sample": sample, "cpu_model": cpu_model(),
                         "step_s": times},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpix_plane_per_s": w * h * dmax * fps / 1e9,
    }
    print(json.dumps(out), flush=True)


def config_block(cfg, args, exact):
    w, h, k, dmax, iters = CONFIGS[cfg]
    return {"workload": f"{cfg}: {k}-camera linear array {w}x{h}, {int(dmax)} depth planes "
                        f"(d_max), max {iters} EM iters with the reference convergence rule; "
                        f"solve + refocus + median per frame",
            "width": w, "height": h, "views": k, "d_max": dmax, "max_iters": iters,
            "scene": "occluder_scene(coverage=0.25, seed=11, p_flip=0.1, blur_radius=2)",
            "inputs_match_reference_digest": bool(exact),
            "l2": f"{args.value_slots} resident frame slots rotate, each on its own compute "
                  f"stream (frames in flight concurrently); their ~{150 * args.value_slots} MB "
                  f"working set exceeds the 126 MB L2, no flush",
            "parallelism": f"frame-parallel x{args.gpus}" if args.gpus > 1 else "1 GPU",
            "forced_iters": args.forced_iters or None}


# -- C5: a 1000-frame sequence of 16 distinct frames, frame-parallel -------------------------

C5_FRAMES, C5_DISTINCT, C5_SEED0 = 1000, 16, 11


def _render_c5(seed):
    """One distinct C5 frame (occluder_scene seeds 11..26),
    rendered on the device."""
    from paper_2003_11076_b200 import synth
    w, h, k, dmax, iters = CONFIGS["C2"]
    sc = dict(SCENE, seed=seed)
    frame, _ = synth.render(synth.occluder_scene(width=w, height=h, cameras=k, **sc))
    return np.stack(frame.images), np.stack(frame.priors)


def measure_sequence(dist, rank, world, flush=None):
    """BASELINE configs[4]: 1000 frames cycling 16 distinct rendered C2 frames,
    split frame-parallel over the ranks (frame i on rank i % N), through the
    pipelined public API from pinned host memory with the artefacts copied
    back (host I/O inside the timed region).  The 16 frames' support points
    and triangulations are computed once (device harvest + host Qhull), not
    timed, as SURVEY.md §8d prescribes.  Total work is fixed: strong
    scaling; time = max over ranks."""
    import torch
    import paper_2003_11076_b200 as st
    from paper_2003_11076_b200 import _native as N
    w, h, k, dmax, iters = CONFIGS["C2"]
    sp, pp = params_for("C2")
    mine = [i for i in range(C5_FRAMES) if i % world == rank]
    need = sorted({i % C5_DISTINCT for i in mine})
    t0 = time.perf_counter()
    rendered = {j: _render_c5(C5_SEED0 + j) for j in need}
    t_render = time.perf_counter() - t0
    from paper_2003_11076_b200 import synth
    rig = synth.occluder_scene(width=w, height=h, cameras=k, **SCENE).rig()
    pairs = {}
    t0 = time.perf_counter()
    for j, (imgs, pris) in rendered.items():
        pin_i = st.device.pinned_empty(imgs.shape, np.uint8)
        pin_p = st.device.pinned_empty(pris.shape, np.float32)
        pin_i[...] = imgs
        pin_p[...] = pris
        frame = st.LightFieldFrame(images=list(pin_i), priors=list(pin_p))
        sup = st.collect_support(frame, rig, pp, threshold=sp.threshold)
        pairs[j] = (frame, st.triangulate(sup, w, h))
    t_prep = time.perf_counter() - t0
    seq = [pairs[i % C5_DISTINCT] for i in mine]

    def run(items):
        n = 0
        for _ in st.reconstruct_stream(items, rig, sp, pp):
            n += 1
        return n

    run(seq[:8])  # warm-up
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    g0 = N.lib().st_tail_graph_count(0)
    t0 = time.perf_counter()
    n = run(seq)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    graph_builds = N.lib().st_tail_graph_count(0) - g0
    if dist is not None:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    assert n == len(mine)
    f0 = pairs[need[0]][0]
    h2d = sum(a.nbytes for a in f0.images) + sum(a.nbytes for a in f0.priors)
    return {"config": "C5", "frames": C5_FRAMES, "distinct_frames": C5_DISTINCT,
            "value": C5_FRAMES / (ms / 1e3), "unit": "frames/s", "n_gpus": world,
            "ms_total": ms, "scaling": "strong",
            "frames_per_rank": len(mine), "distinct_per_rank": len(need),
            "h2d_frame_bytes": int(h2d), "d2h_bytes_per_frame": int(w * h * 18),
            "api": "reconstruct_stream from pinned host frames, artefacts to host, "
                   "host wall clock, max over ranks",
            "untimed_setup_s": {"render": t_render, "support_and_triangulation": t_prep},
            "tail_graphs_built_in_timed_region": int(graph_builds)}


# -- row bands (BASELINE C3/C4: one frame split across the ranks) -------------------------

def measure_row_bands(cfg, steps, warmup, dist, rank, world, flush):
    """One frame per step split into `world` row bands (sharding.BandPipeline):
    per-rank band descriptors, whole-frame surface raster + support groups,
    the banded EM with its per-iteration record all-gather (NCCL), the band
    refocus + median, and the NCCL gather of the artefact bands to rank 0.
    `value`: device-resident inputs (CUDA events, max over ranks); `e2e`:
    each rank's band rows from pinned host memory + the Qhull tables, and
    rank 0's full-frame artefacts back to the host (wall clock, max over
    ranks).  Strong scaling: the frame is fixed, the ranks share it."""
    import torch
    import paper_2003_11076_b200 as st
    from paper_2003_11076_b200.prior import TriDevice
    from paper_2003_11076_b200.sharding import BandPipeline
    w, h, k, dmax, iters = CONFIGS[cfg]
    sp, pp = params_for(cfg)
    frame, rig, tri, exact = load_inputs(cfg)
    bp = BandPipeline(rig, w, h, sp, pp)
    pin_imgs = [st.device.pinned_empty(im.shape, np.uint8) for im in frame.images]
    pin_pris = [st.device.pinned_empty(q.shape, np.float32) for q in frame.priors]
    for d_, s_ in zip(pin_imgs, frame.images):
        d_[...] = s_
    for d_, s_ in zip(pin_pris, frame.priors):
        d_[...] = s_
    bp.load(pin_imgs, pin_pris)
    td = TriDevice(tri)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_ranks(x):
        if dist is not None:
            tt = torch.tensor([x], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            x = float(tt.item())
        return x

    for _ in range(warmup):
        bp.run(td)
        bp.gather()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        bp.run(td)
        bp.gather()
        ev[i][1].record(stream)
    barrier()
    total = max_ranks(float(sum(a.elapsed_time(b) for a, b in ev)))
    stats = bp.stats()
    # e2e: band rows H2D (pinned), Qhull tables H2D, compute, gather, rank-0 D2H
    host = None
    barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        bp.load(pin_imgs, pin_pris)
        tdi = TriDevice(tri)
        bp.run(tdi)
        bp.gather()
        if rank == 0:
            host = bp.pipe.fetch()
        else:
            stream.synchronize()
    torch.cuda.synchronize()
    e2e_ms = max_ranks((time.perf_counter() - t0) * 1e3)
    h2d = max_ranks(float(bp.h2d_bytes() + td.nbytes))
    return {
        "config": cfg, "value": steps / (total / 1e3), "unit": "frames/s", "n_gpus": world,
        "ms_per_step": total / steps, "scaling": "strong",
        "e2e": {"value": steps / (e2e_ms / 1e3), "unit": "frames/s",
                "h2d_bytes_per_step_max_rank": int(h2d),
                "d2h_bytes_per_step": int(bp.pipe.output_bytes()) if host is not None else None,
                "ms_per_step": e2e_ms / steps},
        "band_rows": list(bp.ext["rows"]), "solved_rows": list(bp.ext["solve"]),
        "input_rows": list(bp.ext["images"]),
        "iterations_run": stats.iterations_run, "converged_after": stats.converged_after,
        "inputs_match_reference_digest": bool(exact),
        "replicated_per_rank": "surface raster (Qhull walk replay) and support groups "
                               "over the whole frame",
        "collectives": "per EM iteration all_gather of 96-byte records (NCCL, "
                       "stream-ordered); artefact band gather to rank 0 (NCCL p2p group)",
    }


def run_rows(args):
    """--shard rows: the row-band line (BASELINE configs[2]: C3 at 1/2/4/8)."""
    import torch
    from paper_2003_11076_b200 import _native as N
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import datetime
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=300))
    cfg = args.config
    w, h, k, dmax, iters = CONFIGS[cfg]
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    lib = N.lib()
    l0 = lib.st_launch_count()
    with ClockSampler(local) as clocks:
        r = measure_row_bands(cfg, args.steps, args.warmup, dist, rank, world, flush)
    launches = lib.st_launch_count() - l0
    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        peak = float(json.load(open(peaks_path))["hbm_gbs"]) if os.path.exists(peaks_path) \
            else 6650.0
        out = {
            "metric": METRIC, "value": r["value"], "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference renderer, reference support harvest)",
            "config": dict(config_block(cfg, args, r["inputs_match_reference_digest"]),
                           parallelism=f"row bands x{world}",
                           l2="flushed between steps (256 MiB write)"),
            "e2e": {"value": r["e2e"]["value"], "unit": "frames/s",
                    "h2d_bytes_per_step": r["e2e"]["h2d_bytes_per_step_max_rank"],
                    "d2h_bytes_per_step": r["e2e"]["d2h_bytes_per_step"]},
            "gpu_launches": int(launches), "clocks": clocks.summary(),
            "row_bands": r,
            "roofline": None, "cpu_baseline": None,
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# -- GPU arm ------------------------------------------------------------------------------

def run_ours(args):
    import torch
    import paper_2003_11076_b200 as st
    from paper_2003_11076_b200 import _native as N
    from paper_2003_11076_b200.prior import TriDevice
    from paper_2003_11076_b200.reconstruct import FramePipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    w, h, k, dmax, iters = CONFIGS[cfg]
    sp, pp = params_for(cfg)
    frame, rig, tri, exact = load_inputs(cfg)
    lib = N.lib()

    # device-resident inputs
    pipe = FramePipeline(rig, w, h, sp, pp)
    pipe.load(frame.images, frame.priors)
    tdev = TriDevice(tri)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # -- value: K frames on resident inputs, the production way: VALUE_SLOTS
    # frame slots rotate, each on its own compute stream (the frames are
    # independent: several are in flight, the EM's small latency-bound
    # worklist grids of one frame leave SMs to the others), each frame's
    # pre-solve stages (side streams: surface raster, descriptors, support
    # groups) starting as soon as its slot is free.  The slots' working set
    # (~150 MB each: views, priors, descriptor maps, EM state) exceeds the
    # 126 MB L2, so no flush is needed between steps.
    n_slots = max(1, args.value_slots)
    slots = [(pipe, tdev)]
    for _ in range(n_slots - 1):
        px = FramePipeline(rig, w, h, sp, pp)
        px.load(frame.images, frame.priors)
        slots.append((px, TriDevice(tri)))
    done_ev = [None] * n_slots

    def pipelined(n, start=None):
        """Enqueue n frames over the slots; returns the joined end event."""
        if start is None:
            start = torch.cuda.Event()
            start.record(stream)
        for j in range(n):
            pp_, td_ = slots[j % n_slots]
            cs = pp_.compute
            # the slot is free once its previous frame finished
            cs.wait_event(done_ev[j % n_slots] if done_ev[j % n_slots] is not None else start)
            ready = torch.cuda.Event()
            ready.record(cs)
            with torch.cuda.stream(cs):
                pp_.run(td_, forced_iters=args.forced_iters, ready=ready)
            ev = torch.cuda.Event()
            ev.record(cs)
            done_ev[j % n_slots] = ev
        for pp_, _ in slots:
            stream.wait_stream(pp_.compute)
        end = torch.cuda.Event(enable_timing=True)
        end.record(stream)
        return end

    pipelined(max(args.warmup, 2 * n_slots))
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    launches0 = lib.st_launch_count()
    with ClockSampler(local) as clocks:  # (NVML starts before the first event)
        p0.record(stream)
        p1 = pipelined(args.steps, p0)
        barrier()
    launches = lib.st_launch_count() - launches0
    total_ms = p0.elapsed_time(p1)
    if dist is not None:
        tt = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    fps = world * args.steps / (total_ms / 1e3)

    # -- one frame at a time, L2 flushed before each (the single-frame latency)
    for _ in range(3):
        pipe.run(tdev, forced_iters=args.forced_iters)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        starts[i].record(stream)
        pipe.run(tdev, forced_iters=args.forced_iters)
        ends[i].record(stream)
    barrier()
    latency_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(starts, ends)]))
    # per-stage / per-kernel CUDA-event breakdown of the same workload (the
    # synchronous solve variant records events around every kernel group)
    stats = []
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        stats.append(pipe.run(tdev, forced_iters=args.forced_iters, timing=True))
    barrier()

    if args.quick:
        if rank == 0:
            print(json.dumps({"value": fps, "ms_per_step": total_ms / args.steps,
                              "single_frame_ms": latency_ms,
                              "stage_ms": {n: float(np.mean([s.stage_ms[n] for s in stats]))
                                           for n in stats[0].stage_ms},
                              "kernel_ms": [float(np.mean([s.kernel_ms[j] for s in stats]))
                                            for j in range(4)],
                              "energy_evals": stats[0].energy_evals,
                              "hopeless_msteps": stats[0].hopeless_msteps,
                              "energy_samples": stats[0].energy_samples}), flush=True)
        return

    # -- e2e: public API from pinned host memory, artefacts back to the host ----------
    pin_imgs = [st.device.pinned_empty(im.shape, np.uint8) for im in frame.images]
    pin_pris = [st.device.pinned_empty(p.shape, np.float32) for p in frame.priors]
    for d, s in zip(pin_imgs, frame.images):
        d[...] = s
    for d, s in zip(pin_pris, frame.priors):
        d[...] = s
    host_frame = st.LightFieldFrame(images=pin_imgs, priors=pin_pris)
    e2e_steps = max(3, args.e2e_frames)

    def e2e_single():
        # one synchronous reconstruct() call per frame
        for _ in range(2):
            st.reconstruct(host_frame, rig, tri, sp, pp, forced_iters=args.forced_iters)
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            st.reconstruct(host_frame, rig, tri, sp, pp, forced_iters=args.forced_iters)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    def e2e_stream():
        # the pipelined public API: H2D / compute / D2H of consecutive frames overlap
        for _ in st.reconstruct_stream([(host_frame, tri)] * 8, rig, sp, pp,
                                       forced_iters=args.forced_iters):
            pass
        barrier()
        t0 = time.perf_counter()
        n = 0
        for _ in st.reconstruct_stream([(host_frame, tri)] * e2e_steps, rig, sp, pp,
                                       forced_iters=args.forced_iters):
            n += 1
        torch.cuda.synchronize()
        assert n == e2e_steps
        return (time.perf_counter() - t0) * 1e3

    def max_ranks(ms):
        if dist is not None:
            tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    def e2e_dropin(n):
        # the reference's own entry points (solver.py:505-508 em_solve,
        # refocus.py:109 synthesize) on pageable numpy frames, a fresh
        # LightFieldFrame per step (descriptors recomputed, as the reference
        # computes them per frame), numpy artefacts back
        imgs = [np.array(x) for x in frame.images]
        pris = [np.array(x) for x in frame.priors]

        def one():
            f = st.LightFieldFrame(images=imgs, priors=pris)
            dmap, seg, _ = st.em_solve(f, rig, tri, sp, pp)
            st.synthesize(f, rig, dmap, seg, min_static_rays=sp.min_static_rays,
                          median_radius=1)
        for _ in range(2):
            one()
        barrier()
        t0 = time.perf_counter()
        for _ in range(n):
            one()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    def dyn_stream(n):
        # dynamic_only (PAPER.md:242 person-only mode, solver.py:449-452,
        # pipeline.py:250-260) through the pipelined public API; like e2e:
        # every slot warmed, the median of 3 streams
        for _ in st.reconstruct_stream([(host_frame, tri)] * 12, rig, sp, pp, dynamic_only=True):
            pass
        reps = []
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            for _ in st.reconstruct_stream([(host_frame, tri)] * n, rig, sp, pp,
                                           dynamic_only=True):
                pass
            torch.cuda.synchronize()
            reps.append((time.perf_counter() - t0) * 1e3)
        return float(np.median(reps))

    dropin_n = 10
    dropin_ms = max_ranks(e2e_dropin(dropin_n))
    dyn_n = max(10, e2e_steps)
    dyn_ms = max_ranks(dyn_stream(dyn_n))
    # resident dynamic_only frames (CUDA events, L2 flushed between steps)
    pipe.run(tdev, dynamic_only=True)
    torch.cuda.synchronize()
    dyn_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        dyn_ev[i][0].record(stream)
        pipe.run(tdev, dynamic_only=True)
        dyn_ev[i][1].record(stream)
    barrier()
    dyn_res_ms = max_ranks(float(sum(a.elapsed_time(b) for a, b in dyn_ev)))
    single_ms = max_ranks(e2e_single())
    # host-side throughput is sensitive to host noise: median of five streams,
    # after two untimed ones (the pinned host allocator fills its cache of
    # artefact blocks during the first streams)
    for _ in range(2):
        e2e_stream()
    e2e_reps = [max_ranks(e2e_stream()) for _ in range(5)]
    e2e_ms = float(np.median(e2e_reps))
    e2e_fps = world * e2e_steps / (e2e_ms / 1e3)
    tdv = TriDevice(tri)
    h2d = sum(a.nbytes for a in pin_imgs) + sum(a.nbytes for a in pin_pris) + tdv.nbytes
    d2h = pipe.output_bytes()

    # -- forced-5 (non-reference bench mode): exactly max_iters EM iterations -----------
    forced = None
    if not args.forced_iters and args.forced_steps > 0:
        pipe.run(tdev, forced_iters=iters)
        torch.cuda.synchronize()
        fs = torch.cuda.Event(enable_timing=True)
        fe = torch.cuda.Event(enable_timing=True)
        fms = 0.0
        for _ in range(args.forced_steps):
            flush.fill_(1)
            fs.record(stream)
            pipe.run(tdev, forced_iters=iters)
            fe.record(stream)
            fe.synchronize()
            fms += fs.elapsed_time(fe)
        forced = {"iterations": iters, "fps_per_gpu": args.forced_steps / (fms / 1e3),
                  "ms_per_frame": fms / args.forced_steps}

    # -- BASELINE configs[2]: the C3 frame split into row bands over the same ranks
    row_bands = None
    if args.row_band_steps > 0 and not args.forced_iters:
        try:
            row_bands = measure_row_bands("C3", args.row_band_steps, 3, dist, rank, world, flush)
        except Exception as exc:  # noqa: BLE001 -- reported, the frame-parallel line stands
            row_bands = {"error": f"{type(exc).__name__}: {exc}"}

    # -- BASELINE configs[4]: the C5 sequence (1000 frames, 16 distinct) over the ranks
    sequence = None
    if args.sequence and not args.forced_iters:
        try:
            sequence = measure_sequence(dist, rank, world)
        except Exception as exc:  # noqa: BLE001 -- reported, the main line stands
            sequence = {"error": f"{type(exc).__name__}: {exc}"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # -- roofline of the dominant kernel (k_m_step) ---------------------------------------
    s0 = stats[-1]
    ms_m = float(np.mean([s.kernel_ms[0] for s in stats]))
    n_m = s0.kernel_launches[0]
    # 16 B per (pixel, candidate, view) descriptor sample.  The
    # kernel samples only the real candidates it evaluates exactly (the
    # survivors of the exact prior-bound pruning, plus the previous-disparity
    # energies), one sample per static in-margin view: counted on the device
    # (st_stats.energy_samples).  The SURVEY model charges every candidate.
    samples_m = s0.energy_samples
    bytes_m = samples_m * 16
    model_bytes_m = (s0.candidates_total + s0.prev_evals) * k * 16
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured"
    else:
        peak, peak_src = 6650.0, "fallback"
    achieved = bytes_m / (ms_m / 1e3) / 1e9
    model_achieved = model_bytes_m / (ms_m / 1e3) / 1e9
    npx = w * h
    c_bar = s0.candidates_total / max(1, s0.msteps)
    # SURVEY 8d model, charged for the pixel M/E-steps the incremental EM runs
    frame_bytes = s0.msteps * c_bar * k * 16 + s0.esteps * k * 20 + npx * 7 * k
    # the same model charging every pixel every iteration (full recompute)
    model_full = npx * (s0.iterations_run * (c_bar * k * 16 + k * 20) + 7 * k)
    step_ms_mean = total_ms / args.steps
    traffic = None
    pipes = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    if os.path.exists(prof):
        tj = json.load(open(prof))
        traffic = tj.get("k_m_step_dram_bytes_per_launch")
        pipes = tj.get("k_m_step_pipes")
        if pipes is not None:
            pipes = dict(pipes, source=tj.get("source"),
                         note="the bound that binds: FP64 issue + latency, not HBM")

    # the bound that binds k_m_step: FP64 issue.  The device's DFMA peak is
    # measured here; the kernel's FP64 flops per launch come from the ncu
    # capture summarised in profiles/traffic_<cfg>.json
    fp64_peak = N.C.c_double(0.0)
    N.check(lib.st_fp64_peak(N.C.byref(fp64_peak), N.stream_handle()))
    fp64 = {"peak_tflops": fp64_peak.value, "peak_source": "measured (st_fp64_peak: 8 "
            "independent DFMA chains per thread)"}
    if prof and os.path.exists(prof):
        tj = json.load(open(prof))
        fl = tj.get("k_m_step_fp64_flops_per_launch")
        if fl:
            fp64["k_m_step_flops_per_launch"] = fl
            fp64["k_m_step_tflops"] = fl / (ms_m / max(1, n_m) / 1e3) / 1e12
            fp64["frac"] = fp64["k_m_step_tflops"] / fp64_peak.value
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_block(frame, rig, tri, cfg)

    nxt = None
    if world == 1 and not args.no_next_rows:
        nxt = next_rows(frame, rig, cfg, pipe, host_frame, peak,
                        cpu_leg=not args.no_cpu_baseline)

    out = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_mean,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference renderer, reference support harvest; "
                f"digest match {exact})",
        "config": config_block(cfg, args, exact),
        "roofline": {"bound": "hbm", "kernel": "k_m_step", "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "pipes": pipes, "fp64": fp64,
                     "algorithmic_bytes_per_launch": bytes_m / max(1, n_m),
                     "unit_note": "16 B per descriptor sample the kernel takes: (pixel, "
                                  "evaluated real candidate, static in-margin view), "
                                  "counted on the device",
                     "launch_ms": ms_m / max(1, n_m), "launches_per_step": n_m,
                     # the step as ncu sees it: one frame at a time (the launch list
                     # is serialised), not the concurrent slots' 1/fps
                     "share_of_step": ms_m / latency_ms,
                     "share_of_concurrent_step": ms_m / step_ms_mean,
                     "model": {"algorithmic_bytes_per_launch": model_bytes_m / max(1, n_m),
                               "achieved": model_achieved, "frac": model_achieved / peak,
                               "note": "SURVEY 8d charges every candidate; exact pruning "
                                       "evaluates a small fraction of them, hence "
                                       "frac > 1"}},
        "frame_roofline": {"model_bytes": frame_bytes, "achieved_gbs":
                           frame_bytes / (step_ms_mean / 1e3) / 1e9,
                           "frac": frame_bytes / (step_ms_mean / 1e3) / 1e9 / peak,
                           "model_bytes_full_recompute": model_full,
                           "frac_full_recompute_model":
                               model_full / (step_ms_mean / 1e3) / 1e9 / peak},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms / e2e_steps,
                "api": "reconstruct_stream (pipelined), host wall clock incl. all streams; "
                       "median of 5 streams",
                "reps_ms_per_step": [x / e2e_steps for x in e2e_reps],
                "single_call_fps": world * e2e_steps / (single_ms / 1e3),
                "dropin_fps": world * dropin_n / (dropin_ms / 1e3),
                "dropin_api": "em_solve + synthesize (the reference entry points) on "
                              "pageable numpy frames, fresh LightFieldFrame per step"},
        "dynamic_only": {"e2e_stream_fps": world * dyn_n / (dyn_ms / 1e3),
                         "resident_fps": world * args.steps / (dyn_res_ms / 1e3),
                         "resident_ms_per_step": dyn_res_ms / args.steps,
                         "note": "person-only mode (PAPER.md:242; solver.py:449-452): "
                                 "st_solve_rows (the active count stays on the device: no host "
                                 "read-back; iterations >= 3 in the graph loop)"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "em": {"iterations_run": s0.iterations_run, "converged_after": s0.converged_after,
               "candidates_per_mstep": c_bar,
               "energy_evals_per_mstep": s0.energy_evals / max(1, s0.msteps),
               "samples_per_mstep": s0.energy_samples / max(1, s0.msteps),
               "hopeless_msteps": s0.hopeless_msteps,
               "pixel_msteps": s0.msteps, "pixel_esteps": s0.esteps,
               "kernel_ms": {"m_step": ms_m,
                             "e_step": float(np.mean([s.kernel_ms[1] for s in stats])),
                             "initial_masks": float(np.mean([s.kernel_ms[2] for s in stats])),
                             "reduce": float(np.mean([s.kernel_ms[3] for s in stats]))},
               "stage_ms": {n: float(np.mean([s.stage_ms[n] for s in stats]))
                            for n in stats[0].stage_ms}},
        "gpix_plane_per_s": w * h * dmax * fps / 1e9,
        "forced_iters_mode": forced,
        "row_bands_C3": row_bands,
        "sequence_C5": sequence,
        "next_rows": nxt,
        "single_frame": {"value": 1e3 / latency_ms, "unit": "frames/s",
                         "ms_per_frame": latency_ms,
                         "note": "one frame at a time on one slot, L2 flushed (256 MiB "
                                 "write) before each: the per-frame latency"},
    }
    print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default C2 (C3 with --shard rows)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--forced-iters", type=int, default=0)
    ap.add_argument("--forced-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="value loop only (profiling)")
    ap.add_argument("--no-next-rows", action="store_true",
                    help="skip the harvest / triangulation / frame-in measurements")
    ap.add_argument("--e2e-frames", type=int, default=60,
                    help="frames per timed e2e stream (steady-state throughput)")
    ap.add_argument("--shard", default="frames", choices=["frames", "rows"],
                    help="multi-GPU split: frames (C5 frame-parallel, default) or rows "
                         "(one frame in row bands, C3/C4)")
    ap.add_argument("--value-slots", type=int, default=4,
                    help="resident frame slots (each its own compute stream) in the value loop")
    ap.add_argument("--row-band-steps", type=int, default=10,
                    help="frame-parallel runs also time C3 row bands over the same ranks "
                         "(0 = skip)")
    ap.add_argument("--no-sequence", dest="sequence", action="store_false",
                    help="skip the C5 sequence (1000 frames, 16 distinct) measurement")
    ap.add_argument("--budget", type=float, default=150.0,
                    help="reference arm: seconds for the whole run")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.config is None:
        args.config = "C3" if args.shard == "rows" else "C2"
    if args.impl == "reference":
        run_reference(args)
    elif args.shard == "rows":
        run_rows(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
