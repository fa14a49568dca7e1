"""Frame directories in, artefact sets out.

Drop-in for the reference's `pipeline.run_reconstruct` (pipeline.py:
233-287) and the frame-directory loader it uses (pipeline.py:154-184),
with the same file names, config keys, error texts and artefact bytes:

    disparity.pgm (16-bit, fixed point x256), disparity_scale.txt,
    refocused.ppm, provenance.pgm, status.pgm, n_rays.pgm, seg_XX.pgm,
    valid_XX.pgm, config_used.txt, em_stats.txt, timings.txt

The compute stages run on the device (`reconstruct_frame`: device harvest
+ native dedup, host Qhull, device solve + refocus); only parsing, file
I/O and PNM framing stay on the host.  `run_reconstruct_sequence` streams
many frame directories through `reconstruct_frames` (pinned H2D, Qhull
process pool, pipelined device solve) with the artefact writes on a
thread pool, for sequence throughput (BASELINE C5).
"""

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import pnm
from .frame import LightFieldFrame
from .geometry import CalibrationError, load_calibration
from .prior import PriorParams
from .refocus import PROV_COPIED, PROV_FALLBACK, PROV_REFOCUSED  # noqa: F401
from .solver import STATUS_VALID, SolverParams

DISPARITY_SCALE = 256.0


class PipelineError(Exception):
    """Input or artefact problem; maps to process exit code 2 (pipeline.py:44-47)."""

    exit_code = 2


# -- configuration (pipeline.py:52-113) --------------------------------------------

def _boolean(text):
    word = text.strip().lower()
    if word in ("1", "true", "yes", "on"):
        return True
    if word in ("0", "false", "no", "off"):
        return False
    raise ValueError(f"not a boolean: {text!r}")


_OPTIONS = {
    "beta": float, "sigma": float, "gamma": float, "d_max": float, "threshold": float,
    "max_iters": int, "min_static_rays": int, "epsilon_prior": float,
    "median_radius": int, "dynamic_only": _boolean,
}
_SOLVER_KEYS = ("beta", "threshold", "max_iters", "min_static_rays", "epsilon_prior")
_PRIOR_KEYS = ("sigma", "gamma", "d_max")


def parse_config(path):
    """`key = value` lines with '#' comments -> dict of typed overrides."""
    out = {}
    with open(path, "r") as fh:
        for n, raw in enumerate(fh, start=1):
            text = raw.split("#", 1)[0].strip()
            if not text:
                continue
            if "=" not in text:
                raise PipelineError(f"{path}:{n}: expected key = value")
            key, _, value = (s.strip() for s in text.partition("="))
            if key not in _OPTIONS:
                raise PipelineError(f"{path}:{n}: unknown option {key!r}")
            try:
                out[key] = _OPTIONS[key](value)
            except ValueError:
                raise PipelineError(f"{path}:{n}: bad value for {key}: {value!r}")
    return out


def resolve_params(overrides=None):
    """overrides -> (SolverParams, PriorParams, median_radius, dynamic_only)."""
    rest = dict(overrides or {})
    solver, prior = SolverParams(), PriorParams()
    for key in _SOLVER_KEYS:
        if key in rest:
            setattr(solver, key, rest.pop(key))
    for key in _PRIOR_KEYS:
        if key in rest:
            setattr(prior, key, rest.pop(key))
    median_radius = int(rest.pop("median_radius", 1))
    dynamic_only = bool(rest.pop("dynamic_only", False))
    if rest:
        raise PipelineError(f"unknown options: {sorted(rest)}")
    if median_radius < 0:
        raise PipelineError("median_radius must be >= 0")
    return solver, prior, median_radius, dynamic_only


# -- frame directories (pipeline.py:151-184) ----------------------------------------

def view_name(stem, k, ext):
    return f"{stem}_{k:02d}.{ext}"


def load_frame_dir(rig, frames_dir, priors_dir=None):
    """view_XX.ppm + prior_XX.pgm for every camera of the rig -> LightFieldFrame."""
    priors_dir = priors_dir or frames_dir
    images, priors = [], []
    for k in range(len(rig)):
        vpath = os.path.join(frames_dir, view_name("view", k, "ppm"))
        ppath = os.path.join(priors_dir, view_name("prior", k, "pgm"))
        for what, path in (("image", vpath), ("prior", ppath)):
            if not os.path.exists(path):
                raise PipelineError(f"view {k}: missing {what} {path}")
        img = pnm.read_pnm(vpath)
        if img.ndim != 3:
            raise PipelineError(f"view {k}: {vpath} is not a color image")
        intr = rig.intrinsics(k)
        if img.shape[:2] != (intr.height, intr.width):
            raise PipelineError(f"view {k}: image is {img.shape[1]}x{img.shape[0]}, "
                                f"calibration says {intr.width}x{intr.height}")
        pri = pnm.read_pnm(ppath)
        if pri.ndim != 2:
            raise PipelineError(f"view {k}: {ppath} is not grayscale")
        if pri.shape != img.shape[:2]:
            raise PipelineError(f"view {k}: prior is {pri.shape[1]}x{pri.shape[0]}, "
                                f"image is {img.shape[1]}x{img.shape[0]}")
        full = 65535.0 if pri.dtype == np.uint16 else 255.0
        images.append(img)
        priors.append(pri.astype(np.float32) / full)
    return LightFieldFrame(images=images, priors=priors)


def write_frame_dir(out_dir, frame, rig):
    """The input half of the reference's run_synth writes (pipeline.py:338-345):
    calib.txt, view_XX.ppm and the 8-bit coded prior_XX.pgm."""
    from .geometry import save_calibration
    os.makedirs(out_dir, exist_ok=True)
    save_calibration(rig, os.path.join(out_dir, "calib.txt"))
    for k in range(frame.num_views):
        pnm.write_ppm(os.path.join(out_dir, view_name("view", k, "ppm")), frame.images[k])
        code = np.clip(np.rint(np.asarray(frame.priors[k]) * 255.0), 0, 255).astype(np.uint8)
        pnm.write_pgm(os.path.join(out_dir, view_name("prior", k, "pgm")), code)


# -- artefacts (pipeline.py:187-193, 247-305) -------------------------------------

def disparity_code(disparity):
    """16-bit fixed point x256, 0 where the status is not VALID."""
    code = np.zeros(disparity.values.shape, dtype=np.uint16)
    ok = disparity.status == STATUS_VALID
    code[ok] = np.clip(np.rint(disparity.values[ok] * DISPARITY_SCALE), 0, 65535).astype(np.uint16)
    return code


def _config_text(solver, prior, median_radius, dynamic_only):
    rows = [("beta", repr(solver.beta)), ("sigma", repr(prior.sigma)),
            ("gamma", repr(prior.gamma)), ("d_max", repr(prior.d_max)),
            ("threshold", repr(solver.threshold)), ("max_iters", str(solver.max_iters)),
            ("min_static_rays", str(solver.min_static_rays)),
            ("epsilon_prior", repr(solver.epsilon_prior)),
            ("median_radius", str(median_radius)), ("dynamic_only", str(int(dynamic_only)))]
    return "".join(f"{k} = {v}\n" for k, v in rows)


def _stats_text(stats):
    def row(values):
        return ",".join(repr(float(v)) for v in values)
    conv = "none" if stats.converged_after is None else str(stats.converged_after)
    return (f"iterations_run = {stats.iterations_run}\n"
            f"converged_after = {conv}\n"
            f"mean_energy = {row(stats.mean_energy)}\n"
            f"prev_energy = {row(stats.prev_energy)}\n"
            f"changed_fraction = {row(stats.changed_fraction)}\n")


def artefact_files(rec, num_views, solver, prior, median_radius, dynamic_only):
    """{file name: bytes} of one run's artefact set, timings.txt excluded."""
    files = {
        "disparity.pgm": pnm.encode_pgm(disparity_code(rec.disparity)),
        "disparity_scale.txt": f"{int(DISPARITY_SCALE)}\n".encode(),
        "refocused.ppm": pnm.encode_ppm(rec.image),
        "provenance.pgm": pnm.encode_pgm(rec.provenance),
        "status.pgm": pnm.encode_pgm(rec.disparity.status),
        "n_rays.pgm": pnm.encode_pgm(rec.n_rays),
    }
    sb = rec.segmentation.static_bits.astype(np.uint32)
    vb = rec.segmentation.valid_bits.astype(np.uint32)
    for k in range(num_views):
        files[view_name("seg", k, "pgm")] = pnm.encode_pgm(
            (((sb >> np.uint32(k)) & np.uint32(1)) * 255).astype(np.uint8))
        files[view_name("valid", k, "pgm")] = pnm.encode_pgm(
            (((vb >> np.uint32(k)) & np.uint32(1)) * 255).astype(np.uint8))
    files["config_used.txt"] = _config_text(solver, prior, median_radius, dynamic_only).encode()
    files["em_stats.txt"] = _stats_text(rec.stats).encode()
    return files


def _write_files(out_dir, files):
    os.makedirs(out_dir, exist_ok=True)
    for name, data in files.items():
        with open(os.path.join(out_dir, name), "wb") as fh:
            fh.write(data)


def _encode_and_write(out_dir, rec, num_views, solver, prior, median_radius, dynamic_only):
    _write_files(out_dir, artefact_files(rec, num_views, solver, prior, median_radius,
                                         dynamic_only))


def _write_timings(out_dir, timings, threads):
    text = "" if threads is None else f"# threads_hint = {threads}\n"
    text += "".join(f"{name} {sec:.3f}\n" for name, sec in timings)
    text += f"total {sum(s for _, s in timings):.3f}\n"
    with open(os.path.join(out_dir, "timings.txt"), "w") as fh:
        fh.write(text)


def _setup(calib_path, config, ref_index, dynamic_only):
    overrides = parse_config(config) if isinstance(config, str) else dict(config or {})
    solver, prior, median_radius, cfg_dynamic = resolve_params(overrides)
    if dynamic_only is not None:
        cfg_dynamic = bool(dynamic_only)
    try:
        rig = load_calibration(calib_path, ref_index=ref_index)
    except (CalibrationError, OSError) as exc:
        raise PipelineError(f"calibration: {exc}")
    return rig, solver, prior, median_radius, cfg_dynamic


def _load(rig, frames_dir, priors_dir):
    try:
        return load_frame_dir(rig, frames_dir, priors_dir)
    except PipelineError:
        raise
    except (ValueError, OSError) as exc:
        raise PipelineError(str(exc))


def run_reconstruct(calib_path, frames_dir, out_dir, priors_dir=None, config=None,
                    ref_index=None, dynamic_only=None, threads=None):
    """pipeline.py:233-287: solve one frame directory and write its artefacts.

    `threads` is a hint only, as in the reference: no output depends on it.
    Returns {"out_dir", "stats", "timings", "total_seconds"}."""
    from .reconstruct import reconstruct_frame
    rig, solver, prior, median_radius, dyn = _setup(calib_path, config, ref_index, dynamic_only)
    frame = _load(rig, frames_dir, priors_dir)
    os.makedirs(out_dir, exist_ok=True)
    stage = {}
    try:
        rec, _ = reconstruct_frame(frame, rig, solver, prior, dynamic_only=dyn,
                                   median_radius=median_radius, timings=stage)
    except ValueError as exc:  # e.g. a degenerate support set (prior.py:330-349)
        raise PipelineError(str(exc))
    t0 = time.perf_counter()
    _write_files(out_dir, artefact_files(rec, frame.num_views, solver, prior, median_radius, dyn))
    timings = [("support", stage["support"]), ("triangulate", stage["triangulate"]),
               ("solve_refocus", stage["solve_refocus"]), ("write", time.perf_counter() - t0)]
    _write_timings(out_dir, timings, threads)
    return {"out_dir": out_dir, "stats": rec.stats, "timings": dict(timings),
            "total_seconds": sum(s for _, s in timings)}


def run_reconstruct_sequence(calib_path, frame_dirs, out_dirs, priors_dirs=None, config=None,
                             ref_index=None, dynamic_only=None, threads=None, workers=None):
    """run_reconstruct over a sequence of frame directories, streamed: frames
    are read ahead on a thread pool, reconstructed by `reconstruct_frames`
    (device harvest, Qhull process pool, pipelined device solve) and their
    artefacts written on the same pool.  Every directory's artefacts equal
    those of run_reconstruct on it alone.  Returns the per-frame EMStats."""
    from .reconstruct import reconstruct_frames
    frame_dirs, out_dirs = list(frame_dirs), list(out_dirs)
    if len(frame_dirs) != len(out_dirs):
        raise PipelineError("frame_dirs and out_dirs differ in length")
    priors_dirs = list(priors_dirs) if priors_dirs is not None else [None] * len(frame_dirs)
    rig, solver, prior, median_radius, dyn = _setup(calib_path, config, ref_index, dynamic_only)
    io = ThreadPoolExecutor(max_workers=max(2, min(8, os.cpu_count() or 2)))
    try:
        reads = [io.submit(_load, rig, f, p) for f, p in zip(frame_dirs, priors_dirs)]
        frames = (r.result() for r in reads)
        writes, stats = [], []
        t_start = time.perf_counter()
        for out_dir, rec in zip(out_dirs, reconstruct_frames(
                frames, rig, solver, prior, dynamic_only=dyn, median_radius=median_radius,
                workers=workers)):
            writes.append(io.submit(_encode_and_write, out_dir, rec, len(rig), solver, prior,
                                    median_radius, dyn))
            stats.append(rec.stats)
        for w in writes:
            w.result()
        total = time.perf_counter() - t_start
        for out_dir in out_dirs:
            _write_timings(out_dir, [("sequence_total", total)], threads)
    except ValueError as exc:
        if isinstance(exc, PipelineError):
            raise
        raise PipelineError(str(exc))
    finally:
        io.shutdown(wait=True)
    return stats


# -- synthetic frame directories and evaluation ---------------------

def _presets():
    from . import synth
    return {"two_plane": synth.two_plane_scene, "occluder": synth.occluder_scene,
            "low_texture": synth.low_texture_scene}


def run_synth(out_dir, scene=None, preset=None, seed=None):
    """pipeline.py:320-358: render a scene file or preset (the renderer port,
    bit-exact with synth.py:244-309) into a frame directory with ground truth:
    calib.txt, scene.txt, view_XX.ppm, prior_XX.pgm, gt_mask_XX.pgm,
    gt_disparity.pgm, disparity_scale.txt, gt_background.ppm."""
    from dataclasses import replace

    from . import synth
    if (scene is None) == (preset is None):
        raise PipelineError("give exactly one of scene or preset")
    if scene is not None:
        try:
            spec = synth.load_scene(scene)
        except (ValueError, OSError) as exc:
            raise PipelineError(str(exc))
    else:
        presets = _presets()
        if preset not in presets:
            raise PipelineError(f"unknown preset {preset!r}; choose from {sorted(presets)}")
        spec = presets[preset]()
    if seed is not None:
        spec = replace(spec, seed=int(seed))
    try:
        spec.validate()
    except ValueError as exc:
        raise PipelineError(str(exc))
    frame, gt = synth.render(spec)
    rig = spec.rig()
    write_frame_dir(out_dir, frame, rig)
    synth.save_scene(spec, os.path.join(out_dir, "scene.txt"))
    for k in range(frame.num_views):
        pnm.write_pgm(os.path.join(out_dir, view_name("gt_mask", k, "pgm")),
                      np.asarray(gt.masks[k]).astype(np.uint8) * 255)
    code = np.clip(np.rint(gt.disparity * DISPARITY_SCALE), 0, 65535).astype(np.uint16)
    pnm.write_pgm(os.path.join(out_dir, "gt_disparity.pgm"), code)
    with open(os.path.join(out_dir, "disparity_scale.txt"), "w") as fh:
        fh.write(f"{int(DISPARITY_SCALE)}\n")
    pnm.write_ppm(os.path.join(out_dir, "gt_background.ppm"), gt.background)
    return {"out_dir": out_dir, "num_views": frame.num_views}


def _keyvals(path):
    out = {}
    with open(path, "r") as fh:
        for raw in fh:
            text = raw.split("#", 1)[0].strip()
            if text and "=" in text:
                key, _, value = text.partition("=")
                out[key.strip()] = value.strip()
    return out


def run_evaluate(run_dir, gt_dir, out_path=None):
    """pipeline.py:361-458: score a run directory against rendered ground
    truth and write report.txt (key = value).  Disparity metrics over
    status-valid pixels; refocus RMSE over refocused pixels; per-ray
    segmentation accuracy of the thresholded input priors (before) and the
    solved masks (after) against the ground-truth occluder masks, at rays
    cast with the true disparity (the prior samples through the device
    bilinear, st_bilinear)."""
    from .refocus import PROV_COPIED, PROV_FALLBACK, PROV_REFOCUSED
    from .sampling import bilinear, flatten_channels

    def need(path):
        if not os.path.exists(path):
            raise PipelineError(f"missing artifact: {path}")
        return path

    try:
        rig = load_calibration(need(os.path.join(gt_dir, "calib.txt")))
    except CalibrationError as exc:
        raise PipelineError(f"calibration: {exc}")
    gt_disp = pnm.read_pnm(need(os.path.join(gt_dir, "gt_disparity.pgm"))).astype(
        np.float64) / DISPARITY_SCALE
    gt_bg = pnm.read_pnm(need(os.path.join(gt_dir, "gt_background.ppm")))
    est = pnm.read_pnm(need(os.path.join(run_dir, "disparity.pgm"))).astype(
        np.float64) / DISPARITY_SCALE
    status = pnm.read_pnm(need(os.path.join(run_dir, "status.pgm")))
    refocused = pnm.read_pnm(need(os.path.join(run_dir, "refocused.ppm")))
    prov = pnm.read_pnm(need(os.path.join(run_dir, "provenance.pgm")))
    config = _keyvals(need(os.path.join(run_dir, "config_used.txt")))
    stats = _keyvals(need(os.path.join(run_dir, "em_stats.txt")))
    threshold = float(config.get("threshold", SolverParams().threshold))
    h, w = gt_disp.shape
    if est.shape != (h, w) or refocused.shape[:2] != (h, w):
        raise PipelineError("run and ground truth dimensions do not match")

    nan = float("nan")
    rep = {}
    ok = status == STATUS_VALID
    err = np.abs(est - gt_disp)[ok]
    rep["disparity_mae"] = float(err.mean()) if err.size else nan
    rep["disparity_rmse"] = float(np.sqrt((err ** 2).mean())) if err.size else nan
    rep["disparity_bad1"] = float((err > 1.0).mean()) if err.size else nan
    rep["disparity_invalid_frac"] = float(1.0 - ok.mean())
    sel = prov == PROV_REFOCUSED
    diff = (refocused.astype(np.float64) - gt_bg.astype(np.float64))[sel]
    rep["refocus_rmse"] = float(np.sqrt((diff ** 2).mean()) / 255.0) if diff.size else nan
    npx = float(h * w)
    rep["refocus_refocused_frac"] = float(sel.sum() / npx)
    rep["refocus_fallback_frac"] = float((prov == PROV_FALLBACK).sum() / npx)
    rep["refocus_copied_frac"] = float((prov == PROV_COPIED).sum() / npx)

    hits_before = hits_after = rays = 0
    uu, vv = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    u, v, d = uu.ravel(), vv.ravel(), gt_disp.ravel()
    for k in range(len(rig)):
        seg = pnm.read_pnm(need(os.path.join(run_dir, view_name("seg", k, "pgm"))))
        val = pnm.read_pnm(need(os.path.join(run_dir, view_name("valid", k, "pgm"))))
        pri = pnm.read_pnm(need(os.path.join(gt_dir, view_name("prior", k, "pgm"))))
        mask = pnm.read_pnm(need(os.path.join(gt_dir, view_name("gt_mask", k, "pgm"))))
        pu, pv, front = rig.warp(u, v, d, k)
        kh, kw = mask.shape
        keep = front & (pu >= 0.0) & (pu <= kw - 1.0) & (pv >= 0.0) & (pv <= kh - 1.0)
        keep &= val.ravel() > 0  # rays the solver classified
        idx = np.flatnonzero(keep)
        iu = np.clip(np.rint(pu[idx]), 0, kw - 1).astype(np.int64)
        iv = np.clip(np.rint(pv[idx]), 0, kh - 1).astype(np.int64)
        truth = mask[iv, iu] == 0
        flat, ph, pw = flatten_channels(pri.astype(np.float32) / 255.0)
        q = bilinear(flat, ph, pw, pu[idx], pv[idx])[:, 0]
        hits_before += int(((q >= threshold) == truth).sum())
        hits_after += int(((seg.ravel()[idx] > 0) == truth).sum())
        rays += idx.size
    rep["seg_accuracy_before"] = hits_before / rays if rays else nan
    rep["seg_accuracy_after"] = hits_after / rays if rays else nan
    rep["iterations_run"] = int(stats.get("iterations_run", "0"))
    conv = stats.get("converged_after", "none")
    rep["converged_after"] = -1 if conv == "none" else int(conv)
    text = "".join(f"{k} = {v:.6f}\n" if isinstance(v, float) else f"{k} = {v}\n"
                   for k, v in rep.items())
    with open(out_path or os.path.join(run_dir, "report.txt"), "w") as fh:
        fh.write(text)
    return rep
