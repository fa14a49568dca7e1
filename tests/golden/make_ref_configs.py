"""Reference outputs at BASELINE.json's bench configs (build container only).

Runs the REFERENCE (`/root/reference/pkg/src`, imported, not copied) on the
exact bench inputs of C1/C2/C3 -- the reference renderer's frame and the
support list the reference harvested for it (tests/golden/bench_<cfg>.npz,
tools/make_bench_inputs.py) -- and records what the GPU path must match:

  * `ref_<cfg>.npz`: em_solve + synthesize outputs (values, status,
    static/valid bits, image, provenance, n_rays), EMStats, and the
    FINAL-iteration decision margins: the M-step margin at
    the masks the last M-step saw (best minus second-best energy over
    candidates with |d - d_best| > 1e-9) and the E-step margin at the last
    M-step's disparity (top-1 minus top-2 mask score).  Pixels whose margin
    is <= 1e-5 are listed; everywhere else the GPU must be exact.
  * `forced_<name>.npz`: the forced-iteration bench mode (SURVEY.md §8c,
    "compose the reference's own methods without the early break":
    initial_masks, then m_step / e_step_at I times, solver.py:455-482).
  * `c4rows.npz`: C4 (3840x2160, K=9, d_max 128) iteration-1 M-step and
    E-step on 16 strided rows, with their margins.

The margins are computed with the oracle (oracle/em.py m_margins/e_margins,
itself pinned bit-exact to the reference by tests/test_oracle.py); the
outputs and statistics come from the reference.

  * `ref_<cfg>_dynamic.npz`: the same for dynamic_only (the person-only mode).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_ref_configs.py C1 C2 C3 forced C4rows \
        C1dynamic C2dynamic
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("SEETHROUGH_REF", "/root/reference/pkg/src"))
import seethrough as st  # noqa: E402

import oracle  # noqa: E402

CONFIGS = {"C1": (640, 480, 5, 32.0, 5), "C2": (1280, 720, 5, 64.0, 5),
           "C3": (1920, 1080, 5, 128.0, 10), "C4": (3840, 2160, 9, 128.0, 10)}
SCENE = dict(coverage=0.25, seed=11, p_flip=0.1, blur_radius=2)
MARGIN = 1e-5
CHUNK = 1 << 16


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def bench_inputs(cfg):
    w, h, k, dmax, iters = CONFIGS[cfg]
    spec = st.occluder_scene(width=w, height=h, cameras=k, **SCENE)
    frame, _ = st.render(spec)
    rig = spec.rig()
    z = np.load(os.path.join(HERE, f"bench_{cfg}.npz"))
    assert digest(frame.images) == str(z["image_digest"])
    assert digest(frame.priors) == str(z["prior_digest"])
    pts = [st.SupportPoint(int(u), int(v), float(d), int(s))
           for (u, v), d, s in zip(z["support_uv"], z["support_d"], z["support_src"])]
    tri = st.triangulate(pts, w, h)
    sp = st.SolverParams(max_iters=iters)
    pp = st.PriorParams(d_max=dmax)
    return frame, rig, tri, sp, pp


def oracle_of(frame, rig, tri, sp, pp, solver):
    k = len(rig)
    a = np.stack([rig.warp_coefficients(i)[0] for i in range(k)])
    b = np.stack([rig.warp_coefficients(i)[1] for i in range(k)])
    uv, d = tri.support_points()
    p = oracle.OracleParams(beta=sp.beta, threshold=sp.threshold, max_iters=sp.max_iters,
                            min_static_rays=sp.min_static_rays, epsilon_prior=sp.epsilon_prior,
                            sigma=pp.sigma, gamma=pp.gamma, d_max=pp.d_max,
                            neighborhood_radius=pp.neighborhood_radius)
    # the reference solver's own (raw) surface: OracleSolver clips it like solver.py:185-186
    mu_raw = tri.disparity_map(frame.shape[1], frame.shape[0])
    return oracle.OracleSolver(list(frame.images), list(frame.priors), a, b, rig.ref_index,
                               mu_raw, uv, d, params=p)


def traced_solve(solver, forced=None):
    """solver.py:436-485 composed from the reference's own methods, keeping
    the state the final iteration saw (forced: no early break)."""
    h, w = solver.height, solver.width
    allp = np.arange(h * w, dtype=np.int64)
    static, valid = solver.initial_masks(allp)
    d_prev = None
    last = None
    iters = forced if forced else solver.params.max_iters
    stats = dict(iterations_run=0, converged_after=None, mean_energy=[], prev_energy=[],
                 changed_fraction=[])
    for it in range(1, iters + 1):
        stats["iterations_run"] = it
        before = static
        d, e, status = solver.m_step(allp, static)
        fin = e[np.isfinite(e)]
        stats["mean_energy"].append(float(fin.mean()))
        changed = None
        if d_prev is not None:
            pe, _ = solver._energy(allp, d_prev, static)
            pf = pe[np.isfinite(pe)]
            stats["prev_energy"].append(float(pf.mean()))
            with np.errstate(invalid="ignore"):
                changed = float(np.mean(np.abs(d - d_prev) > 0.5))
            stats["changed_fraction"].append(changed)
        ok = status != st.STATUS_LOW_TEXTURE
        s_new, v_new = solver.e_step_at(allp[ok], d[ok])
        static = static.copy()
        valid = valid.copy()
        static[allp[ok]] = s_new
        valid[allp[ok]] = v_new
        last = (before, d, status)
        if not forced and changed is not None and changed < 1e-3:
            stats["converged_after"] = it - 1
            break
        d_prev = d
    before, d, status = last
    values = d.astype(np.float32)
    values[~np.isfinite(d)] = 0.0
    return dict(values=values.reshape(h, w), status=status.reshape(h, w),
                static_bits=static.reshape(h, w), valid_bits=valid.reshape(h, w),
                stats=stats, last_masks=before, last_d=d)


def traced_dynamic(solver):
    """solver.py:436-502 with dynamic_only=True (active = ref prior < threshold),
    keeping the final iteration's masks and disparities (full-frame arrays,
    NaN / LOW_TEXTURE outside the active set)."""
    h, w = solver.height, solver.width
    allp = np.arange(h * w, dtype=np.int64)
    ref_prior = solver.frame.priors[solver.rig.ref_index].ravel()
    active = allp[ref_prior < solver.params.threshold]
    static, valid = solver.initial_masks(allp)
    d_prev = None
    last = None
    for it in range(1, solver.params.max_iters + 1):
        before = static
        d, e, status = solver.m_step(active, static)
        changed = None
        if d_prev is not None:
            with np.errstate(invalid="ignore"):
                changed = float(np.mean(np.abs(d - d_prev) > 0.5))
        ok = status != st.STATUS_LOW_TEXTURE
        s_new, v_new = solver.e_step_at(active[ok], d[ok])
        static = static.copy()
        static[active[ok]] = s_new
        last = (before, d, status)
        if changed is not None and changed < 1e-3:
            break
        d_prev = d
    before, d, status = last
    d_full = np.full(h * w, np.nan)
    d_full[active] = d
    st_full = np.full(h * w, st.STATUS_LOW_TEXTURE, dtype=np.uint8)
    st_full[active] = status
    return before, d_full, st_full, active


def make_dynamic(cfg):
    """dynamic_only (PAPER.md:242 person-only mode; solver.py:449-452,
    pipeline.py:250-260) at a bench config: the reference's solve + refocus
    with the copy mask, and the final-iteration margins on the active set."""
    frame, rig, tri, sp, pp = bench_inputs(cfg)
    t1 = time.time()
    dmap, seg, stats = st.em_solve(frame, rig, tri, params=sp, prior_params=pp,
                                   dynamic_only=True)
    copy_mask = frame.priors[rig.ref_index] >= sp.threshold
    img, prov, nr = st.synthesize(frame, rig, dmap, seg, min_static_rays=sp.min_static_rays,
                                  median_radius=1, copy_mask=copy_mask)
    t2 = time.time()
    solver = st.DisparitySolver(frame, rig, tri, params=sp, prior_params=pp)
    masks, d, status, active = traced_dynamic(solver)
    orc = oracle_of(frame, rig, tri, sp, pp, solver)
    n = masks.size
    m = np.full(n, np.inf)
    e = np.full(n, np.inf)
    for lo in range(0, active.size, CHUNK):
        act = active[lo:lo + CHUNK]
        db, eb, mm = orc.m_margins(act, masks)
        m[act] = mm
        ok = status[act] != st.STATUS_LOW_TEXTURE
        if ok.any():
            e[act[ok]] = orc.e_margins(act[ok], d[act[ok]])
    summ = margin_summary(m, e)
    print(f"{cfg} dynamic_only: solve+refocus {t2 - t1:.1f}s, active {active.size}, "
          f"iterations {stats.iterations_run}, {summ}", flush=True)
    np.savez_compressed(
        os.path.join(HERE, f"ref_{cfg}_dynamic.npz"),
        values=dmap.values, status=dmap.status, static_bits=seg.static_bits,
        valid_bits=seg.valid_bits, image=img, provenance=prov, n_rays=nr,
        stats=json.dumps(dict(iterations_run=stats.iterations_run,
                              converged_after=stats.converged_after,
                              mean_energy=stats.mean_energy, prev_energy=stats.prev_energy,
                              changed_fraction=stats.changed_fraction)),
        m_low=np.flatnonzero(~(m > MARGIN)).astype(np.int64),
        e_low=np.flatnonzero(~(e > MARGIN)).astype(np.int64),
        margins=json.dumps(summ),
        inputs=json.dumps(dict(config=cfg, scene=SCENE, dynamic_only=True,
                               image_digest=digest(frame.images))))


def margins(orc, masks, d, status):
    """Final-iteration M and E margins for every pixel (chunked)."""
    n = masks.size
    m_marg = np.empty(n)
    e_marg = np.full(n, np.inf)
    for lo in range(0, n, CHUNK):
        act = np.arange(lo, min(lo + CHUNK, n), dtype=np.int64)
        db, eb, mm = orc.m_margins(act, masks)
        assert np.array_equal(db.astype(np.float32)[np.isfinite(db)],
                              d[act].astype(np.float32)[np.isfinite(db)])
        m_marg[act] = mm
        ok = status[act] != st.STATUS_LOW_TEXTURE
        if ok.any():
            e_marg[act[ok]] = orc.e_margins(act[ok], d[act[ok]])
    return m_marg, e_marg


def margin_summary(m, e):
    return {f"{tag}_lt_{t:g}": int((x < t).sum()) for tag, x in (("m", m), ("e", e))
            for t in (1e-5, 1e-4, 1e-3)}


def make_config(cfg):
    t0 = time.time()
    frame, rig, tri, sp, pp = bench_inputs(cfg)
    h, w = frame.shape
    t1 = time.time()
    dmap, seg, stats = st.em_solve(frame, rig, tri, params=sp, prior_params=pp)
    img, prov, nr = st.synthesize(frame, rig, dmap, seg, min_static_rays=sp.min_static_rays,
                                  median_radius=1)
    t2 = time.time()
    solver = st.DisparitySolver(frame, rig, tri, params=sp, prior_params=pp)
    tr = traced_solve(solver)
    for key, ref in (("values", dmap.values), ("status", dmap.status),
                     ("static_bits", seg.static_bits), ("valid_bits", seg.valid_bits)):
        assert np.array_equal(tr[key], ref), key
    t3 = time.time()
    orc = oracle_of(frame, rig, tri, sp, pp, solver)
    m, e = margins(orc, tr["last_masks"], tr["last_d"], tr["status"].ravel())
    t4 = time.time()
    summ = margin_summary(m, e)
    print(f"{cfg}: solve+refocus {t2 - t1:.1f}s, trace {t3 - t2:.1f}s, margins {t4 - t3:.1f}s, "
          f"iterations {stats.iterations_run}, {summ}", flush=True)
    np.savez_compressed(
        os.path.join(HERE, f"ref_{cfg}.npz"),
        values=dmap.values, status=dmap.status, static_bits=seg.static_bits,
        valid_bits=seg.valid_bits, image=img, provenance=prov, n_rays=nr,
        stats=json.dumps(dict(iterations_run=stats.iterations_run,
                              converged_after=stats.converged_after,
                              mean_energy=stats.mean_energy, prev_energy=stats.prev_energy,
                              changed_fraction=stats.changed_fraction)),
        m_low=np.flatnonzero(~(m > MARGIN)).astype(np.int64),
        e_low=np.flatnonzero(~(e > MARGIN)).astype(np.int64),
        margins=json.dumps(summ),
        m_margin_min=np.float64(np.nanmin(m)), e_margin_min=np.float64(np.min(e)),
        inputs=json.dumps(dict(config=cfg, scene=SCENE, image_digest=digest(frame.images),
                               seconds=dict(reference_solve_refocus=t2 - t1))))


def make_forced(name):
    """Forced 5 iterations: occ320_noisy golden scene, C1 and C2."""
    iters = 5
    if name in CONFIGS:
        frame, rig, tri, sp, pp = bench_inputs(name)
    else:  # the occ320_noisy golden scene (make_golden.py main)
        sys.path.insert(0, HERE)
        from make_golden import rendered  # noqa: E402
        frame, _, rig, tri = rendered(st.occluder_scene(width=320, height=240, p_flip=0.1,
                                                        blur_radius=2))
        sp, pp = st.SolverParams(), st.PriorParams()
    solver = st.DisparitySolver(frame, rig, tri, params=sp, prior_params=pp)
    tr = traced_solve(solver, forced=iters)
    seg = st.SegmentationState(static_bits=tr["static_bits"], valid_bits=tr["valid_bits"])
    dmap = st.DisparityMap(values=tr["values"], status=tr["status"])
    img, prov, nr = st.synthesize(frame, rig, dmap, seg, min_static_rays=sp.min_static_rays,
                                  median_radius=1)
    orc = oracle_of(frame, rig, tri, sp, pp, solver)
    m, e = margins(orc, tr["last_masks"], tr["last_d"], tr["status"].ravel())
    summ = margin_summary(m, e)
    print(f"forced {name}: {summ}", flush=True)
    np.savez_compressed(
        os.path.join(HERE, f"forced_{name}.npz"),
        values=tr["values"], status=tr["status"], static_bits=tr["static_bits"],
        valid_bits=tr["valid_bits"], image=img, provenance=prov, n_rays=nr,
        stats=json.dumps(tr["stats"]), m_low=np.flatnonzero(~(m > MARGIN)),
        e_low=np.flatnonzero(~(e > MARGIN)), margins=json.dumps(summ))


def make_c4rows(n_rows=16):
    """C4 iteration 1 on strided rows: reference m_step at the initial masks,
    reference e_step_at at its winners, and the oracle's margins."""
    frame, rig, tri, sp, pp = bench_inputs("C4")
    h, w = frame.shape
    rows = np.linspace(8, h - 9, n_rows).astype(np.int64)
    pix = (rows[:, None] * w + np.arange(w)[None, :]).ravel()
    solver = st.DisparitySolver(frame, rig, tri, params=sp, prior_params=pp)
    s0, v0 = solver.initial_masks(np.arange(h * w, dtype=np.int64))
    d, e, status = solver.m_step(pix, s0)
    ok = status != st.STATUS_LOW_TEXTURE
    s1, v1 = solver.e_step_at(pix[ok], d[ok])
    orc = oracle_of(frame, rig, tri, sp, pp, solver)
    db, eb, mm = orc.m_margins(pix, s0)
    em = np.full(pix.size, np.inf)
    em[ok] = orc.e_margins(pix[ok], d[ok])
    summ = margin_summary(mm, em)
    print(f"C4 rows: {summ}", flush=True)
    np.savez_compressed(os.path.join(HERE, "c4rows.npz"), rows=rows, pix=pix,
                        init_static=s0[pix], init_valid=v0[pix], d=d, e=e, status=status,
                        e_pix=pix[ok], e_static=s1, e_valid=v1,
                        m_low=np.flatnonzero(~(mm > MARGIN)), e_low=np.flatnonzero(~(em > MARGIN)),
                        margins=json.dumps(summ))


def main(args):
    for a in args:
        if a in CONFIGS:
            make_config(a)
        elif a == "forced":
            make_forced("occ320_noisy")
            make_forced("C1")
        elif a == "C4rows":
            make_c4rows()
        elif a == "forcedC2":
            make_forced("C2")
        elif a.endswith("dynamic") and a[:2] in CONFIGS:
            make_dynamic(a[:2])
        else:
            raise SystemExit(f"unknown target {a}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "forced"])
