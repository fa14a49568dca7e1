"""Frame-directory I/O and the artefact set, synthetic
frame directories and evaluation (§8(f)4).

CPU tests mirror the reference's test_pnm.py and test_pipeline.py:51-147
(PNM wire format, config parsing, frame-directory validation) and check
that the frame directories this package writes are byte-identical to the
reference's run_synth output (golden digests from
tests/golden/make_pipeline_golden.py).  The GPU tests run run_reconstruct /
run_reconstruct_sequence and require every artefact (timings.txt aside) to
be byte-identical to the reference's run_reconstruct on the same directory.
"""

import hashlib
import json
import os
import shutil
import struct

import numpy as np
import pytest

from paper_2003_11076_b200 import pipeline as pl
from paper_2003_11076_b200 import pnm
from oracle.synth import render
from paper_2003_11076_b200.synth import occluder_scene

HERE = os.path.dirname(os.path.abspath(__file__))
_GOLD = json.load(open(os.path.join(HERE, "golden", "pipeline_cases.json")))
CASES = {k: v for k, v in _GOLD.items() if not k.startswith("_")}
SYNTH = _GOLD["_synth"]


def _digest(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def _frame_dir(tmp_path, name):
    case = CASES[name]
    spec = occluder_scene(**case["scene"])
    frame, _ = render(spec)
    out = str(tmp_path / name / "frames")
    pl.write_frame_dir(out, frame, spec.rig())
    return out


# -- PNM (reference test_pnm.py) --------------------------------------------------

def test_pgm_roundtrips_and_wire_format(tmp_path):
    rng = np.random.default_rng(0)
    a8 = rng.integers(0, 256, size=(13, 7), dtype=np.uint8)
    pnm.write_pgm(tmp_path / "a.pgm", a8)
    back = pnm.read_pnm(tmp_path / "a.pgm")
    assert back.dtype == np.uint8 and np.array_equal(back, a8)
    a16 = rng.integers(0, 65536, size=(5, 9), dtype=np.uint16)
    pnm.write_pgm(tmp_path / "b.pgm", a16)
    back = pnm.read_pnm(tmp_path / "b.pgm")
    assert back.dtype == np.uint16 and np.array_equal(back, a16)
    raw = (tmp_path / "b.pgm").read_bytes()
    head = b"P5\n9 5\n65535\n"
    assert raw.startswith(head)
    assert struct.unpack(">H", raw[len(head):len(head) + 2])[0] == int(a16[0, 0])
    rgb = rng.integers(0, 256, size=(6, 4, 3), dtype=np.uint8)
    pnm.write_ppm(tmp_path / "c.ppm", rgb)
    assert np.array_equal(pnm.read_pnm(tmp_path / "c.ppm"), rgb)


def test_pnm_header_rules(tmp_path):
    img = np.arange(12, dtype=np.uint8).reshape(3, 4)
    p = tmp_path / "d.pgm"
    p.write_bytes(b"P5\n# a comment\n 4   3 \n# another\n255\n" + img.tobytes())
    assert np.array_equal(pnm.read_pnm(p), img)
    ws = np.full((2, 2), 0x0A, dtype=np.uint8)  # payload byte that looks like whitespace
    pnm.write_pgm(tmp_path / "e.pgm", ws)
    assert np.array_equal(pnm.read_pnm(tmp_path / "e.pgm"), ws)


def test_pnm_rejects_bad_inputs(tmp_path):
    with pytest.raises(ValueError):
        pnm.write_pgm(tmp_path / "x.pgm", np.zeros((2, 2), dtype=np.float32))
    with pytest.raises(ValueError):
        pnm.write_pgm(tmp_path / "x.pgm", np.zeros((2, 2, 3), dtype=np.uint8))
    with pytest.raises(ValueError):
        pnm.write_ppm(tmp_path / "x.ppm", np.zeros((2, 2), dtype=np.uint8))
    (tmp_path / "bad.pnm").write_bytes(b"P7\n2 2\n255\n" + bytes(4))
    with pytest.raises(ValueError, match="magic"):
        pnm.read_pnm(tmp_path / "bad.pnm")
    (tmp_path / "trunc.pgm").write_bytes(b"P5\n2")
    with pytest.raises(ValueError, match="truncated"):
        pnm.read_pnm(tmp_path / "trunc.pgm")


def test_pnm_bytes_equal_reference(reference, tmp_path):
    from seethrough import pnm as rpnm
    rng = np.random.default_rng(7)
    for img, enc, wr in ((rng.integers(0, 256, (9, 11), dtype=np.uint8), pnm.encode_pgm,
                          rpnm.write_pgm),
                         (rng.integers(0, 65536, (4, 3), dtype=np.uint16), pnm.encode_pgm,
                          rpnm.write_pgm),
                         (rng.integers(0, 256, (5, 6, 3), dtype=np.uint8), pnm.encode_ppm,
                          rpnm.write_ppm)):
        wr(str(tmp_path / "r"), img)
        assert enc(img) == (tmp_path / "r").read_bytes()


# -- configuration (reference test_pipeline.py:51-86) -----------------------------

def test_parse_config(tmp_path):
    p = tmp_path / "cfg.txt"
    p.write_text("# comment\nsigma = 1.5\nmax_iters=3\ndynamic_only = yes\n")
    assert pl.parse_config(str(p)) == {"sigma": 1.5, "max_iters": 3, "dynamic_only": True}


@pytest.mark.parametrize("text,needle", [
    ("sigma 1.5\n", "expected key = value"),
    ("teapots = 2\n", "unknown option"),
    ("sigma = abc\n", "bad value"),
    ("dynamic_only = maybe\n", "bad value"),
])
def test_parse_config_errors(tmp_path, text, needle):
    p = tmp_path / "cfg.txt"
    p.write_text(text)
    with pytest.raises(pl.PipelineError) as exc:
        pl.parse_config(str(p))
    assert f"{p}:1" in str(exc.value) and needle in str(exc.value)
    assert exc.value.exit_code == 2


def test_resolve_params():
    solver, prior, med, dyn = pl.resolve_params({})
    assert solver.max_iters == 5 and prior.sigma == 2.0 and med == 1 and dyn is False
    solver, prior, med, dyn = pl.resolve_params(
        {"beta": 0.001, "sigma": 3.0, "median_radius": 2, "dynamic_only": True})
    assert solver.beta == 0.001 and prior.sigma == 3.0 and med == 2 and dyn is True
    with pytest.raises(pl.PipelineError, match="unknown options"):
        pl.resolve_params({"bogus": 1})
    with pytest.raises(pl.PipelineError, match="median_radius"):
        pl.resolve_params({"median_radius": -1})


def test_config_text_equals_reference(reference):
    from seethrough import pipeline as rp
    for overrides in ({}, {"beta": 0.001, "d_max": 30.3, "median_radius": 0, "max_iters": 3}):
        ours = pl._config_text(*pl.resolve_params(overrides))
        import tempfile
        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "c.txt")
            rp._write_config(path, *rp.resolve_params(overrides))
            assert open(path).read() == ours


# -- frame directories ------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(CASES))
def test_written_frame_dir_matches_reference_digests(tmp_path, name):
    """Renderer port + calibration writer + PNM writer == the reference's
    run_synth files, byte for byte."""
    fdir = _frame_dir(tmp_path, name)
    got = {f: _digest(os.path.join(fdir, f)) for f in sorted(os.listdir(fdir))}
    assert got == CASES[name]["inputs"]


def test_frame_dir_validation(tmp_path):
    from paper_2003_11076_b200.geometry import load_calibration
    fdir = _frame_dir(tmp_path, "occ160_noisy")
    rig = load_calibration(os.path.join(fdir, "calib.txt"))
    frame = pl.load_frame_dir(rig, fdir)
    assert frame.num_views == 5 and frame.priors[0].dtype == np.float32
    with pytest.raises(pl.PipelineError, match="view 0: missing image"):
        pl.load_frame_dir(rig, str(tmp_path / "empty"))
    broken = tmp_path / "broken"
    shutil.copytree(fdir, broken)
    img = pnm.read_pnm(os.path.join(fdir, "view_01.ppm"))
    pnm.write_ppm(str(broken / "view_01.ppm"), img[:-2])
    with pytest.raises(pl.PipelineError, match=r"view 1: image is 160x118.*says 160x120"):
        pl.load_frame_dir(rig, str(broken))
    pnm.write_ppm(str(broken / "view_01.ppm"), img)
    pnm.write_ppm(str(broken / "prior_01.pgm"), img)
    with pytest.raises(pl.PipelineError, match="view 1.*not grayscale"):
        pl.load_frame_dir(rig, str(broken))
    os.remove(broken / "prior_01.pgm")
    with pytest.raises(pl.PipelineError, match="view 1: missing prior"):
        pl.load_frame_dir(rig, str(broken))


def test_frame_dir_equals_reference_loader(reference, tmp_path):
    from seethrough import pipeline as rp
    from seethrough.geometry import load_calibration as rload
    fdir = _frame_dir(tmp_path, "occ160_noisy")
    from paper_2003_11076_b200.geometry import load_calibration
    ours = pl.load_frame_dir(load_calibration(os.path.join(fdir, "calib.txt")), fdir)
    ref = rp.load_frame_dir(rload(os.path.join(fdir, "calib.txt")), fdir)
    for a, b in zip(ours.images + ours.priors, ref.images + ref.priors):
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_run_reconstruct_error_paths_before_the_device(tmp_path):
    fdir = _frame_dir(tmp_path, "occ160_noisy")
    with pytest.raises(pl.PipelineError, match="calibration"):
        pl.run_reconstruct(str(tmp_path / "none.txt"), fdir, str(tmp_path / "o"))
    bad = tmp_path / "bad.txt"
    bad.write_text("sigma = -\n")
    with pytest.raises(pl.PipelineError, match="bad value"):
        pl.run_reconstruct(os.path.join(fdir, "calib.txt"), fdir, str(tmp_path / "o"),
                           config=str(bad))


# -- artefacts on the device ------------------------------------------------------

def _check_run(run_dir, case):
    got = {f: _digest(os.path.join(run_dir, f))
           for f in sorted(os.listdir(run_dir)) if f != "timings.txt"}
    want = case["artefacts"]
    assert sorted(got) == sorted(want)
    # every artefact byte for byte except em_stats.txt: its means are summed
    # in numpy's order (st_mean.cu) but the energies' log prior uses numpy's
    # AVX-512 exp/log on the reference side (~1 ulp apart), so the numbers
    # are compared to 1e-14
    for f in want:
        if f != "em_stats.txt":
            assert got[f] == want[f], f
    text = open(os.path.join(run_dir, "em_stats.txt")).read()
    vals = dict(line.split(" = ", 1) for line in text.strip().splitlines())
    es = case["em_stats"]
    assert int(vals["iterations_run"]) == es["iterations_run"]
    conv = vals["converged_after"]
    assert (None if conv == "none" else int(conv)) == es["converged_after"]
    for key in ("mean_energy", "prev_energy", "changed_fraction"):
        v = [float(x) for x in vals[key].split(",") if x.strip()]
        tol = 0 if key == "changed_fraction" else 1e-14
        assert np.allclose(v, es[key], rtol=tol, atol=0), key


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_run_reconstruct_artefacts_equal_reference(tmp_path, name):
    from paper_2003_11076_b200.device import require_cuda
    require_cuda()
    case = CASES[name]
    fdir = _frame_dir(tmp_path, name)
    out = str(tmp_path / name / "run")
    res = pl.run_reconstruct(os.path.join(fdir, "calib.txt"), fdir, out, **case["options"])
    assert res["stats"].iterations_run == case["em_stats"]["iterations_run"]
    _check_run(out, case)
    # the thread hint changes nothing (reference test_pipeline.py:169-176)
    out8 = str(tmp_path / name / "run8")
    pl.run_reconstruct(os.path.join(fdir, "calib.txt"), fdir, out8, threads=8,
                       **case["options"])
    for f in os.listdir(out):
        if f != "timings.txt":
            assert _digest(os.path.join(out, f)) == _digest(os.path.join(out8, f)), f


@pytest.mark.gpu
def test_run_reconstruct_sequence_equals_single_runs(tmp_path):
    from paper_2003_11076_b200.device import require_cuda
    require_cuda()
    case = CASES["occ160_noisy"]
    fdir = _frame_dir(tmp_path, "occ160_noisy")
    outs = [str(tmp_path / f"seq{i}") for i in range(4)]
    stats = pl.run_reconstruct_sequence(os.path.join(fdir, "calib.txt"), [fdir] * 4, outs)
    assert len(stats) == 4
    for out in outs:
        _check_run(out, case)


# -- run_synth / run_evaluate (§8(f)4) ----------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SYNTH))
def test_run_synth_matches_reference_files(tmp_path, name):
    """Every file run_synth writes (scene.txt, calibration, views, priors,
    ground-truth masks / disparity / background; the device renderer)
    equals the reference's."""
    case = SYNTH[name]
    out = str(tmp_path / "synth")
    pl.run_synth(out, preset=case["preset"], seed=case["seed"])
    got = {f: _digest(os.path.join(out, f)) for f in sorted(os.listdir(out))}
    assert got == case["synth"]


@pytest.mark.parametrize("name", sorted(SYNTH))
def test_run_synth_writers_with_the_oracle_renderer(tmp_path, monkeypatch, name):
    """run_synth's writers on CPU: with the numpy renderer (oracle/synth.py)
    in place of the device one, every file equals the reference's."""
    from paper_2003_11076_b200 import synth
    monkeypatch.setattr(synth, "render", render)
    case = SYNTH[name]
    out = str(tmp_path / "synth")
    pl.run_synth(out, preset=case["preset"], seed=case["seed"])
    got = {f: _digest(os.path.join(out, f)) for f in sorted(os.listdir(out))}
    assert got == case["synth"]


@pytest.mark.gpu
def test_run_synth_scene_file_and_errors(tmp_path):
    from paper_2003_11076_b200 import synth
    a = str(tmp_path / "a")
    pl.run_synth(a, preset="occluder")
    b = str(tmp_path / "b")
    pl.run_synth(b, scene=os.path.join(a, "scene.txt"))
    for f in os.listdir(a):
        assert _digest(os.path.join(a, f)) == _digest(os.path.join(b, f)), f
    with pytest.raises(pl.PipelineError, match="exactly one"):
        pl.run_synth(str(tmp_path / "c"))
    with pytest.raises(pl.PipelineError, match="unknown preset"):
        pl.run_synth(str(tmp_path / "c"), preset="teapot")
    bad = tmp_path / "bad.txt"
    bad.write_text("width 64\nteapot 3\n")
    with pytest.raises(pl.PipelineError, match="unknown directive"):
        pl.run_synth(str(tmp_path / "c"), scene=str(bad))
    spec = synth.load_scene(os.path.join(a, "scene.txt"))
    assert spec.cameras == 5 and len(spec.occluders) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SYNTH))
def test_run_evaluate_report_equals_reference(tmp_path, name):
    """run_synth -> run_reconstruct -> run_evaluate: the artefacts and the
    report.txt text equal the reference pipeline's on the same preset."""
    from paper_2003_11076_b200.device import require_cuda
    require_cuda()
    case = SYNTH[name]
    sdir = str(tmp_path / "synth")
    rdir = str(tmp_path / "run")
    pl.run_synth(sdir, preset=case["preset"], seed=case["seed"])
    pl.run_reconstruct(os.path.join(sdir, "calib.txt"), sdir, rdir)
    for f, want in case["artefacts"].items():
        if f != "em_stats.txt":
            assert _digest(os.path.join(rdir, f)) == want, f
    pl.run_evaluate(rdir, sdir)
    assert open(os.path.join(rdir, "report.txt")).read() == case["report_txt"]
    with pytest.raises(pl.PipelineError, match="missing artifact"):
        pl.run_evaluate(str(tmp_path / "nothing"), sdir)
