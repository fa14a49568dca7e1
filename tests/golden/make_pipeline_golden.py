"""Generate tests/golden/pipeline_cases.json by running the REFERENCE pipeline.

Run in the build container only (the reference is not on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_pipeline_golden.py

For each case it renders a seeded scene with the reference renderer, writes
the frame directory exactly as the reference's run_synth does
(pipeline.py:338-345: calib.txt, view_XX.ppm, 8-bit prior_XX.pgm), runs the
reference's run_reconstruct (pipeline.py:233-287) with the case's options,
and records the sha256 of every input file and every artefact except
timings.txt, plus the em_stats values.  Nothing here is product code.
"""

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF_SRC = os.environ.get("SEETHROUGH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
import seethrough as st  # noqa: E402
from seethrough import pipeline as rp  # noqa: E402
from seethrough import pnm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# (name, scene kwargs, run_reconstruct options)
CASES = [
    ("occ160_noisy", dict(width=160, height=120, cameras=5, coverage=0.25, seed=11, p_flip=0.1,
                          blur_radius=2), {}),
    ("occ160_noisy_dyn", dict(width=160, height=120, cameras=5, coverage=0.25, seed=11,
                              p_flip=0.1, blur_radius=2), {"dynamic_only": True}),
    ("occ160_nomedian", dict(width=160, height=120, cameras=4, coverage=0.3, seed=5,
                             p_flip=0.0, blur_radius=0), {"config": {"median_radius": 0,
                                                                      "max_iters": 3}}),
]


def digest(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def write_frame_dir(out, frame, rig):
    rp.save_calibration(rig, os.path.join(out, "calib.txt"))
    for k in range(frame.num_views):
        pnm.write_ppm(os.path.join(out, rp._view_name("view", k, "ppm")), frame.images[k])
        coded = np.clip(np.rint(frame.priors[k] * 255.0), 0, 255).astype(np.uint8)
        pnm.write_pgm(os.path.join(out, rp._view_name("prior", k, "pgm")), coded)


def main():
    out = {}
    with tempfile.TemporaryDirectory() as tmp:  # noqa: SIM117
        for name, scene, opts in CASES:
            spec = st.occluder_scene(**scene)
            frame, _ = st.render(spec)
            rig = spec.rig()
            fdir = os.path.join(tmp, name, "frames")
            rdir = os.path.join(tmp, name, "run")
            os.makedirs(fdir)
            write_frame_dir(fdir, frame, rig)
            opts = dict(opts)
            res = rp.run_reconstruct(os.path.join(fdir, "calib.txt"), fdir, rdir, **opts)
            stats = res["stats"]
            out[name] = {
                "scene": scene, "options": opts,
                "inputs": {f: digest(os.path.join(fdir, f)) for f in sorted(os.listdir(fdir))},
                "artefacts": {f: digest(os.path.join(rdir, f))
                              for f in sorted(os.listdir(rdir)) if f != "timings.txt"},
                "em_stats": {"iterations_run": stats.iterations_run,
                             "converged_after": stats.converged_after,
                             "mean_energy": list(stats.mean_energy),
                             "prev_energy": list(stats.prev_energy),
                             "changed_fraction": list(stats.changed_fraction)},
            }
            print(name, "artefacts", len(out[name]["artefacts"]), "iterations",
                  stats.iterations_run)
        # run_synth presets (pipeline.py:320-358) -> run_reconstruct -> run_evaluate
        # (pipeline.py:361-458): every synth file, the artefacts and report.txt
        synth_cases = {}
        for preset, seed in (("occluder", None), ("two_plane", 7), ("low_texture", None)):
            name = f"synth_{preset}"
            sdir = os.path.join(tmp, name, "synth")
            rdir = os.path.join(tmp, name, "run")
            rp.run_synth(sdir, preset=preset, seed=seed)
            rp.run_reconstruct(os.path.join(sdir, "calib.txt"), sdir, rdir)
            rep = rp.run_evaluate(rdir, sdir)
            synth_cases[name] = {
                "preset": preset, "seed": seed,
                "synth": {f: digest(os.path.join(sdir, f)) for f in sorted(os.listdir(sdir))},
                "artefacts": {f: digest(os.path.join(rdir, f))
                              for f in sorted(os.listdir(rdir))
                              if f not in ("timings.txt", "report.txt")},
                "report_txt": open(os.path.join(rdir, "report.txt")).read(),
                "report": {k: (None if isinstance(v, float) and v != v else v)
                           for k, v in rep.items()},
            }
            print(name, rep)
        out["_synth"] = synth_cases
    with open(os.path.join(HERE, "pipeline_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
