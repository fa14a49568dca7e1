"""Record the reference's bench inputs for configs C1-C4 (build container only).

For each BASELINE.json config this renders the synthetic scene with the
REFERENCE renderer, runs the reference's upstream support harvest
(prior.py:233-260, out of scope for the GPU path) once, and stores
  - the support list (u, v, d) the reference triangulates, and
  - sha256 digests of the rendered images/priors,
in tests/golden/bench_<cfg>.npz.  On the GPU box, bench.py re-renders the
frame with paper_2003_11076_b200.synth (checked against the digests) and
re-triangulates the recorded support with scipy, so the benchmark runs on
exactly the reference's inputs without the reference being present.

    python tools/make_bench_inputs.py C1 C2 C3 C4
"""

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import seethrough as st  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# (width, height, cameras, d_max, max_iters) -- BASELINE.json configs[0..3]
CONFIGS = {
    "C1": (640, 480, 5, 32.0, 5),
    "C2": (1280, 720, 5, 64.0, 5),
    "C3": (1920, 1080, 5, 128.0, 10),
    "C4": (3840, 2160, 9, 128.0, 10),
}
SCENE = dict(coverage=0.25, seed=11, p_flip=0.1, blur_radius=2)


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main(names):
    for name in names:
        w, h, k, dmax, iters = CONFIGS[name]
        t0 = time.time()
        spec = st.occluder_scene(width=w, height=h, cameras=k, **SCENE)
        frame, gt = st.render(spec)
        t1 = time.time()
        pp = st.PriorParams(d_max=dmax)
        sup = st.collect_support(frame, spec.rig(), pp, threshold=0.7)
        t2 = time.time()
        uv = np.array([[p.u, p.v] for p in sup], dtype=np.int32)
        d = np.array([p.d for p in sup], dtype=np.float64)
        src = np.array([p.source_view for p in sup], dtype=np.int8)
        np.savez_compressed(os.path.join(OUT, f"bench_{name}.npz"), support_uv=uv, support_d=d,
                            support_src=src, image_digest=digest(frame.images),
                            prior_digest=digest(frame.priors),
                            config=np.array([w, h, k, dmax, iters]),
                            scene=str(SCENE))
        print(f"{name}: {len(sup)} support points, render {t1 - t0:.1f}s, "
              f"support {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2"])
