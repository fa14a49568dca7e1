"""M-step screening diagnostics (run on the GPU box): exact-evaluation counts
and kernel times with and without the fp32 screen."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import bench
import paper_2003_11076_b200 as st
cfg = sys.argv[1]
frame, rig, tri, _ = bench.load_inputs(cfg)
sp, pp = bench.params_for(cfg)
for _ in range(3):
    r = st.reconstruct(frame, rig, tri, sp, pp)
pipe = st.reconstruct._pipeline_for if hasattr(st.reconstruct, "_pipeline_for") else None
s = r.stats
print(cfg, "evals/msteps", s.energy_evals / max(s.msteps, 1), "cand/msteps",
      s.candidates_total / max(s.msteps, 1), "msteps", s.msteps)
''' % ROOT


def main():
    for cfg in sys.argv[1:] or ["C2"]:
        for mode in ("", "1", "2"):
            env = dict(os.environ)
            env.pop("ST_MSTEP_EXHAUSTIVE", None)
            if mode:
                env["ST_MSTEP_EXHAUSTIVE"] = mode
            out = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env,
                                 capture_output=True, text=True)
            print(f"mode={mode or 'screen'}:", out.stdout.strip(), out.stderr.strip()[-500:])
            b = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--quick",
                                "--config", cfg], env=env, capture_output=True, text=True)
            print("   bench:", b.stdout.strip()[-400:])


if __name__ == "__main__":
    main()
