"""Diagnostic: mu raster stage times and ambiguity statistics at a config
(ST_MU_PROFILE=1 prints the per-stage CUDA-event times from st_mu_raster)."""
import os
import sys

import numpy as np

os.environ["ST_MU_PROFILE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
frame, rig, tri, exact = bench.load_inputs(cfg)
sp, pp = bench.params_for(cfg)
for _ in range(3):
    r = st.reconstruct(frame, rig, tri, sp, pp)
print("triangles", len(tri.triangles), "points", len(tri.points))
