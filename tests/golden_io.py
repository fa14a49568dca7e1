"""Loading helpers for the reference-generated fixtures in tests/golden/."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = ("occ160", "occ160_tilt", "occ160_noisy", "two160", "low160", "occ128_k9",
          "occ320_noisy")


def load(name):
    z = np.load(os.path.join(GOLDEN, f"scene_{name}.npz"))
    out = {k: z[k] for k in z.files}
    out["params"] = json.loads(str(out["params"]))
    for tag in ("full", "dyn"):
        out[f"{tag}_stats"] = json.loads(str(out[f"{tag}_stats"]))
    return out


def support(g):
    n = g["tri_points"].shape[0] - int(g["tri_num_anchors"])
    return g["tri_points"][:n], g["tri_disp"][:n]


def oracle_solver(g):
    import oracle
    p = oracle.OracleParams(**g["params"])
    uv, d = support(g)
    return oracle.OracleSolver(list(g["images"]), list(g["priors"]), g["warp_a"], g["warp_b"],
                               int(g["ref_index"]), g["mu_raw"], uv, d, params=p)


def cases(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: z[k] for k in z.files}
