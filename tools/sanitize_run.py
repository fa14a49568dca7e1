"""Small end-to-end workload for compute-sanitizer (one tool per GPU call):
every kernel family of the product path on golden scenes (full and
dynamic_only, K = 5 and K = 9, a tilted non-rectified rig) and one C2 frame,
plus the frame-in path (device harvest), the row-band pipeline (world 1) and
the numpy-mean kernels.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2003_11076_b200 as st  # noqa: E402
from golden_io import load  # noqa: E402
from test_gpu_parity import _Rig, _Tri, _frame, _params  # noqa: E402

quick = "--quick" in sys.argv
scenes = ("occ160_noisy", "occ160_tilt", "occ128_k9") if quick else (
    "occ160", "occ160_tilt", "occ160_noisy", "two160", "low160", "occ128_k9")
for name in scenes:
    g = load(name)
    sp, pp = _params(st, g)
    frame, rig, tri = _frame(st, g), _Rig(g), _Tri(g)
    for dyn in (False, True):
        r = st.reconstruct(frame, rig, tri, sp, pp, dynamic_only=dyn)
        d, s, stats = st.em_solve(frame, rig, tri, sp, pp, dynamic_only=dyn)
        st.synthesize(frame, rig, d, s, median_radius=2)
        assert np.array_equal(d.values, r.disparity.values), name
    print(name, "ok", flush=True)
if not quick:
    import bench
    from paper_2003_11076_b200.sharding import reconstruct_band
    f, r, t, _ = bench.load_inputs("C2")
    sp, pp = bench.params_for("C2")
    a = st.reconstruct(f, r, t, sp, pp)
    b = reconstruct_band(f, r, t, sp, pp)
    assert np.array_equal(a.image, b.image)
    rec, _ = st.reconstruct_frame(f, r, sp, pp)
    print("C2 ok", flush=True)
import torch  # noqa: E402
from paper_2003_11076_b200 import _native as N  # noqa: E402
x = torch.randn(100003, dtype=torch.float64, device="cuda")
x[17] = float("inf")
out = torch.empty(1, dtype=torch.float64, device="cuda")
ws = torch.empty(int(N.lib().st_numpy_mean_workspace(x.numel())), dtype=torch.uint8, device="cuda")
N.invoke("st_numpy_mean", x, x.numel(), out, ws, ws.numel())
torch.cuda.synchronize()
print("sanitize workload done", flush=True)
