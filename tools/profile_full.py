"""Stage times of the frame-in path (harvest -> dedup -> triangulate -> solve)
on the GPU box:  python tools/profile_full.py [C2]"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_11076_b200 as st  # noqa: E402
from paper_2003_11076_b200.prior import TriDevice, deduplicate_arrays, triangulate_arrays  # noqa: E402
from paper_2003_11076_b200.reconstruct import _pipeline_for, reconstruct_frame  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    frame, rig, tri_ref, exact = bench.load_inputs(cfg)
    sp, pp = bench.params_for(cfg)
    h, w = frame.shape
    pipe = _pipeline_for(rig, w, h, sp, pp)
    pipe.load(frame.images, frame.priors)
    for _ in range(3):
        pipe.harvest()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pipe.harvest()
    e1.record()
    e1.synchronize()
    print(f"{cfg}: descriptors+harvest (device) {e0.elapsed_time(e1) / 10:.3f} ms")
    u, v, d, s, n = pipe.harvest()
    cnt = int(n.item())
    t0 = time.perf_counter()
    hu, hv, hd, hs = (x[:cnt].cpu().numpy() for x in (u, v, d, s))
    t1 = time.perf_counter()
    keep = deduplicate_arrays(hu, hv, hd, hs, rig.ref_index, w, h)
    t2 = time.perf_counter()
    tri = triangulate_arrays(hu[keep], hv[keep], hd[keep], w, h)
    t3 = time.perf_counter()
    td = TriDevice(tri)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"collected {cnt}, kept {len(keep)}; D2H {1e3 * (t1 - t0):.2f} ms, dedup "
          f"{1e3 * (t2 - t1):.2f} ms, triangulate {1e3 * (t3 - t2):.2f} ms "
          f"({tri.triangles.shape[0]} triangles), TriDevice {1e3 * (t4 - t3):.2f} ms")
    same = (np.array_equal(tri.points, tri_ref.points)
            and np.array_equal(tri.triangles, tri_ref.triangles))
    print("support/triangulation identical to the reference harvest:", same)
    for _ in range(2):
        reconstruct_frame(frame, rig, sp, pp)
    tm = {}
    t0 = time.perf_counter()
    n_rep = 5
    for _ in range(n_rep):
        rec, _ = reconstruct_frame(frame, rig, sp, pp, timings=tm)
    dt = (time.perf_counter() - t0) / n_rep
    print(f"reconstruct_frame: {1e3 * dt:.2f} ms/frame ({1 / dt:.1f} fps); last stages "
          + ", ".join(f"{k} {1e3 * x:.2f} ms" for k, x in tm.items()))
    ref = st.reconstruct(frame, rig, tri_ref, sp, pp)
    print("outputs identical to the golden-support path:",
          np.array_equal(rec.disparity.values, ref.disparity.values)
          and np.array_equal(rec.image, ref.image))


if __name__ == "__main__":
    main()
