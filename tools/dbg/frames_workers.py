import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
import paper_2003_11076_b200 as st
from paper_2003_11076_b200.qhull_pool import make_pool


def main():
    frame, rig, tri, _ = bench.load_inputs("C2")
    sp, pp = bench.params_for("C2")
    pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
    pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
    for d, s in zip(pin_i, frame.images): d[...] = s
    for d, s in zip(pin_p, frame.priors): d[...] = s
    hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
    for nw in (int(x) for x in sys.argv[1:]):
        make_pool(nw)
        for _ in st.reconstruct_frames([hf] * 4, rig, sp, pp, workers=nw): pass
        t0 = time.perf_counter(); n = 64
        for _ in st.reconstruct_frames([hf] * n, rig, sp, pp, workers=nw): pass
        print(f"workers {nw}: {n / (time.perf_counter() - t0):.1f} fps", flush=True)


if __name__ == "__main__":
    main()
