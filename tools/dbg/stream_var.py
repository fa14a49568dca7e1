import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
import paper_2003_11076_b200 as st
frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pin_i = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pin_p = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pin_i, frame.images): d[...] = s
for d, s in zip(pin_p, frame.priors): d[...] = s
hf = st.LightFieldFrame(images=pin_i, priors=pin_p)
for _ in st.reconstruct_stream([(hf, tri)] * 2, rig, sp, pp): pass
os.environ["ST_STREAM_PROFILE"] = "1"
for rep in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); n = 0
    for _ in st.reconstruct_stream([(hf, tri)] * 60, rig, sp, pp): n += 1
    torch.cuda.synchronize()
    print(f"rep {rep}: {(time.perf_counter() - t0) / n * 1e3:.3f} ms/frame", flush=True)
