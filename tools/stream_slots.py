"""reconstruct_stream throughput vs the number of frame slots (C2, pinned host frames)."""
import os
import subprocess
import sys

code = r"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench, paper_2003_11076_b200 as st
frame, rig, tri, _ = bench.load_inputs('C2'); sp, pp = bench.params_for('C2')
pi = [st.device.pinned_empty(x.shape, np.uint8) for x in frame.images]
pq = [st.device.pinned_empty(x.shape, np.float32) for x in frame.priors]
for d, s in zip(pi, frame.images): d[...] = s
for d, s in zip(pq, frame.priors): d[...] = s
hf = st.LightFieldFrame(images=pi, priors=pq)
res = []
for rep in range(6):
    t0 = time.perf_counter(); n = 0
    for _ in st.reconstruct_stream([(hf, tri)] * 60, rig, sp, pp): n += 1
    torch.cuda.synchronize(); res.append((time.perf_counter() - t0) / n * 1e3)
print(min(res[2:]), sorted(res[2:])[len(res[2:]) // 2])
"""
for slots in (3, 4, 5, 6, 8):
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env=dict(os.environ, ST_STREAM_SLOTS=str(slots)))
    print(slots, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
