import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2003_11076_b200 as st
from paper_2003_11076_b200.prior import TriDevice
from paper_2003_11076_b200.reconstruct import FramePipeline, _outputs_of
import test_gpu_parity as T
g = T.load("occ160_noisy")
sp, pp = T._params(st, g)
frame = T._frame(st, g)
rig, tri = T._Rig(g), T._Tri(g)
h, w = frame.shape
pipe = FramePipeline(rig, w, h, sp, pp)
pipe.load(frame.images, frame.priors)
td = TriDevice(tri)
a = _outputs_of(pipe, pipe.run(td), pipe.fetch())
pipe.load(frame.images, frame.priors)
cur = pipe.t.cuda.current_stream()
block, stats = pipe.run_native(td, out_stream=cur)
cur.synchronize()
b = _outputs_of(pipe, stats, pipe.host_views(block))
print("golden agree py", (a.disparity.values == g["full_values"]).mean(), "native", (b.disparity.values == g["full_values"]).mean())
print("py stats", a.stats.iterations_run, a.stats.mean_energy[:2], "native", b.stats.iterations_run, b.stats.mean_energy[:2])
print(a.disparity.values[50, 60:66], b.disparity.values[50, 60:66])
print("mu equal", np.array_equal(a.disparity.values, b.disparity.values))
import ctypes as C
P = pipe._plan
print("plan W H K", P.rig.width, P.rig.height, P.rig.num_views, "d_max", P.params.d_max, "msr", P.params.min_static_rays, "mr", P.median_radius)
