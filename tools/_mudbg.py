import sys, torch, numpy as np
sys.path.insert(0,'.')
import bench
from paper_2003_11076_b200 import _native as N
from paper_2003_11076_b200.prior import TriDevice
from paper_2003_11076_b200.sharding import band_extents
frame, rig, tri, _ = bench.load_inputs("C4")
sp, pp = bench.params_for("C4")
h, w = frame.shape
td = TriDevice(tri)
ws = torch.empty(int(N.lib().st_mu_raster_workspace(w, h, td.n_tri)), dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
# locate the MuWs cnt array: offset 0 of the layout (cnt is off[0])
for world in (2, 8):
    for rank in range(world):
        e0, e1 = band_extents(h, world, rank, 1, True)["solve"]
        mu = torch.empty(h * w, dtype=torch.float64, device="cuda")
        N.invoke("st_mu_raster_rows", td.st, w, h, float(pp.d_max), mu, ws, ws.numel(), e0, e1, flag)
        f = int(flag.item())
        if f:
            cnt = ws[:h*w*4].view(torch.int32).cpu().numpy().reshape(h, w)
            lo = max(0, e0 - 2)
            rows = cnt[lo:e0]
            print(world, rank, e0, e1, "flagged; halo rows claim counts hist:",
                  {int(k): int(v) for k, v in zip(*np.unique(rows, return_counts=True))},
                  "band first row hist", {int(k): int(v) for k, v in zip(*np.unique(cnt[e0], return_counts=True))})
