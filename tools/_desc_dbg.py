import sys, torch, numpy as np
sys.path.insert(0, '.')
import bench
from paper_2003_11076_b200 import _native as N
from paper_2003_11076_b200.reconstruct import FramePipeline
from paper_2003_11076_b200.prior import TriDevice
frame, rig, tri, _ = bench.load_inputs("C2")
sp, pp = bench.params_for("C2")
pipe = FramePipeline(rig, 1280, 720, sp, pp)
pipe.load(frame.images, frame.priors)
torch.cuda.synchronize(); print("load ok", flush=True)
N.invoke("st_descriptors", pipe.images, 5, 720, 1280, 3, pipe.desc, None, None)
torch.cuda.synchronize(); print("descriptors ok", flush=True)
import os
os.environ["ST_DESC_NO_TMA"] = "1"
