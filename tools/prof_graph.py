"""Replay the bench's CUDA-graph iteration a few times (for warm-cache ncu launch lists:
ncu --cache-control none profiles each graph kernel node in its real context)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_04004_b200 import mapper as M  # noqa: E402
from paper_2507_04004_b200 import rasterizer as R  # noqa: E402
from paper_2507_04004_b200.gaussians import GaussianMap  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sc = bench.make_scene(name)
g = GaussianMap.from_rows(sc.rows)
kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
eng = M.MapOptimizer(g, kfs, R.default_lrs(3.0))
eng.capture()
for i in range(4):
    eng.step(i % len(kfs))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(iters):
    eng.step(i % len(kfs))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", eng.counters())
