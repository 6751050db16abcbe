"""Statistics of the large-footprint cull at the bench workload (counters + candidate-tile histogram)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_04004_b200 import mapper as M  # noqa: E402
from paper_2507_04004_b200 import rasterizer as R  # noqa: E402
from paper_2507_04004_b200.gaussians import GaussianMap  # noqa: E402

sc = bench.make_scene(bench.DEFAULT)
g = GaussianMap.from_rows(sc.rows)
kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
eng = M.MapOptimizer(g, kfs, R.default_lrs(3.0))
for k in range(4):
    eng.step(k)
    torch.cuda.synchronize()
    c = eng.ws.counters.cpu().numpy()
    names = {1: "entries", 2: "touched", 5: "big", 7: "big_bits", 16: "huge", 17: "huge_e", 18: "small_e",
             19: "huge_n", 20: "cullq1"}
    print(k, {v: int(c[i]) for i, v in names.items()})
ws = eng.ws
nb = int(ws.counters[5].item())
big = ws.view("big_list", "i32", (len(g),))[:nb].long()
rect = ws.view("rect", "i32", (len(g), 4))[big].cpu().numpy()
ncand = (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1)
nb_rows = rect[:, 3] - rect[:, 2] + 1
print("big:", nb, "ncand percentiles", np.percentile(ncand, [10, 50, 90, 99, 100]).astype(int),
      "bands percentiles", np.percentile(nb_rows, [10, 50, 90, 99, 100]).astype(int),
      "sum ncand", int(ncand.sum()), "huge(>256)", int((ncand > 256).sum()))
