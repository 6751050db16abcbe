"""Where does the e2e path lose time against the device-only loop?  Times K iterations of
(a) graph replay with device keyframes, (b) run_host, (c) run_host with the H2D copies skipped
(slots pre-filled), (d) run_host without the loss read-back."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_04004_b200 import mapper as M  # noqa: E402
from paper_2507_04004_b200 import rasterizer as R  # noqa: E402
from paper_2507_04004_b200.gaussians import GaussianMap  # noqa: E402

sc = bench.make_scene(bench.DEFAULT)
g = GaussianMap.from_rows(sc.rows)
kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
eng = M.MapOptimizer(g, kfs, R.default_lrs(3.0))
eng.capture()
eng.attach_host_keyframes(kfs)
init = eng.save_state()
K = 100


def timeit(fn):
    eng.restore_state(init)
    fn(10)
    eng.restore_state(init)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    fn(K)
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / K, (time.perf_counter() - t0) * 1e3 / K


print("graph step      ms/it", timeit(lambda n: [eng.step(i % 4) for i in range(n)]))
print("run_host        ms/it", timeit(lambda n: eng.run_host([i % 4 for i in range(n)])))
up = eng.host.upload
eng.host.upload = lambda j, k: (torch.cuda.Event(), eng.host.slots[j % 3]["view"].copy_(eng.host.views[k][j % 3]))[0]
for sl in range(3):  # slots hold keyframe sl's data once
    up(sl, sl)
torch.cuda.synchronize()
print("run_host no H2D ms/it", timeit(lambda n: eng.run_host([i % 3 for i in range(n)])))
eng.host.upload = up
hl = eng._h_loss
eng._h_loss = torch.zeros(1024, dtype=torch.float64, device="cuda")
print("run_host no D2H ms/it", timeit(lambda n: eng.run_host([i % 4 for i in range(n)])))
