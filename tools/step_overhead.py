"""Cost of the engine's per-step host bookkeeping (counter snapshot D2H + event) between graph
replays: eng.step() vs bare graph replays of the same views (device time, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_2507_04004_b200 import mapper as M, rasterizer as R
from paper_2507_04004_b200.gaussians import GaussianMap
sc = bench.make_scene(bench.DEFAULT)
g = GaussianMap.from_rows(sc.rows)
kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
eng = M.MapOptimizer(g, kfs, R.default_lrs(3.0))
eng.capture()
init = eng.save_state()
N = 200
def run(fn):
    eng.restore_state(init); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(N): fn(i)
    e.record(); e.synchronize()
    return s.elapsed_time(e) / N
for r in range(2):
    print("step()", run(lambda i: eng.step(i % 4)), "bare replay", run(lambda i: eng._graph_for(eng.views[i % 4].ptr).replay()))
