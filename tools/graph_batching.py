"""Gap between graph launches: 4 single-iteration graph replays (one per keyframe) against one
graph holding the same 4 iterations (programmatic launches across the iteration boundaries)."""
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
singles = [eng._graph_for(v.ptr) for v in eng.views]
torch.cuda.synchronize()
big = torch.cuda.CUDAGraph()
with torch.cuda.graph(big):
    for v in eng.views:
        eng._launch(v.ptr)
N = 50
def run(fn):
    eng.restore_state(init); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(N): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / (4 * N)
for r in range(2):
    print("4 single graphs ms/iter", run(lambda: [gr.replay() for gr in singles]), "one 4-iteration graph", run(lambda: big.replay()))
