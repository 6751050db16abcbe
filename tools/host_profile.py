import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2507_04004_b200 import mapper as M, rasterizer as R
from paper_2507_04004_b200.gaussians import GaussianMap
sc = bench.make_scene(bench.DEFAULT)
g = GaussianMap.from_rows(sc.rows)
kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
eng = M.MapOptimizer(g, kfs, R.default_lrs(3.0))
eng.capture()
eng.attach_host_keyframes(kfs)
for i in range(20): eng.step(i % 4)
eng.run_host([i % 4 for i in range(20)]); torch.cuda.synchronize()
# instrument
import collections
acc = collections.Counter()
H = eng.host
orig_upload = H.upload
def up(j, k):
    t = time.perf_counter(); r = orig_upload(j, k); acc['upload'] += time.perf_counter() - t; return r
H.upload = up
orig_check = eng._check
def ck(keep):
    t = time.perf_counter(); orig_check(keep); acc['check(sync)'] += time.perf_counter() - t
eng._check = ck
orig_run = eng._run_view
def rv(vp):
    t = time.perf_counter(); orig_run(vp); acc['replay'] += time.perf_counter() - t
eng._run_view = rv
orig_rec = eng._record
def rec(*a, **kw):
    t = time.perf_counter(); orig_rec(*a, **kw); acc['record'] += time.perf_counter() - t
eng._record = rec
N = 500
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); s.record()
eng.run_host([i % 4 for i in range(N)])
e.record(); e.synchronize(); wall = time.perf_counter() - t0
print("device ms/iter", s.elapsed_time(e) / N, "wall ms/iter", wall * 1e3 / N)
for k, v in acc.items(): print(k, "us/iter", v * 1e6 / N)
# graph-only
torch.cuda.synchronize(); s.record()
for i in range(N): eng.step(i % 4)
e.record(); e.synchronize(); print("step() device ms/iter", s.elapsed_time(e) / N)
