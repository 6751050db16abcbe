import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_04004_b200 import rasterizer as R, scenes
from paper_2507_04004_b200.gaussians import GaussianMap
sc = scenes.scene_room(1 << 20, 1280, 720, lidar=32)
g = GaussianMap.from_rows(sc.rows)
out = R.forward(g, R.camera_from(sc.cams[0]))
ws = out.ctx["workspace"]
rect = ws.view("rect", "i32", (len(g), 4)).cpu().numpy()
kept = ws.view("kept", "i32", (len(g),)).cpu().numpy()
nc = np.where(rect[:, 1] >= rect[:, 0], (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1), 0)
s2 = ws.splat2d.cpu().numpy(); cov = ws.cov2d.cpu().numpy()
act = nc > 0
print("active", act.sum(), "sum ncand", nc.sum(), "kept", kept.sum())
for lo, hi in [(1, 4), (5, 16), (17, 64), (65, 256), (257, 1024), (1025, 4000)]:
    m = (nc >= lo) & (nc <= hi)
    print(f"ncand {lo}-{hi}: splats {m.sum()} cand {nc[m].sum()} kept {kept[m].sum()}")
big = nc > 16
print("big depth pct", np.percentile(s2[big, 6], [5, 50, 95]), "radius pct", np.percentile(cov[big, 3], [5, 50, 95]))
# ellipse bbox candidates
qcut = s2[:, 7]
hx = np.sqrt(np.maximum(qcut * cov[:, 0], 0)); hy = np.sqrt(np.maximum(qcut * cov[:, 2], 0))
mx, my = s2[:, 0], s2[:, 1]
tx0 = np.clip(np.floor((mx - hx) / 16), 0, 79); tx1 = np.clip(np.floor((mx + hx) / 16), 0, 79)
ty0 = np.clip(np.floor((my - hy) / 16), 0, 44); ty1 = np.clip(np.floor((my + hy) / 16), 0, 44)
tx0 = np.maximum(tx0, rect[:, 0]); tx1 = np.minimum(tx1, rect[:, 1]); ty0 = np.maximum(ty0, rect[:, 2]); ty1 = np.minimum(ty1, rect[:, 3])
nc2 = np.where(act & (tx1 >= tx0) & (ty1 >= ty0), (tx1 - tx0 + 1) * (ty1 - ty0 + 1), 0)
print("ellipse-bbox cand", nc2.sum(), "big", (nc2 > 16).sum(), "cand of big", nc2[nc2 > 16].sum())
print("touched", (kept > 0).sum(), "E", int(out.ctx["counters"][1]))
c = out.ctx["counters"].cpu().numpy() if hasattr(out.ctx["counters"], "cpu") else out.ctx["counters"]
print("counters", [int(x) for x in c[:32]])
torch.cuda.synchronize()
print("all counters", [int(x) for x in ws.counters.cpu().numpy()])
