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
s2 = ws.splat2d.cpu().numpy()
nc = np.where(rect[:, 1] >= rect[:, 0], (rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1), 0)
big = np.flatnonzero(nc > 16)
np.savez_compressed("gpurun_out/big.npz", ids=big, s2=s2[big], rect=rect[big], kept=kept[big])
print("saved", len(big))
