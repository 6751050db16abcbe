import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_04004_b200 import rasterizer as R, scenes
from paper_2507_04004_b200.gaussians import GaussianMap
sc = scenes.scene_room(1 << 20, 1280, 720, lidar=32)
g = GaussianMap.from_rows(sc.rows)
out = R.forward(g, R.camera_from(sc.cams[0]))
ws = out.ctx["workspace"]
T = ws.tiles_x * ws.tiles_y
ts = ws.view("tile_scratch", "i32", (3 * (T + 1),)).cpu().numpy()
hc = ts[T + 1:2 * T + 1]; boff = ts[2 * (T + 1):]; nb = np.diff(boff)
nc = out.n_contrib.cpu().numpy()
H, W = nc.shape
tmax = np.zeros(T, int)
for ty in range(ws.tiles_y):
    for tx in range(ws.tiles_x):
        tmax[ty * ws.tiles_x + tx] = nc[ty*16:(ty+1)*16, tx*16:(tx+1)*16].max()
print("nb per tile: mean %.1f median %d p99 %d max %d" % (nb.mean(), np.median(nb), np.percentile(nb, 99), nb.max()))
print("huge per tile: mean %.1f max %d" % (hc.mean(), hc.max()))
print("max n_contrib per tile: mean %.1f p50 %d p99 %d max %d" % (tmax.mean(), np.median(tmax), np.percentile(tmax, 99), tmax.max()))
print("tiles whose blend reaches the bucket (max n_contrib > huge count):", int((tmax > hc).sum()), "of", T)
print("n_contrib mean", nc.mean())
