import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2507_04004_b200 import rasterizer as R
from paper_2507_04004_b200.gaussians import GaussianMap
z = np.load("tests/golden/room4096.npz")
cam = R.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]), z["rot_cw"], z["trans_cw"])
g = GaussianMap.from_rows(z["rows"])
out = R.forward(g, cam)
g2d_gpu = [t.double().cpu().numpy() for t in R.backward_2d(out, z["g_color"], z["g_depth"], z["g_opac"])[:5]]
names = ["mean2d", "conic", "op", "color", "depth"]
for nm, a in zip(names, g2d_gpu):
    ref = z["g2d_" + nm]
    err = np.abs(a - ref).reshape(len(ref), -1).max(axis=1)
    i = int(np.argmax(err))
    print(nm, "normwise", err.max() / np.abs(ref).max(), "worst row", i, "depth", z["pdepth"][i], a.reshape(len(ref), -1)[i], ref.reshape(len(ref), -1)[i])
grads, touched, _ = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
gr = grads["_rows"].double().cpu().numpy()[:, :59]
ref = z["grads"]
e = np.abs(gr[:, :3] - ref[:, :3]).max(axis=1); i = int(np.argmax(e))
print("pos worst", i, "depth", z["pdepth"][i], gr[i, :3], ref[i, :3], "max|ref|", np.abs(ref[:, :3]).max())
print("top pos rows by |ref|:", np.argsort(-np.abs(ref[:, :3]).max(axis=1))[:5], "depths", z["pdepth"][np.argsort(-np.abs(ref[:, :3]).max(axis=1))[:5]])
