import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
from paper_2507_04004_b200 import rasterizer as R
from paper_2507_04004_b200.gaussians import GaussianMap
z = np.load("tests/golden/small0.npz")
cam = R.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]), z["rot_cw"], z["trans_cw"])
g = GaussianMap.from_rows(z["rows"])
out = R.forward(g, cam)
grads, touched, _ = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
gr = grads["_rows"].double().cpu().numpy()[:, :59]
ref = z["grads"]
groups = {"pos": (0, 3), "log_scale": (3, 6), "quat": (6, 10), "opacity_logit": (10, 11), "sh_low": (11, 14), "sh_high": (14, 59)}
for k, (a, b) in groups.items():
    print(k, np.abs(gr[:, a:b] - ref[:, a:b]).max(), np.abs(ref[:, a:b]).max())
i = int(np.argmax(np.abs(gr[:, 0:3] - ref[:, 0:3]).max(axis=1)))
print("worst row", i, gr[i, :11], ref[i, :11])
# oracle chain with the GPU's own g2d
g2d = out.ctx["workspace"].g2d.double().cpu().numpy()[:, :10]
oc = O.chain(z["rows"], O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.rot_cw, cam.trans_cw), g2d, z["touched"])
print("oracle-chain(gpu g2d) vs gpu", np.abs(oc[:, 0:3] - gr[:, 0:3]).max(), "vs ref", np.abs(oc[:,0:3]-ref[:,0:3]).max())
print("row", oc[i, :11])
