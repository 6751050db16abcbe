"""Diagnostic: what share of the backward's (tile, entry) work belongs to near-camera Gaussians
in the benchmark scene (S2r-1M-1280x720)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04004_b200 import rasterizer as R, scenes
from paper_2507_04004_b200.gaussians import GaussianMap

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
sc = scenes.scene_room(n, 1280, 720, lidar=32, render_views=(0, 8, 16, 24))
g = GaussianMap.from_rows(sc.rows)
for k in range(len(sc.cams)):
    cam = R.camera_from(sc.cams[k])
    out = R.forward(g, cam)
    z = out.ctx["proj"]["depth"].cpu().numpy()
    ent = out.ctx["entry_splat"].cpu().numpy()
    offs = out.ctx["tile_offsets"].cpu().numpy()
    nc = out.n_contrib.cpu().numpy()
    tx = (cam.width + 15) // 16
    ty, tx_ = np.mgrid[0:cam.height, 0:cam.width] // 16
    tid = (ty * tx + tx_).ravel()
    mx = np.zeros(len(offs) - 1, np.int64)
    np.maximum.at(mx, tid, nc.ravel())
    proc = np.concatenate([ent[offs[t]:offs[t] + mx[t]] for t in range(len(mx))])
    zz = z[proc]
    print(f"view {k}: E={len(ent)} processed={len(proc)} pairs(px)={int(nc.sum())}",
          " ".join(f"z<{t}:{np.mean(zz < t):.3f}" for t in (0.05, 0.1, 0.2, 0.5)),
          f"gauss z<0.05: {int(((z > 0.01) & (z < 0.05)).sum())}")
