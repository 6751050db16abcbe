"""Diagnostic: large-footprint cull workload of the bench scene (counters after gs_preprocess_ex)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2507_04004_b200 import _lib, rasterizer as R
from paper_2507_04004_b200.gaussians import GaussianMap, stream_ptr
sc = bench.make_scene(bench.DEFAULT)
g = GaussianMap.from_rows(sc.rows)
for k in range(len(sc.cams)):
    view = R.DeviceView(R.camera_from(sc.cams[k]), device=g.device)
    ws, cnt = R._bin_frame(g, view, True)
    _lib.call("gs_preprocess_ex", ws.fptr, g.data.data_ptr(), view.ptr, _lib.GS_PP_LAZY_SH, stream_ptr())
    torch.cuda.synchronize()
    c = ws.counters.cpu().numpy()
    big = int(c[5]); nb = ws.view("big_list", "i32", (len(g),))[:big].long()
    rect = ws.view("rect", "i32", (len(g), 4))[nb]
    ncand = ((rect[:, 1] - rect[:, 0] + 1) * (rect[:, 3] - rect[:, 2] + 1)).cpu().numpy()
    nbands = (rect[:, 3] - rect[:, 2] + 1).cpu().numpy()
    print(f"view {k}: touched {c[2]} big {big} huge_n {c[19]} queued tiles {c[20]} big_bits_words {c[7]} "
          f"ncand sum {ncand.sum()} (>256: {(ncand > 256).sum()}, 17-256: {((ncand > 16) & (ncand <= 256)).sum()}) "
          f"bands sum {nbands.sum()} huge_E {c[17]}")
