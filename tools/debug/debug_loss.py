import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes
from paper_2507_04004_b200 import rasterizer as R, losses as L, scenes, _lib
h, w = 120, 160
ws = R.Workspace(0, w, h, 0)
f = ws.frame
print("buf", hex(ws.buf.data_ptr()), ws.buf.numel(), "loss_parts", hex(f.loss_parts), "blocks", f.loss_blocks, "loss", hex(f.loss), "color", hex(f.color))
print("tab_x", hex(f.loss_parts + 8 * 3 * f.loss_blocks), "end", hex(ws.buf.data_ptr() + ws.buf.numel()))
cam = R.Camera(w, h, 1.0, 1.0, 0.0, 0.0, np.eye(3), np.zeros(3))
v = R.DeviceView(cam, target=np.random.rand(h, w, 3), sparse_depth=np.zeros((h, w)))
raw = v.buf.cpu().numpy().tobytes()
s = _lib.GsView.from_buffer_copy(raw)
print("view target", hex(s.target), hex(v.target.data_ptr()), "k", s.lidar_k, "cam", s.cam.width, s.cam.height)
L.frame_loss(ws, v, 0.2, 0.005)
torch.cuda.synchronize(); print("loss ok", ws.loss.cpu())
