"""Photometric pose refinement on the device (R/odometry.py:305-336).

`photometric_refine(gmap, image, cam, n_iters, lr, grad_gate, opac_gate)` keeps the reference's
signature and returns `(rot_cw, trans_cw, final_loss)`.  Each iteration is forward -> tracking
loss (L1 + D-SSIM with lam 0.5, no depth term) -> gradient masked by the image-gradient and
rendered-opacity gates -> pose gradient (gs_chain_pose, attribute gradients not materialised) ->
Adam on the 6-vector with the left SO(3) update (gs_pose_adam).  The pose state stays on the
device and the camera is rewritten in place by the Adam kernel, so the n_iters iterations are one
CUDA graph replayed back to back -- the host reads the pose once at the end.  The map is
read-only (the tracker renders a published snapshot, R/cli.py:337-344).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call
from .errors import DataError
from .gaussians import as_device_map, stream_ptr
from .rasterizer import DeviceView, Workspace, _bin_frame, camera_from

STATE = 25  # rot_cw 9, trans_cw 3, Adam m 6, v 6, iteration


class PoseRefiner:
    """Device-resident refinement of one camera against a fixed map (graph-captured iteration)."""

    def __init__(self, gmap, image, cam, lr: float = 2e-3, grad_gate: float = 1.0 / 255.0,
                 opac_gate: float = 0.5, headroom: float = 1.5):
        self.g = as_device_map(gmap)
        if len(self.g) == 0:
            raise DataError("map not initialized")
        self.dev = self.g.device
        self.cam = camera_from(cam)
        w, h = int(self.cam.width), int(self.cam.height)
        self.view = DeviceView(self.cam, image, None, self.dev)  # target = the frame, no LiDAR term
        self.lr, self.opac_gate = float(lr), float(opac_gate)
        _, cnt = _bin_frame(self.g, self.view, True)
        self.ws = Workspace(len(self.g), w, h, int(int(cnt[_lib.CNT_ENTRIES]) * headroom) + 4096, self.dev)
        call("gs_loss", self.ws.fptr, self.view.ptr, 0.5, 0.0, stream_ptr())  # builds the reflection tables
        self.mask = torch.empty(h * w, dtype=torch.uint8, device=self.dev)
        call("gs_track_mask", self.view.target.data_ptr(), w, h, float(grad_gate), self.mask.data_ptr(), stream_ptr())
        self.pose_grad = torch.zeros(6, dtype=torch.float64, device=self.dev)
        self.state = torch.zeros(STATE, dtype=torch.float64, device=self.dev)
        self.graph = None
        self.reset(self.cam.rot_cw, self.cam.trans_cw)

    def reset(self, rot_cw, trans_cw) -> None:
        """Start a refinement at pose (rot_cw, trans_cw) with fresh Adam moments."""
        st = np.zeros(STATE)
        st[0:9] = np.asarray(rot_cw, float).reshape(9)
        st[9:12] = np.asarray(trans_cw, float).reshape(3)
        self.state.copy_(torch.as_tensor(st))
        v = _lib.GsView()
        v.cam = self.cam.with_pose(rot_cw, trans_cw).struct()
        v.target = self.view.target.data_ptr()
        v.lidar_k = 0
        raw = torch.frombuffer(bytearray(bytes(memoryview(v).cast("B"))), dtype=torch.uint8)
        self.view.buf.copy_(raw.to(self.dev))

    def _launch(self) -> None:
        f, s, v = self.ws.fptr, stream_ptr(), self.view.ptr
        call("gs_preprocess_ex", f, self.g.data.data_ptr(), v, _lib.GS_PP_LAZY_SH, s)
        call("gs_bin", f, _lib.GS_BIN_LAZY, s)
        call("gs_render_fwd_ex", f, _lib.GS_FWD_EARLY_STOP | _lib.GS_FWD_CLEAR_G2D, s)
        # R/odometry.py:323: photometric_loss(lam=0.5).  No LiDAR term (lidar_k = 0): the depth /
        # opacity gradient images stay as the table-building gs_loss left them, zero
        call("gs_loss_ex", f, v, 0.5, 0.0, _lib.GS_LOSS_TABLES_READY | _lib.GS_LOSS_DEPTH_GRADS_ZERO, s)
        call("gs_track_grad", f, self.mask.data_ptr(), self.opac_gate, s)
        call("gs_render_bwd_ex", f, _lib.GS_BWD_ROWS_ZERO, s)  # gs_render_fwd cleared the rows (lazy lists)
        call("gs_chain_pose", f, self.g.data.data_ptr(), None, None, v, self.pose_grad.data_ptr(), s)
        call("gs_pose_adam", v, self.state.data_ptr(), self.pose_grad.data_ptr(), self.lr, s)

    def capture(self) -> None:
        torch.cuda.current_stream().synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch()
        self.graph = g

    def run(self, n_iters: int) -> None:
        for _ in range(int(n_iters)):
            if self.graph is not None:
                self.graph.replay()
            else:
                self._launch()

    def result(self):
        st = self.state.cpu().numpy()
        if int(self.ws.counters[_lib.CNT_OVERFLOW].item()):
            raise DataError("tile entry capacity overflowed during refinement; raise headroom")
        return st[0:9].reshape(3, 3).copy(), st[9:12].copy(), float(self.ws.loss[0].item())


def photometric_refine(gmap, image, cam, n_iters: int = 30, lr: float = 2e-3, grad_gate: float = 1.0 / 255.0,
                       opac_gate: float = 0.5):
    """R/odometry.py:305-336: Adam on the camera pose tangent against the map rendering.
    Returns (rot_cw, trans_cw, final_loss)."""
    r = PoseRefiner(gmap, image, cam, lr, grad_gate, opac_gate)
    r.capture()
    r.run(n_iters)
    return r.result()
