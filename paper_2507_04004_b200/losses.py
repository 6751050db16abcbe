"""Drop-in mirror of R/losses.py over the fused sm_100a loss kernels.

`mapping_loss(color, depth, opac, target, sparse_depth, lam, xi)` returns the reference's
(L, dL/dcolor, xi dLd/ddepth, xi dLd/dopacity).  The photometric term (R/losses.py:89-130)
runs as one fused L1 + D-SSIM kernel with the exact mirror-padding adjoint; the depth term
(R/losses.py:133-154) runs only on the LiDAR pixels (sparse_depth > 0 compacted to a K-list).
"""

from __future__ import annotations

import torch

from ._lib import call
from .errors import DomainError
from .gaussians import default_device, stream_ptr
from .rasterizer import Camera, DeviceView, Workspace, _f32

WINDOW = 11
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2
GUARD = 1e-6

_WS: dict = {}


def _loss_workspace(h: int, w: int, device) -> Workspace:
    key = (h, w, str(device))
    ws = _WS.get(key)
    if ws is None:
        ws = Workspace(0, w, h, 0, device)
        _WS[key] = ws
    return ws


def frame_loss(ws: Workspace, view: DeviceView, lam: float, xi: float) -> None:
    """Loss + image gradients of a rendered frame, in place (no host sync)."""
    call("gs_loss", ws.fptr, view.ptr, float(lam), float(xi), stream_ptr())


def _run(color, depth, opac, target, sparse_depth, lam, xi):
    dev = default_device()
    c = _f32(color, dev)
    h, w = int(c.shape[0]), int(c.shape[1])
    if c.ndim != 3 or c.shape[2] != 3:
        raise DomainError("colour images must be (H, W, 3)")
    ws = Workspace(0, w, h, 0, dev)
    ws.color.copy_(c)
    ws.depth.copy_(_f32(depth, dev).reshape(h, w) if depth is not None else torch.zeros((h, w), device=dev))
    ws.opacity.copy_(_f32(opac, dev).reshape(h, w) if opac is not None else torch.zeros((h, w), device=dev))
    cam = Camera(w, h, 1.0, 1.0, 0.0, 0.0, [[1, 0, 0], [0, 1, 0], [0, 0, 1]], [0, 0, 0])
    sd = sparse_depth if sparse_depth is not None else torch.zeros((h, w), device=dev)
    view = DeviceView(cam, target=target, sparse_depth=sd, device=dev)
    frame_loss(ws, view, lam, xi)
    return ws


def mapping_loss(color, depth, opac, target_color, sparse_depth, lam: float, xi: float):
    """R/losses.py:157-161: L = Lc + xi Ld; returns (L, gC, xi gD, xi gO)."""
    ws = _run(color, depth, opac, target_color, sparse_depth, lam, xi)
    return float(ws.loss[0].item()), ws.g_color.clone(), ws.g_depth.clone(), ws.g_opac.clone()


def photometric_loss(rendered, target, lam: float):
    """R/losses.py:122-130: (1-lam) L1 + lam D-SSIM and its gradient."""
    ws = _run(rendered, None, None, target, None, lam, 0.0)
    return float(ws.loss[1].item()), ws.g_color.clone()


def dssim_and_grad(rendered, target):
    """R/losses.py:89-119: (1 - SSIM)/2 and its exact gradient."""
    ws = _run(rendered, None, None, target, None, 1.0, 0.0)
    return float(ws.loss[3].item()), ws.g_color.clone()


def depth_ratio_loss(depth, opac, sparse_depth, guard: float = GUARD):
    """R/losses.py:133-154 (value, d/d depth, d/d opacity), evaluated on the LiDAR pixels."""
    if guard != GUARD:
        raise DomainError("the fused depth loss is compiled for guard = 1e-6 (the reference default)")
    dev = default_device()
    d = _f32(depth, dev)
    h, w = int(d.shape[0]), int(d.shape[1])
    zeros = torch.zeros((h, w, 3), device=dev)
    ws = _run(zeros, d, opac, zeros, sparse_depth, 0.0, 1.0)
    return float(ws.loss[2].item()), ws.g_depth.clone(), ws.g_opac.clone()
