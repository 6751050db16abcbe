"""Drop-in mirror of R/losses.py over the fused sm_100a loss kernels.

`mapping_loss(color, depth, opac, target, sparse_depth, lam, xi)` returns the reference's
(L, dL/dcolor, xi dLd/ddepth, xi dLd/dopacity).  The photometric term (R/losses.py:89-130)
runs as one fused L1 + D-SSIM kernel with the exact mirror-padding adjoint; the depth term
(R/losses.py:133-154) runs only on the LiDAR pixels (sparse_depth > 0 compacted to a K-list).
"""

from __future__ import annotations

import threading

import numpy as np
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

# one loss workspace per (thread, image size): the entry points are re-entrant across threads
# (tracker and mapper, R/cli.py:298-344) and do not allocate after the first call of a size
_TLS = threading.local()


def _workspace(h: int, w: int, dev) -> tuple:
    cache = getattr(_TLS, "ws", None)
    if cache is None:
        cache = _TLS.ws = {}
    key = (h, w, str(dev))
    if key not in cache:
        cam = Camera(w, h, 1.0, 1.0, 0.0, 0.0, np.eye(3), np.zeros(3))
        cache[key] = (Workspace(0, w, h, 0, dev), DeviceView(cam, target=np.zeros((h, w, 3)),
                                                                sparse_depth=np.zeros((h, w)), device=dev))
    return cache[key]


def frame_loss(ws: Workspace, view: DeviceView, lam: float, xi: float) -> None:
    """Loss + image gradients of a rendered frame, in place (no host sync)."""
    call("gs_loss", ws.fptr, view.ptr, float(lam), float(xi), stream_ptr())


def _run(color, depth, opac, target, sparse_depth, lam, xi):
    dev = default_device()
    c = _f32(color, dev)
    if c.ndim != 3 or c.shape[2] != 3:
        raise DomainError("colour images must be (H, W, 3)")
    h, w = int(c.shape[0]), int(c.shape[1])
    ws, view = _workspace(h, w, dev)
    ws.color.copy_(c)
    if depth is None:
        ws.depth.zero_()
    else:
        ws.depth.copy_(_f32(depth, dev).reshape(h, w))
    if opac is None:
        ws.opacity.zero_()
    else:
        ws.opacity.copy_(_f32(opac, dev).reshape(h, w))
    view.set_supervision(target, sparse_depth)
    frame_loss(ws, view, lam, xi)
    return ws


def _out(host: bool, *grads):
    """Copies of the gradient images: numpy (float64) for numpy inputs, as the reference."""
    if host:
        return tuple(g.double().cpu().numpy() for g in grads)
    return tuple(g.clone() for g in grads)


def mapping_loss(color, depth, opac, target_color, sparse_depth, lam: float, xi: float):
    """R/losses.py:157-161: L = Lc + xi Ld; returns (L, gC, xi gD, xi gO)."""
    ws = _run(color, depth, opac, target_color, sparse_depth, lam, xi)
    return (float(ws.loss[0].item()),) + _out(not isinstance(color, torch.Tensor), ws.g_color, ws.g_depth, ws.g_opac)


def photometric_loss(rendered, target, lam: float):
    """R/losses.py:122-130: (1-lam) L1 + lam D-SSIM and its gradient."""
    ws = _run(rendered, None, None, target, None, lam, 0.0)
    return (float(ws.loss[1].item()),) + _out(not isinstance(rendered, torch.Tensor), ws.g_color)


def dssim_and_grad(rendered, target):
    """R/losses.py:89-119: (1 - SSIM)/2 and its exact gradient."""
    ws = _run(rendered, None, None, target, None, 1.0, 0.0)
    return (float(ws.loss[3].item()),) + _out(not isinstance(rendered, torch.Tensor), ws.g_color)


def depth_ratio_loss(depth, opac, sparse_depth, guard: float = GUARD):
    """R/losses.py:133-154 (value, d/d depth, d/d opacity), evaluated on the LiDAR pixels."""
    if guard != GUARD:
        raise DomainError("the fused depth loss is compiled for guard = 1e-6 (the reference default)")
    dev = default_device()
    d = _f32(depth, dev)
    h, w = int(d.shape[0]), int(d.shape[1])
    zeros = torch.zeros((h, w, 3), device=dev)
    ws = _run(zeros, d, opac, zeros, sparse_depth, 0.0, 1.0)
    return (float(ws.loss[2].item()),) + _out(not isinstance(depth, torch.Tensor), ws.g_depth, ws.g_opac)
