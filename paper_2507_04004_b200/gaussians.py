"""Device-resident Gaussian map (mirror of R/gaussians.py) and projection / SH entry points.

`GaussianMap` keeps every splat as one 256-B row of float32 in HBM (59 used columns, in the
order of the reference's GaussianMap.parameters(), R/gaussians.py:150-153, which is also the
Gaussian PLY field order, R/gaussians.py:255-256).  The reference's attribute arrays are
exposed as strided torch views of those rows, so `gmap.pos`, `gmap.sh_high[:, 3, 1]` ... read
and write the device map in place.  Rows make the sparse Adam update and checkpointing one
contiguous 256-B read/write per touched Gaussian.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import GS_ROW, call

SH_C0 = 0.28209479177387814
N_SH = 16
DILATION = 0.3
NEAR_CLIP = 0.01
ALPHA_CLAMP = 0.99
INIT_OPACITY = 0.1

SLICES = {"pos": (0, 3), "log_scale": (3, 6), "quat": (6, 10), "opacity_logit": (10, 11),
          "sh_low": (11, 14), "sh_high": (14, 59)}
NAMES = ("pos", "log_scale", "quat", "opacity_logit", "sh_low", "sh_high")


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_04004_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    return _lib.P(torch.cuda.current_stream().cuda_stream)


def _as_f32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float32)
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device=device)


def sigmoid(x):
    return torch.sigmoid(x) if isinstance(x, torch.Tensor) else 1.0 / (1.0 + np.exp(-x))


def logit(p):
    return torch.log(p / (1.0 - p)) if isinstance(p, torch.Tensor) else np.log(p / (1.0 - p))


class GaussianMap:
    """Structure of parameter rows on the device; rows are individual splats."""

    def __init__(self, pos=None, log_scale=None, quat=None, opacity_logit=None, sh_low=None, sh_high=None,
                 device=None, capacity: int | None = None):
        self.device = torch.device(device) if device is not None else default_device()
        n = 0 if pos is None else len(pos)
        cap = max(int(capacity or 0), n, 1)
        self.data = torch.zeros((cap, GS_ROW), dtype=torch.float32, device=self.device)
        self.n = n
        if n:
            cols = {"pos": pos, "log_scale": log_scale, "quat": quat, "opacity_logit": opacity_logit,
                    "sh_low": sh_low, "sh_high": sh_high}
            for name, (a, b) in SLICES.items():
                self.data[:n, a:b] = _as_f32(cols[name], self.device).reshape(n, b - a)

    # -- construction ---------------------------------------------------------------
    @staticmethod
    def from_rows(rows, device=None, capacity=None) -> "GaussianMap":
        g = GaussianMap(device=device, capacity=capacity or len(rows))
        r = _as_f32(rows, g.device)
        g.data[:len(r), :r.shape[1]] = r[:, :GS_ROW]
        g.n = len(r)
        return g

    @staticmethod
    def from_reference(ref_map, device=None) -> "GaussianMap":
        """From a reference-style GaussianMap (numpy attribute arrays)."""
        n = len(ref_map.pos)
        return GaussianMap(ref_map.pos, ref_map.log_scale, ref_map.quat, ref_map.opacity_logit,
                           ref_map.sh_low, np.asarray(ref_map.sh_high).reshape(n, 15, 3), device=device)

    # -- reference surface (R/gaussians.py:118-153) ------------------------------------
    def __len__(self) -> int:
        return self.n

    def rows(self) -> torch.Tensor:
        return self.data[:self.n]

    def _col(self, name):
        a, b = SLICES[name]
        v = self.data[:self.n, a:b]
        if name == "opacity_logit":
            return v[:, 0]
        if name == "sh_high":
            return v.view(self.n, 15, 3) if self.n else v.reshape(0, 15, 3)
        return v

    pos = property(lambda self: self._col("pos"))
    log_scale = property(lambda self: self._col("log_scale"))
    quat = property(lambda self: self._col("quat"))
    opacity_logit = property(lambda self: self._col("opacity_logit"))
    sh_low = property(lambda self: self._col("sh_low"))
    sh_high = property(lambda self: self._col("sh_high"))

    def parameters(self) -> dict:
        return {k: self._col(k) for k in NAMES}

    def reserve(self, capacity: int) -> None:
        if capacity > self.data.shape[0]:
            new = torch.zeros((capacity, GS_ROW), dtype=torch.float32, device=self.device)
            new[:self.n] = self.data[:self.n]
            self.data = new

    def append(self, other: "GaussianMap") -> None:
        """R/gaussians.py:132-134, with capacity doubling instead of a concatenation."""
        need = self.n + len(other)
        if need > self.data.shape[0]:
            self.reserve(max(need, 2 * self.data.shape[0]))
        self.data[self.n:need] = other.rows().to(self.device)
        self.n = need

    def snapshot(self) -> "GaussianMap":
        """Independent copy safe to render from while the original trains (R/gaussians.py:136-139)."""
        return GaussianMap.from_rows(self.rows().clone(), device=self.device)

    def opacity(self) -> torch.Tensor:
        return torch.sigmoid(self.opacity_logit)

    def scale(self) -> torch.Tensor:
        return torch.exp(self.log_scale)

    def to_numpy_rows(self) -> np.ndarray:
        return self.rows()[:, :59].double().cpu().numpy()


def as_device_map(gmap, device=None) -> GaussianMap:
    if isinstance(gmap, GaussianMap):
        return gmap
    return GaussianMap.from_reference(gmap, device=device)


def init_from_points(points, colors, depths, focal: float, device=None) -> GaussianMap:
    """R/gaussians.py:227-248 through gs_init_rows: isotropic footprint scale log(max(depth /
    focal, 1e-9)), identity rotation, opacity 0.1, degree-0 SH matching the colour."""
    dev = torch.device(device) if device is not None else default_device()
    pts = _as_f32(points, dev).reshape(-1, 3).contiguous()
    col = _as_f32(colors, dev).reshape(-1, 3).contiguous()
    dep = _as_f32(depths, dev).reshape(-1).contiguous()
    m = len(pts)
    g = GaussianMap(device=dev, capacity=max(m, 1))
    call("gs_init_rows", pts.data_ptr(), col.data_ptr(), dep.data_ptr(), m, float(focal), g.data.data_ptr(),
         stream_ptr())
    g.n = m
    return g


# ---------------------------------------------------------------------------
# projection / SH (R/gaussians.py:102-111, 180-215)


def camera_struct(rot_cw, trans_cw, intrinsics, width=0, height=0) -> _lib.GsCamera:
    c = _lib.GsCamera()
    c.width, c.height = int(width), int(height)
    c.fx, c.fy, c.cx, c.cy = (float(v) for v in intrinsics)
    r = np.asarray(rot_cw, dtype=np.float64).reshape(9)
    t = np.asarray(trans_cw, dtype=np.float64).reshape(3)
    for k in range(9):
        c.rot_cw[k] = float(r[k])
    for k in range(3):
        c.trans_cw[k] = float(t[k])
    _lib.lib().gs_camera_init(c)
    return c


def struct_to_device(s, device) -> torch.Tensor:
    raw = bytes(memoryview(s).cast("B"))
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def _host_dict(d: dict) -> dict:
    return {k: (v.double() if v.is_floating_point() else v).cpu().numpy() for k, v in d.items()}


def project(gmap, rot_cw, trans_cw, intrinsics) -> dict:
    """R/gaussians.py:180-215 on the device; returns the reference's record dict (numpy arrays for
    a reference-typed map, device tensors for a device map)."""
    if not isinstance(gmap, GaussianMap) or _lib.HOST_ARRAYS:
        host_mode, _lib.HOST_ARRAYS = _lib.HOST_ARRAYS, False
        try:
            return _host_dict(project(as_device_map(gmap), rot_cw, trans_cw, intrinsics))
        finally:
            _lib.HOST_ARRAYS = host_mode
    g = gmap
    n = len(g)
    dev = g.device
    cam_buf = struct_to_device(camera_struct(rot_cw, trans_cw, intrinsics), dev)
    out = {"mu_cam": torch.empty((n, 3), device=dev), "mean2d": torch.empty((n, 2), device=dev),
           "cov2d": torch.empty((n, 2, 2), device=dev), "conic": torch.empty((n, 3), device=dev),
           "depth": torch.empty(n, device=dev), "valid": torch.empty(n, dtype=torch.uint8, device=dev),
           "jproj": torch.empty((n, 2, 3), device=dev), "m": torch.empty((n, 2, 3), device=dev),
           "cov3d": torch.empty((n, 3, 3), device=dev)}
    if n:
        call("gs_project", g.data.data_ptr(), n, cam_buf.data_ptr(), *(out[k].data_ptr() for k in
             ("mu_cam", "mean2d", "cov2d", "conic", "depth", "valid", "jproj", "m", "cov3d")), stream_ptr())
    out["valid"] = out["valid"].bool()
    return out


def eval_sh(sh_low, sh_high, dirs):
    """R/gaussians.py:102-111: returns (colors, preclamp) -- numpy for numpy inputs."""
    if not isinstance(dirs, torch.Tensor):
        col, pre = eval_sh(sh_low, sh_high, _as_f32(dirs, default_device()))
        return col.double().cpu().numpy(), pre.double().cpu().numpy()
    dev = default_device()
    sl = _as_f32(sh_low, dev).reshape(-1, 3).contiguous()
    sh = _as_f32(sh_high, dev).reshape(-1, 45).contiguous()
    d = _as_f32(dirs, dev).reshape(-1, 3).contiguous()
    n = len(d)
    col = torch.empty((n, 3), device=dev)
    pre = torch.empty((n, 3), device=dev)
    if n:
        call("gs_eval_sh", sl.data_ptr(), sh.data_ptr(), d.data_ptr(), n, col.data_ptr(), pre.data_ptr(),
             stream_ptr())
    return col, pre
