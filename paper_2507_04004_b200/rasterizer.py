"""Drop-in mirror of R/rasterizer.py over the sm_100a kernels.

Same entry points and argument meaning as the reference (`forward`, `backward`, `backward_2d`,
`cull_tiles`, `sparse_adam_step`, `AdamState`, `default_lrs`, `Camera`, `RenderOutput`); arrays
are torch CUDA tensors (numpy inputs are accepted and uploaded).  Each call runs on the
current torch stream through the C ABI of include/gslic.h; per-view transient state lives in
a `Workspace` owned by the returned RenderOutput, so concurrent renders (tracker thread vs
mapper thread, R/cli.py:298-344) never share scratch memory.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import GS_G2D, GS_ROW, GS_SPLAT, call
from .errors import DataError
from .gaussians import (GaussianMap, NAMES, SLICES, as_device_map, camera_struct, default_device,
                        stream_ptr, struct_to_device)

TILE = 16
CULL_ALPHA = 1.0 / 255.0
EARLY_STOP_T = 1e-4
BUCKET = 32  # the reference's checkpoint bucket; the B200 backward needs no checkpoints

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-15


@dataclass
class Camera:
    """R/rasterizer.py:47-67 (world->camera pose, pixel centres at integers)."""
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    rot_cw: np.ndarray
    trans_cw: np.ndarray

    @property
    def intrinsics(self):
        return (self.fx, self.fy, self.cx, self.cy)

    def center(self) -> np.ndarray:
        return -np.asarray(self.rot_cw).T @ np.asarray(self.trans_cw)

    def with_pose(self, rot_cw, trans_cw) -> "Camera":
        return Camera(self.width, self.height, self.fx, self.fy, self.cx, self.cy,
                      np.asarray(rot_cw, float), np.asarray(trans_cw, float))

    def struct(self) -> _lib.GsCamera:
        return camera_struct(self.rot_cw, self.trans_cw, self.intrinsics, self.width, self.height)


def camera_from(c) -> Camera:
    if isinstance(c, Camera):
        return c
    if isinstance(c, dict):
        return Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"], c["trans_cw"])
    return Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, np.asarray(c.rot_cw), np.asarray(c.trans_cw))


@dataclass
class RenderOutput:
    """R/rasterizer.py:70-77."""
    color: torch.Tensor
    depth: torch.Tensor
    opacity: torch.Tensor
    transmittance: torch.Tensor
    n_contrib: torch.Tensor
    ctx: dict


# ---------------------------------------------------------------------------
# device-side view (camera + supervision) and workspace


class DeviceView:
    """A gs_view struct in device memory, plus the tensors it points at."""

    def __init__(self, cam, target=None, sparse_depth=None, device=None):
        cam = camera_from(cam)
        self.cam = cam
        self.device = torch.device(device) if device is not None else default_device()
        s = _lib.GsView()
        s.cam = cam.struct()
        h, w = int(cam.height), int(cam.width)
        self.target = None
        if target is not None:
            self.target = _f32(target, self.device).reshape(h, w, 3).contiguous()
            s.target = self.target.data_ptr()
        self.sparse = None
        if sparse_depth is not None:
            self.sparse = _f32(sparse_depth, self.device).reshape(h, w).contiguous()
            self.lidar_idx = torch.empty(h * w + (h * w + 1023) // 1024, dtype=torch.int32, device=self.device)
            self.lidar_z = torch.empty(h * w, dtype=torch.float32, device=self.device)
            s.lidar_idx = self.lidar_idx.data_ptr()
            s.lidar_z = self.lidar_z.data_ptr()
        s.lidar_k = 0
        self.buf = struct_to_device(s, self.device)
        if self.sparse is not None:
            k_ptr = self.buf.data_ptr() + _lib.GsView.lidar_k.offset
            call("gs_lidar_compact", self.sparse.data_ptr(), w, h, self.lidar_idx.data_ptr(),
                 self.lidar_z.data_ptr(), k_ptr, stream_ptr())

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def set_supervision(self, target, sparse_depth) -> None:
        """Overwrite the view's target image and LiDAR returns in place (same image size; a
        view built with both), recompacting the K-list on the device."""
        h, w = int(self.cam.height), int(self.cam.width)
        if target is None:
            self.target.zero_()
        else:
            self.target.copy_(_f32(target, self.device).reshape(h, w, 3))
        if sparse_depth is None:
            self.sparse.zero_()
        else:
            self.sparse.copy_(_f32(sparse_depth, self.device).reshape(h, w))
        k_ptr = self.buf.data_ptr() + _lib.GsView.lidar_k.offset
        call("gs_lidar_compact", self.sparse.data_ptr(), w, h, self.lidar_idx.data_ptr(), self.lidar_z.data_ptr(),
             k_ptr, stream_ptr())


def _f32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float32)
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device=device)


_DT = {"f32": (torch.float32, 4), "i32": (torch.int32, 4), "u8": (torch.uint8, 1), "f64": (torch.float64, 8),
       "u64": (torch.int64, 8)}


class Workspace:
    """One view's transient device state (gs_frame), carved from a single torch buffer."""

    def __init__(self, n: int, width: int, height: int, capacity: int, device=None):
        self.device = torch.device(device) if device is not None else default_device()
        L = _lib.lib()
        self.n, self.width, self.height, self.capacity = int(n), int(width), int(height), int(capacity)
        size = int(L.gs_workspace_size(self.n, self.width, self.height, self.capacity))
        # zero-filled once: the sort look-back words are epoch-tagged and never cleared (gslic.h)
        self.buf = torch.zeros(size + 256, dtype=torch.uint8, device=self.device)
        base = self.buf.data_ptr()
        self.base = (base + 255) & ~255
        self.frame = _lib.GsFrame()
        call("gs_frame_layout", self.n, self.width, self.height, self.capacity, self.base, size, self.frame)
        self.fptr = _lib.ctypes.byref(self.frame)
        self.tiles_x, self.tiles_y = self.frame.tiles_x, self.frame.tiles_y
        h, w, n = self.height, self.width, max(self.n, 0)
        self.color = self.view("color", "f32", (h, w, 3))
        self.depth = self.view("depth", "f32", (h, w))
        self.opacity = self.view("opacity", "f32", (h, w))
        self.trans = self.view("trans", "f32", (h, w))
        self.n_contrib = self.view("n_contrib", "i32", (h, w))
        self.g_color = self.view("g_color", "f32", (h, w, 3))
        self.g_depth = self.view("g_depth", "f32", (h, w))
        self.g_opac = self.view("g_opac", "f32", (h, w))
        self.splat2d = self.view("splat2d", "f32", (n, GS_SPLAT))
        self.cov2d = self.view("cov2d", "f32", (n, 4))
        self.valid = self.view("valid", "u8", (n,))
        self.touched = self.view("touched", "u8", (n,))
        self.g2d_fixed = self.view("g2d", "u64", (n, GS_G2D))
        self.counters = self.view("counters", "i32", (2 * _lib.GS_CNT_SLOTS,))
        self.entry_splat = self.view("entry_splat", "i32", (max(self.capacity, 1),))
        self.tile_offsets = self.view("tile_offsets", "i32", (self.tiles_x * self.tiles_y + 1,))
        self.loss = self.view("loss", "f64", (8 + 5 * _lib.GS_LOSS_RING,))

    @property
    def g2d(self) -> torch.Tensor:
        """(n, 10) float64 screen-space gradient rows (mean2d 2, conic 3, opacity, colour 3, depth)
        by Gaussian, decoded from the fixed-point accumulators: value = hi 2^-24 + lo 2^-64
        (gslic.h GS_G2D).  The device keeps one accumulator row per touched-list slot (the slot is
        float 14 of the Gaussian's splat record); rows of untouched Gaussians read zero."""
        n = self.g2d_fixed.shape[0]
        if n == 0:
            return g2d_decode(self.g2d_fixed)
        slot = self.splat2d[:, 14].contiguous().view(torch.int32).long().clamp_(0, n - 1)
        rows = g2d_decode(self.g2d_fixed.index_select(0, slot))
        return torch.where(self.touched.bool()[:, None], rows, torch.zeros((), dtype=rows.dtype, device=rows.device))

    def view(self, field: str, kind: str, shape) -> torch.Tensor:
        dtype, item = _DT[kind]
        off = getattr(self.frame, field) - self.base + (self.base - self.buf.data_ptr())
        nbytes = int(np.prod(shape)) * item
        return self.buf[off:off + nbytes].view(dtype).view(*shape)


def g2d_decode(fixed: torch.Tensor) -> torch.Tensor:
    """Fixed-point (hi, lo) int64 pairs -> float64 values (same arithmetic as the device's fx_value)."""
    return fixed[:, 0::2].double() * 2.0 ** -24 + fixed[:, 1::2].double() * 2.0 ** -64


_CAP_HINT: dict = {}
_CAP_LOCK = threading.Lock()


def _capacity_hint(n: int, w: int, h: int, cull: bool) -> int:
    with _CAP_LOCK:
        hint = _CAP_HINT.get((n, w, h, cull))
    if hint:
        return hint
    if not cull:
        return max(n * ((w + 15) // 16) * ((h + 15) // 16), 1024)
    return max(8 * n, 1 << 16)


def _remember_capacity(n, w, h, cull, entries):
    with _CAP_LOCK:
        _CAP_HINT[(n, w, h, cull)] = max(int(entries * 1.25) + 1024, 1 << 16)


# Flags of the iteration engines (MapOptimizer, BatchMapOptimizer): the loss reflection tables
# are built once per workspace, and the depth / opacity gradient images stay zero between
# iterations -- the loss writes only the LiDAR pixels and the backward clears them.
LOSS_FLAGS = _lib.GS_LOSS_TABLES_READY | _lib.GS_LOSS_DEPTH_GRADS_ZERO
BWD_FLAGS = _lib.GS_BWD_ROWS_ZERO | _lib.GS_BWD_CLEAR_DEPTH_GRADS
# the engines' forward: early termination, and the g2d rows cleared for the ROWS_ZERO backward
# (from this many touched Gaussians on; below it the chain rule clears the rows it reads)
FWD_FLAGS = _lib.GS_FWD_EARLY_STOP | _lib.GS_FWD_CLEAR_G2D
FWD_CLEAR_MIN_TOUCHED = 65536


def engine_fwd_flags(max_touched: int) -> int:
    """The forward flags an iteration engine keeps for all its iterations (gslic.h GS_FWD_CLEAR_G2D)."""
    return FWD_FLAGS if max_touched >= FWD_CLEAR_MIN_TOUCHED else _lib.GS_FWD_EARLY_STOP


def prime_workspace(ws: Workspace, view_ptr: int, lam: float, xi: float) -> None:
    """Bring a fresh (zero-filled) workspace into the engines' state: one gs_loss builds the
    reflection tables, a backward over its still-empty tiles clears the gradient images."""
    call("gs_loss", ws.fptr, view_ptr, float(lam), float(xi), stream_ptr())
    call("gs_render_bwd_ex", ws.fptr, BWD_FLAGS, stream_ptr())


def _bin_frame(g: GaussianMap, view: DeviceView, cull: bool, ws: Workspace | None = None):
    """preprocess + bin with an exact-capacity retry (one host sync: E is data dependent)."""
    cam = view.cam
    n, w, h = len(g), int(cam.width), int(cam.height)
    cap = _capacity_hint(n, w, h, cull)
    for _ in range(4):
        if ws is None or ws.capacity < cap:
            ws = Workspace(n, w, h, cap, g.device)
        call("gs_preprocess", ws.fptr, g.data.data_ptr(), view.ptr, stream_ptr())
        call("gs_bin", ws.fptr, int(bool(cull)), stream_ptr())
        cnt = ws.counters[:8].cpu()
        entries = int(cnt[_lib.CNT_ENTRIES])
        if not int(cnt[_lib.CNT_OVERFLOW]):
            _remember_capacity(n, w, h, cull, entries)
            return ws, cnt
        cap = int(entries * 1.25) + 1024
    raise DataError("tile binning kept overflowing its entry capacity")


def is_host_map(gmap) -> bool:
    """A reference-typed map (numpy attribute arrays, R/gaussians.py:118-153) rather than a device
    GaussianMap: the reference-shaped entry points then return numpy arrays, as the reference."""
    return not isinstance(gmap, GaussianMap)


def _to_host(x):
    """Device tensor -> numpy (float64 for floating point), recursively through dicts."""
    if isinstance(x, dict):
        return {k: _to_host(v) for k, v in x.items()}
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.is_floating_point():
            t = t.double()
        return t.cpu().numpy()
    return x


def _view_dirs(g: GaussianMap, cam: Camera):
    """R/rasterizer.py:447-452 preamble: camera->Gaussian directions, their norms (< 1e-12 -> 1)
    and the pre-clamp SH colours."""
    from .gaussians import eval_sh
    c = torch.as_tensor(np.asarray(cam.center(), dtype=np.float32), device=g.device)
    u = g.pos - c
    nrm = torch.linalg.norm(u, dim=1, keepdim=True)
    nrm = torch.where(nrm < 1e-12, torch.ones_like(nrm), nrm)
    dirs = u / nrm
    _, pre = eval_sh(g.sh_low, g.sh_high, dirs)
    return dirs, nrm, pre


def forward(gmap, cam, cull: bool = True, early_stop: bool = True) -> RenderOutput:
    """R/rasterizer.py:442-484: render colour, depth (sum z w), opacity, transmittance, n_contrib.
    The reference's ctx keys are all present (R/rasterizer.py:479-483).  A device GaussianMap gives
    CUDA tensors; a reference-typed numpy map gives numpy arrays (float64 images, int64 entry
    lists), so reference callers' numpy code (R/cli.py:153-159, R/mapper.py:218-230,
    R/apps.py:208-223) runs unchanged."""
    host = is_host_map(gmap) or _lib.HOST_ARRAYS
    g = as_device_map(gmap)
    cam = camera_from(cam)
    view = DeviceView(cam, device=g.device)
    ws, cnt = _bin_frame(g, view, cull)
    call("gs_render_fwd", ws.fptr, int(bool(early_stop)), stream_ptr())
    E = int(cnt[_lib.CNT_ENTRIES])
    n = len(g)
    s2 = ws.splat2d
    proj = {"mean2d": s2[:, 0:2], "conic": s2[:, [2, 12, 13]], "depth": s2[:, 6], "valid": ws.valid.bool(),
            "cov2d": ws.cov2d[:, [0, 1, 1, 2]].reshape(n, 2, 2), "radius": ws.cov2d[:, 3]}
    dirs, unorm, pre = _view_dirs(g, cam)
    ctx = {"proj": proj, "opac": s2[:, 5], "colors": s2[:, 8:11], "preclamp": pre, "dirs": dirs, "u_norm": unorm,
           "entry_splat": ws.entry_splat[:E], "tile_offsets": ws.tile_offsets, "tiles_x": ws.tiles_x,
           "tiles_y": ws.tiles_y, "cam": cam}
    images = (ws.color, ws.depth, ws.opacity, ws.trans, ws.n_contrib)
    if host:
        ctx = _to_host(ctx)
        ctx["entry_splat"] = ctx["entry_splat"].astype(np.int64)
        ctx["tile_offsets"] = ctx["tile_offsets"].astype(np.int64)
        images = tuple(_to_host(a) for a in images)
    ctx.update(workspace=ws, view=view, gmap=g, n=n, counters=cnt, host=host)
    return RenderOutput(*images, ctx)


def _load_image_grads(ws: Workspace, g_color_img, g_depth_img, g_opac_img):
    dev = ws.device
    for dst, src in ((ws.g_color, g_color_img), (ws.g_depth, g_depth_img), (ws.g_opac, g_opac_img)):
        if src is None:
            dst.zero_()
        elif isinstance(src, torch.Tensor) and src.data_ptr() == dst.data_ptr():
            continue
        else:
            dst.copy_(_f32(src, dev).reshape(dst.shape))


def backward_2d(out: RenderOutput, g_color_img, g_depth_img=None, g_opac_img=None):
    """R/rasterizer.py:502-540: (g_mean2d, g_conic, g_opacity, g_color, g_depth, touched)."""
    ws: Workspace = out.ctx["workspace"]
    _load_image_grads(ws, g_color_img, g_depth_img, g_opac_img)
    call("gs_render_bwd", ws.fptr, stream_ptr())
    touched = ws.touched.bool()
    g2d = torch.where(touched[:, None], ws.g2d, torch.zeros((), device=ws.device))
    res = (g2d[:, 0:2], g2d[:, 2:5], g2d[:, 5], g2d[:, 6:9], g2d[:, 9], touched)
    return tuple(_to_host(a) for a in res) if out.ctx.get("host") else res


def rows_to_grads(rows: torch.Tensor) -> dict:
    n = rows.shape[0]
    out = {}
    for name in NAMES:
        a, b = SLICES[name]
        v = rows[:, a:b]
        out[name] = v[:, 0] if name == "opacity_logit" else (v.reshape(n, 15, 3) if name == "sh_high" else v)
    out["_rows"] = rows
    return out


def grads_to_rows(grads: dict, n: int, device) -> torch.Tensor:
    if "_rows" in grads:
        return grads["_rows"]
    rows = torch.zeros((n, GS_ROW), dtype=torch.float32, device=device)
    for name in NAMES:
        a, b = SLICES[name]
        rows[:, a:b] = _f32(grads[name], device).reshape(n, b - a)
    return rows


def backward(gmap, out: RenderOutput, g_color_img, g_depth_img=None, g_opac_img=None, with_pose: bool = False):
    """R/rasterizer.py:543-556 -> (grads dict mirroring parameters(), touched, pose_grad).

    pose_grad (with_pose=True) is the 6-vector (rho, theta) on the left tangent of T_cw
    (R/rasterizer.py:646-657) as a float64 tensor, else None.  For a reference-typed map the
    three come back as numpy arrays in the reference's shapes."""
    if is_host_map(gmap) or out.ctx.get("host"):
        out = RenderOutput(out.color, out.depth, out.opacity, out.transmittance, out.n_contrib,
                           {**out.ctx, "host": False})
        grads, touched, pose = backward(out.ctx["gmap"], out, g_color_img, g_depth_img, g_opac_img, with_pose)
        grads.pop("_rows")
        return _to_host(grads), _to_host(touched), _to_host(pose)
    g = as_device_map(gmap)
    ws: Workspace = out.ctx["workspace"]
    view: DeviceView = out.ctx["view"]
    _load_image_grads(ws, g_color_img, g_depth_img, g_opac_img)
    call("gs_render_bwd", ws.fptr, stream_ptr())
    n = len(g)
    rows = torch.zeros((n, GS_ROW), dtype=torch.float32, device=g.device)
    acc = torch.zeros(n, dtype=torch.uint8, device=g.device)
    if with_pose:
        pose = torch.empty(6, dtype=torch.float64, device=g.device)
        call("gs_chain_pose", ws.fptr, g.data.data_ptr(), rows.data_ptr(), acc.data_ptr(), view.ptr,
             pose.data_ptr(), stream_ptr())
        return rows_to_grads(rows), acc.bool(), pose
    call("gs_chain", ws.fptr, g.data.data_ptr(), rows.data_ptr(), acc.data_ptr(), view.ptr, stream_ptr())
    return rows_to_grads(rows), acc.bool(), None


def pose_backward(gmap, out, g_color_img, g_depth_img=None, g_opac_img=None):
    """The pose gradient alone (the tracker's need, R/odometry.py:324-328): the attribute
    gradients are not materialised."""
    if is_host_map(gmap) or out.ctx.get("host"):
        return _to_host(pose_backward(out.ctx["gmap"], out, g_color_img, g_depth_img, g_opac_img))
    g = as_device_map(gmap)
    ws: Workspace = out.ctx["workspace"]
    view: DeviceView = out.ctx["view"]
    _load_image_grads(ws, g_color_img, g_depth_img, g_opac_img)
    call("gs_render_bwd", ws.fptr, stream_ptr())
    pose = torch.empty(6, dtype=torch.float64, device=g.device)
    call("gs_chain_pose", ws.fptr, g.data.data_ptr(), None, None, view.ptr, pose.data_ptr(), stream_ptr())
    return pose


def cull_tiles(mean2d, conic, cov2d, opacity, depth, valid, width, height, cull=True):
    """R/rasterizer.py:169-219 on externally supplied 2D splats.

    cov2d may be (n, 2, 2), (n, 4) or (n, 3) = (c00, c01, c11).  Returns
    (entry_splat, tile_offsets, tiles_x, tiles_y): device tensors for device inputs, int64
    numpy arrays for numpy inputs (the reference's types)."""
    if not isinstance(mean2d, torch.Tensor):
        ent, offs, tx, ty = cull_tiles(_f32(mean2d, default_device()), conic, cov2d, opacity, depth, valid, width,
                                       height, cull)
        return ent.cpu().numpy().astype(np.int64), offs.cpu().numpy().astype(np.int64), tx, ty
    dev = default_device()
    m = _f32(mean2d, dev).reshape(-1, 2).contiguous()
    n = len(m)
    cv = _f32(cov2d, dev).reshape(n, -1)
    if cv.shape[1] == 4:
        cv = cv[:, [0, 1, 3]]
    cv = cv.contiguous()
    cn = _f32(conic, dev).reshape(n, 3).contiguous()
    op = _f32(opacity, dev).reshape(n).contiguous()
    dp = _f32(depth, dev).reshape(n).contiguous()
    vd = torch.as_tensor(np.asarray(valid.cpu() if isinstance(valid, torch.Tensor) else valid, dtype=np.uint8),
                         device=dev).contiguous()
    cap = _capacity_hint(n, width, height, cull)
    for _ in range(4):
        ws = Workspace(n, width, height, cap, dev)
        call("gs_pack_splats", ws.fptr, m.data_ptr(), cn.data_ptr(), cv.data_ptr(), op.data_ptr(), dp.data_ptr(),
             vd.data_ptr(), None, stream_ptr())
        call("gs_bin", ws.fptr, int(bool(cull)), stream_ptr())
        cnt = ws.counters[:8].cpu()
        E = int(cnt[_lib.CNT_ENTRIES])
        if not int(cnt[_lib.CNT_OVERFLOW]):
            _remember_capacity(n, width, height, cull, E)
            return ws.entry_splat[:E].clone(), ws.tile_offsets.clone(), ws.tiles_x, ws.tiles_y
        cap = int(E * 1.25) + 1024
    raise DataError("tile binning kept overflowing its entry capacity")


# ---------------------------------------------------------------------------
# sparse Adam (R/rasterizer.py:674-725)


def default_lrs(scene_extent: float) -> dict:
    """R/rasterizer.py:679-681."""
    return {"pos": 1.6e-4 * scene_extent, "sh_low": 2.5e-3, "sh_high": 1.25e-4,
            "opacity_logit": 0.05, "log_scale": 5e-3, "quat": 1e-3}


def lr_columns(lrs: dict, device) -> torch.Tensor:
    col = torch.zeros(GS_ROW, dtype=torch.float32)
    for name, (a, b) in SLICES.items():
        col[a:b] = float(lrs[name])
    return col.to(device)


class AdamState:
    """R/rasterizer.py:684-704: first/second moments (device parameter rows) plus a per-splat
    int32 step counter (`t_dev`).  `t`, `m`, `v` read as device tensors -- or, once the state has
    stepped a reference-typed (numpy) map, as numpy arrays, as the reference's AdamState."""

    def __init__(self, device=None) -> None:
        self.device = torch.device(device) if device is not None else None
        self.m_rows = None
        self.v_rows = None
        self.t_dev = None
        self.host = False  # numpy views (set by sparse_adam_step on a reference-typed map)

    @property
    def t(self):
        if self.host and self.t_dev is not None:
            return self.t_dev.cpu().numpy().astype(np.int64)
        return self.t_dev

    @t.setter
    def t(self, value) -> None:
        self.t_dev = value

    def ensure(self, gmap) -> None:
        n = len(gmap)
        dev = gmap.device if isinstance(gmap, GaussianMap) else (self.device or default_device())
        if self.t_dev is None:
            self.m_rows = torch.zeros((0, GS_ROW), device=dev)
            self.v_rows = torch.zeros((0, GS_ROW), device=dev)
            self.t_dev = torch.zeros(0, dtype=torch.int32, device=dev)
        have = self.t_dev.numel()
        if have < n:
            cap = max(n, 2 * have)
            if self.m_rows.shape[0] < cap:
                for name in ("m_rows", "v_rows"):
                    old = getattr(self, name)
                    new = torch.zeros((cap, GS_ROW), device=dev)
                    new[:old.shape[0]] = old
                    setattr(self, name, new)
            t = torch.zeros(cap, dtype=torch.int32, device=dev)
            t[:have] = self.t_dev
            self.t_dev = t[:n]
        if self.t_dev.numel() > n:
            self.t_dev = self.t_dev[:n]

    def _view(self, rows) -> dict:
        d = rows_to_grads(rows[:self.t_dev.numel()])
        d.pop("_rows")
        return {k: v.double().cpu().numpy() for k, v in d.items()} if self.host else d

    @property
    def m(self) -> dict:
        return self._view(self.m_rows)

    @property
    def v(self) -> dict:
        return self._view(self.v_rows)


def sparse_adam_step(gmap, grads: dict, touched, state: AdamState, lrs: dict) -> None:
    """R/rasterizer.py:707-725: Adam restricted to touched splats, per-splat bias correction, in
    place.  A device map is updated on the device.  A reference-typed map (numpy attribute
    arrays) is updated in place on the host, at float64: the device computes the fp32 step of
    the touched rows (gs_adam on zero rows yields -step exactly) and `param[idx] += -step` is
    applied to the caller's arrays; untouched rows are not written at all."""
    n = len(gmap)
    host = not isinstance(gmap, GaussianMap)
    dev = gmap.device if not host else default_device()
    state.ensure(gmap if not host else _Sized(n, dev))
    if n == 0:
        return
    rows = grads_to_rows(grads, n, dev).contiguous()
    tm = touched if isinstance(touched, torch.Tensor) else torch.as_tensor(np.asarray(touched))
    tm = tm.to(device=dev, dtype=torch.uint8).contiguous()
    lr = lr_columns(lrs, dev)
    params = gmap.data if not host else torch.zeros((n, GS_ROW), dtype=torch.float32, device=dev)
    call("gs_adam", params.data_ptr(), state.m_rows.data_ptr(), state.v_rows.data_ptr(), state.t_dev.data_ptr(),
         rows.data_ptr(), tm.data_ptr(), n, lr.data_ptr(), stream_ptr())
    if host:
        state.host = True
        idx = np.flatnonzero(tm.cpu().numpy())
        step = params[torch.as_tensor(idx, device=dev)].double().cpu().numpy()
        for name in NAMES:
            a, b = SLICES[name]
            arr = getattr(gmap, name)
            arr[idx] += step[:, a:b].reshape((len(idx),) + arr.shape[1:])


class _Sized:
    """len() + device of a host map, for AdamState.ensure."""

    def __init__(self, n: int, device) -> None:
        self.n, self.device = n, device

    def __len__(self) -> int:
        return self.n
