"""Keyframe-batch data parallelism over NCCL.

Every rank holds a replica of the map and its Adam state.  Per step, a batch of keyframes is
split across the ranks; each rank runs forward -> loss -> backward -> chain rule for its
views, accumulating parameter-row gradients and a touched mask.  The touched masks are OR-ed
(one byte per Gaussian), then only the rows of the union are summed (allreduce_grads_sparse;
allreduce_grads is the dense single-collective form with the flag in padding column 63).  A
touched Gaussian with zero gradient still steps: its moments decay (R/rasterizer.py:714-725).
Every rank then applies the same sparse Adam step, so the replicas stay bitwise identical.

This is a deliberate, documented deviation from the reference's per-keyframe Adam
(R/mapper.py:246-257): the batch oracle is sum of per-view gradients, union of touched,
one sparse_adam_step.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from ._lib import GS_ROW, call
from .errors import DataError
from .gaussians import as_device_map, stream_ptr
from .rasterizer import (BWD_FLAGS, LOSS_FLAGS, AdamState, DeviceView, Workspace, _bin_frame, camera_from, lr_columns,
                         prime_workspace)

TOUCH_COL = GS_ROW - 1  # padding column carrying the touched flag through the allreduce


def allreduce_grads(rows: torch.Tensor, touched: torch.Tensor, group=None) -> None:
    """Sum gradient rows across ranks and OR the touched masks, with one collective."""
    if TOUCH_COL < _lib.GS_NPARAM:
        raise DataError("no padding column for the touched flag")
    rows[:, TOUCH_COL] = touched.to(rows.dtype)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
    touched.copy_((rows[:, TOUCH_COL] > 0).to(touched.dtype))
    rows[:, TOUCH_COL] = 0.0


def allreduce_grads_sparse(rows: torch.Tensor, touched: torch.Tensor, group=None) -> int:
    """Two-phase allreduce that moves only the rows someone touched: (1) the touched masks are
    OR-ed (MAX over uint8, n bytes), (2) the gradient rows of the union -- gathered in id order,
    identical on every rank -- are summed, 60 columns each (the 59 parameters, 16-B aligned), and
    scattered back.  Wire bytes n + 240 |union| instead of 256 n; same result as
    allreduce_grads.  Returns |union|."""
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if multi:
        dist.all_reduce(touched, op=dist.ReduceOp.MAX, group=group)
    idx = torch.nonzero(touched, as_tuple=True)[0]
    if multi and idx.numel():
        packed = rows.index_select(0, idx)[:, :60].contiguous()
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
        rows[idx, :60] = packed
    return int(idx.numel())


class BatchMapOptimizer:
    """Batched (optionally data-parallel) map optimisation over this rank's keyframes."""

    def __init__(self, gmap, keyframes, lrs: dict, lam: float = 0.2, xi: float = 0.005, group=None,
                 adam: AdamState | None = None, headroom: float = 1.3):
        self.g = as_device_map(gmap)
        if len(self.g) == 0:
            raise DataError("map not initialized")
        self.dev = self.g.device
        self.lam, self.xi, self.group = float(lam), float(xi), group
        self.views = [DeviceView(camera_from(kf.cam), kf.image, kf.sparse_depth, self.dev) for kf in keyframes]
        self.W, self.H = int(self.views[0].cam.width), int(self.views[0].cam.height)
        self.adam = adam if adam is not None else AdamState()
        self.adam.ensure(self.g)
        self.lr = lr_columns(lrs, self.dev)
        emax = 1
        for v in self.views:
            _, cnt = _bin_frame(self.g, v, True)
            emax = max(emax, int(cnt[_lib.CNT_ENTRIES]))
        self.ws = Workspace(len(self.g), self.W, self.H, int(emax * headroom) + 4096, self.dev)
        prime_workspace(self.ws, self.views[0].ptr, self.lam, self.xi)  # reflection tables, cleared images
        n = len(self.g)
        self.grads = torch.zeros((n, GS_ROW), dtype=torch.float32, device=self.dev)
        self.sparse_allreduce = True  # two-phase allreduce of the touched rows only
        self.touched = torch.zeros(n, dtype=torch.uint8, device=self.dev)
        self.cur = torch.empty_like(self.views[0].buf)
        self.loss_acc = torch.zeros(1, dtype=torch.float64, device=self.dev)

    def kernels_per_step(self, views: int | None = None) -> int:
        from .mapper import kernels_per_iteration
        per_view = kernels_per_iteration(self.ws.tiles_x * self.ws.tiles_y)
        return per_view * (views if views is not None else len(self.views)) + 2  # + adam, step counters

    def accumulate(self, k: int) -> None:
        """forward -> loss -> backward -> chain rule of view k into (grads, touched)."""
        self.cur.copy_(self.views[k].buf)
        self._accumulate_cur()

    def _accumulate_cur(self) -> None:
        f, s, cur = self.ws.fptr, stream_ptr(), self.cur.data_ptr()
        call("gs_preprocess_ex", f, self.g.data.data_ptr(), cur, _lib.GS_PP_LAZY_SH, s)
        call("gs_bin", f, _lib.GS_BIN_LAZY, s)
        call("gs_render_fwd", f, 1, s)
        call("gs_loss_ex", f, cur, self.lam, self.xi, LOSS_FLAGS, s)
        call("gs_render_bwd_ex", f, BWD_FLAGS, s)  # gs_chain clears the rows it consumes
        call("gs_chain", f, self.g.data.data_ptr(), self.grads.data_ptr(), self.touched.data_ptr(), cur, s)
        self.loss_acc += self.ws.loss[0:1]

    def attach_host_keyframes(self, keyframes) -> None:
        """Keyframes in pinned host memory, streamed per view (mapper.HostKeyframes)."""
        from .mapper import HostKeyframes
        self.host = HostKeyframes(keyframes, self.W, self.H, self.cur, self.dev)
        self.h2d_bytes_per_view = self.host.h2d_bytes
        self._h_loss = torch.zeros(1, dtype=torch.float64).pin_memory()

    def step_host(self, view_ids) -> None:
        """One batch over host keyframes: each view's image + K-list uploaded while the previous
        view runs, then the allreduce and the Adam step; the batch loss is read back (D2H)."""
        self.grads.zero_()
        self.touched.zero_()
        self.host.stream(view_ids, lambda j, k, view_ptr: self._accumulate_cur())
        self._finish()
        self._h_loss.copy_(self.loss_acc, non_blocking=True)

    def step(self, view_ids) -> None:
        self.grads.zero_()
        self.touched.zero_()
        for k in view_ids:
            self.accumulate(int(k))
        self._finish()

    def save_state(self) -> tuple:
        a = self.adam
        return tuple(t.clone() for t in (self.g.data, a.m_rows, a.v_rows, a.t_dev))

    def restore_state(self, state: tuple) -> None:
        a = self.adam
        for dst, src in zip((self.g.data, a.m_rows, a.v_rows, a.t_dev), state):
            dst.copy_(src)

    def _finish(self) -> None:
        if self.sparse_allreduce:
            allreduce_grads_sparse(self.grads, self.touched, self.group)
        else:
            allreduce_grads(self.grads, self.touched, self.group)
        call("gs_adam", self.g.data.data_ptr(), self.adam.m_rows.data_ptr(), self.adam.v_rows.data_ptr(),
             self.adam.t_dev.data_ptr(), self.grads.data_ptr(), self.touched.data_ptr(), len(self.g),
             self.lr.data_ptr(), stream_ptr())
