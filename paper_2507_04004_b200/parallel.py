"""Keyframe-batch data parallelism over NCCL.

Every rank holds a replica of the map and its Adam state.  Per step, a batch of keyframes is
split across the ranks; each rank runs forward -> loss -> backward -> chain rule for its
views, accumulating parameter-row gradients and a touched mask.  The touched masks are OR-ed
(one byte per Gaussian), then only the rows of the union are summed (allreduce_grads_sparse;
allreduce_grads is the dense single-collective form with the flag in padding column 63).  A
touched Gaussian with zero gradient still steps: its moments decay (R/rasterizer.py:714-725).
Every rank then applies the same sparse Adam step, so the replicas stay bitwise identical.
`allreduce_grads` / `allreduce_grads_sparse` are the host-orchestrated (torch) forms of the
reduction, kept for CPU / gloo use; `BatchMapOptimizer` reduces on the device.

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
from .rasterizer import (BWD_FLAGS, FWD_FLAGS, LOSS_FLAGS, AdamState, DeviceView, Workspace, _bin_frame, camera_from, lr_columns,
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


class PeerExchange:
    """Every rank's gradient rows, reduced-shard buffer and two epoch flags, opened in every other
    rank's address space through CUDA IPC (one exchange at set-up), for gs_p2p_reduce_adam: the
    allreduce of the batch step reads peer memory directly (NVLink / NVSwitch on one node; the
    same device when ranks share a GPU) instead of going through NCCL."""

    def __init__(self, grads: torch.Tensor, packed: torch.Tensor, flags: torch.Tensor, group=None):
        import ctypes
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        mine = []
        try:
            for t in (grads, packed, flags):
                h = (ctypes.c_uint8 * 64)()
                off = ctypes.c_int64(0)
                call("gs_ipc_export", t.data_ptr(), ctypes.cast(h, ctypes.c_void_p), ctypes.byref(off))
                mine.append((bytes(h), int(off.value)))
        except Exception:  # noqa: BLE001 -- every rank still joins the exchange below
            mine = None
        allx = [None] * self.world
        dist.all_gather_object(allx, mine, group=group)
        self.bases = []
        if any(x is None for x in allx):
            raise RuntimeError("a rank could not export its buffers through CUDA IPC")
        ptrs = [[0] * self.world for _ in range(3)]
        for k in range(self.world):
            for j, t in enumerate((grads, packed, flags)):
                if k == self.rank:
                    ptrs[j][k] = t.data_ptr()
                    continue
                hb, off = allx[k][j]
                p, b = ctypes.c_void_p(), ctypes.c_void_p()
                hbuf = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
                call("gs_ipc_import", ctypes.cast(hbuf, ctypes.c_void_p), off, ctypes.byref(p), ctypes.byref(b))
                ptrs[j][k] = p.value
                self.bases.append(b.value)
        arr = ctypes.c_void_p * self.world
        # host arrays of device pointers (the C ABI copies them into the kernel's parameters)
        self._arrays = [arr(*ptrs[0]), arr(*ptrs[1]), arr(*ptrs[2]), arr(*[p + 8 for p in ptrs[2]])]
        self.grads, self.packed, self.gready, self.rdone = (ctypes.cast(a, ctypes.c_void_p) for a in self._arrays)

    def close(self) -> None:
        for b in self.bases:
            call("gs_ipc_close", b)
        self.bases = []


class BatchMapOptimizer:
    """Batched (optionally data-parallel) map optimisation over this rank's keyframes.

    A step: every view of the batch (this rank's share) runs forward -> loss -> backward ->
    chain rule into (grads, touched) -- the view loop graph-captured once per batch; then the
    touched masks are OR-ed across ranks (n bytes), the union is compacted in id order on the
    device (gs_compact_flags), its rows gathered into one packed buffer (gs_gather_rows), summed
    across ranks in CHUNKS collectives issued back to back, and each chunk's Adam step
    (gs_adam_packed: straight from the packed rows, clearing the consumed gradient rows and
    flags) runs as soon as its collective lands, overlapping the ones still on the wire.  The
    union's size is the one host read per batch (it sizes the collective; the entry-overflow
    flag of the batch's views rides along).  On one rank nothing is gathered: Adam reads the
    gradient rows in place."""

    CHUNKS = 4

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
        self.headroom = headroom
        emax = 1
        for v in self.views:
            _, cnt = _bin_frame(self.g, v, True)
            emax = max(emax, int(cnt[_lib.CNT_ENTRIES]))
        self.ws = self._workspace(int(emax * headroom) + 4096)
        n = len(self.g)
        self.grads = torch.zeros((n, GS_ROW), dtype=torch.float32, device=self.dev)
        self.touched = torch.zeros(n, dtype=torch.uint8, device=self.dev)
        self.idx = torch.zeros(max(n, 1), dtype=torch.int32, device=self.dev)
        self.scratch = torch.zeros((n + 1023) // 1024 + 1, dtype=torch.int32, device=self.dev)
        self.count = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # (union size, overflow, the previous batch's peer-wait error) read back once per batch
        self._h = torch.zeros(3, dtype=torch.int32).pin_memory()
        self.packed = torch.zeros((0, 60), dtype=torch.float32, device=self.dev)
        self.cur = torch.empty_like(self.views[0].buf)
        self.loss_acc = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.graphs: dict = {}
        self.union = 0
        self.replayed = 0
        self.keep_reduced = False  # tests: keep (union ids, reduced gradient rows) of the last batch
        self.reduced = None
        # world > 1: the allreduce + Adam over peer memory (gs_p2p_reduce_adam) unless
        # GSLIC_P2P=0 selects the NCCL collectives + gs_adam_packed
        import os
        self.p2p = None
        self.epoch = 0
        if self._world() > 1 and os.environ.get("GSLIC_P2P", "1") != "0":
            self.packed = torch.zeros((max(n, 1), 60), dtype=torch.float32, device=self.dev)
            self._flags = torch.zeros(2, dtype=torch.int64, device=self.dev)  # (gready, rdone) epochs
            self._ticket = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self.p2p_err = torch.zeros(1, dtype=torch.int32, device=self.dev)
            # every rank must take the same path: the peer-memory form only if every rank could
            # open every peer's buffers (CUDA IPC), else the NCCL collectives for all
            ex, ok = None, 1
            try:
                ex = PeerExchange(self.grads, self.packed, self._flags, group)
            except Exception as e:  # noqa: BLE001 -- recorded, and the ranks agree below
                self.p2p_reason = f"CUDA IPC unavailable: {e}"
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=self.dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()):
                self.p2p = ex
            else:
                if ex is not None:
                    ex.close()
                self.p2p_reason = getattr(self, "p2p_reason", "a peer rank could not open CUDA IPC handles")

    def _workspace(self, capacity: int) -> Workspace:
        ws = Workspace(len(self.g), self.W, self.H, capacity, self.dev)
        prime_workspace(ws, self.views[0].ptr, self.lam, self.xi)  # reflection tables, cleared images
        return ws

    def _world(self) -> int:
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def kernels_per_step(self, views: int | None = None) -> int:
        from .mapper import kernels_per_iteration
        per_view = kernels_per_iteration(self.ws.tiles_x * self.ws.tiles_y, chain_only=True)
        if self._world() > 1:  # compaction 2, then the fused P2P kernel or gather + Adam chunks
            extra = 2 + (1 if self.p2p is not None else 1 + self.CHUNKS)
        else:
            extra = 2 + 1
        return per_view * (views if views is not None else len(self.views)) + extra

    def accumulate(self, k: int) -> None:
        """forward -> loss -> backward -> chain rule of view k into (grads, touched)."""
        self.cur.copy_(self.views[k].buf)
        self._accumulate_cur()

    def _accumulate_cur(self, view_ptr: int | None = None) -> None:
        f, s = self.ws.fptr, stream_ptr()
        cur = self.cur.data_ptr() if view_ptr is None else view_ptr
        call("gs_preprocess_ex", f, self.g.data.data_ptr(), cur, _lib.GS_PP_LAZY_SH, s)
        call("gs_bin", f, _lib.GS_BIN_LAZY, s)
        call("gs_render_fwd_ex", f, FWD_FLAGS, s)
        call("gs_loss_ex", f, cur, self.lam, self.xi, LOSS_FLAGS, s)
        call("gs_render_bwd_ex", f, BWD_FLAGS, s)  # gs_render_fwd cleared the rows (lazy lists)
        call("gs_chain", f, self.g.data.data_ptr(), self.grads.data_ptr(), self.touched.data_ptr(), cur, s)
        self.loss_acc += self.ws.loss[0:1]
        # an overflowed view contributed nothing: remember it for the batch's check
        torch.maximum(self.overflow, self.ws.counters[_lib.CNT_OVERFLOW:_lib.CNT_OVERFLOW + 1], out=self.overflow)

    def _views(self, view_ids) -> None:
        """The batch's views, one CUDA graph replay per distinct view tuple."""
        key = tuple(int(k) for k in view_ids)
        gr = self.graphs.get(key)
        if gr is None:
            torch.cuda.current_stream().synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for k in key:
                    self._accumulate_cur(self.views[k].ptr)
            self.graphs[key] = gr
        gr.replay()

    def attach_host_keyframes(self, keyframes) -> None:
        """Keyframes in pinned host memory, streamed per view (mapper.HostKeyframes)."""
        from .mapper import HostKeyframes
        self.host = HostKeyframes(keyframes, self.W, self.H, self.cur, self.dev)
        self.h2d_bytes_per_view = self.host.h2d_bytes
        self._h_loss = torch.zeros(1, dtype=torch.float64).pin_memory()

    def step_host(self, view_ids) -> None:
        """One batch over host keyframes: each view's image + K-list uploaded while the previous
        view runs, then the reduction and the Adam step; the batch loss is read back (D2H)."""
        self.loss_acc.zero_()
        self.host.stream(view_ids, lambda j, k, view_ptr: self._accumulate_cur(view_ptr), use_cur=False)
        self._finish(lambda: self.host.stream(view_ids, lambda j, k, vp: self._accumulate_cur(vp), use_cur=False))
        self._h_loss.copy_(self.loss_acc, non_blocking=True)

    def step(self, view_ids) -> None:
        self.loss_acc.zero_()
        self._views(view_ids)
        self._finish(lambda: self._views(view_ids))

    def save_state(self) -> tuple:
        a = self.adam
        return tuple(t.clone() for t in (self.g.data, a.m_rows, a.v_rows, a.t_dev))

    def restore_state(self, state: tuple) -> None:
        a = self.adam
        for dst, src in zip((self.g.data, a.m_rows, a.v_rows, a.t_dev), state):
            dst.copy_(src)

    def _finish(self, rerun) -> None:
        s = stream_ptr()
        world = self._world()
        if world > 1:
            # every rank re-runs the batch if any view of any rank overflowed (the collectives
            # below must pair up), then the touched union
            dist.all_reduce(self.overflow, op=dist.ReduceOp.MAX, group=self.group)
            dist.all_reduce(self.touched, op=dist.ReduceOp.MAX, group=self.group)
        n = len(self.g)
        call("gs_compact_flags", self.touched.data_ptr(), n, self.idx.data_ptr(), self.count.data_ptr(),
             self.scratch.data_ptr(), s)
        self._h[0:1].copy_(self.count, non_blocking=True)
        self._h[1:2].copy_(self.overflow, non_blocking=True)
        if self.p2p is not None:
            self._h[2:3].copy_(self.p2p_err, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if int(self._h[2]):
            raise DataError("gs_p2p_reduce_adam: a peer rank never reached the batch (bounded wait expired)")
        if int(self._h[1]):  # some view overflowed its entry capacity: redo the batch's views
            torch.cuda.synchronize(self.dev)
            self.grads.zero_()
            self.touched.zero_()
            self.overflow.zero_()
            self.loss_acc.zero_()
            self.ws = self._workspace(int(self.ws.capacity * 2))
            self.graphs = {}
            self.replayed += 1
            rerun()
            self._finish(rerun)
            return
        u = self.union = int(self._h[0])
        adam_args = (self.g.data.data_ptr(), self.adam.m_rows.data_ptr(), self.adam.v_rows.data_ptr(),
                     self.adam.t_dev.data_ptr())
        if world == 1:
            if self.keep_reduced:
                ids = self.idx[:u].long()
                self.reduced = (ids.clone(), self.grads[ids, :60].clone())
            call("gs_adam_packed", *adam_args, None, self.idx.data_ptr(), self.count.data_ptr(), 0, u,
                 self.lr.data_ptr(), self.grads.data_ptr(), self.touched.data_ptr(), s)
            return
        if self.p2p is not None:  # allreduce fused with Adam over peer memory
            self.epoch += 1
            keep = torch.empty((u, 60), dtype=torch.float32, device=self.dev) if self.keep_reduced else None
            x = self.p2p
            call("gs_p2p_reduce_adam", world, x.rank, x.grads, x.packed, x.gready, x.rdone, self.epoch, u,
                 self.idx.data_ptr(), *adam_args, self.lr.data_ptr(), self.grads.data_ptr(), self.touched.data_ptr(),
                 self._ticket.data_ptr(), keep.data_ptr() if keep is not None else None, self.p2p_err.data_ptr(), s)
            if keep is not None:
                self.reduced = (self.idx[:u].long().clone(), keep)
            self.overflow.zero_()
            return
        if self.packed.shape[0] < u:
            self.packed = torch.zeros((int(u * 1.25) + 1024, 60), dtype=torch.float32, device=self.dev)
        call("gs_gather_rows", self.grads.data_ptr(), self.idx.data_ptr(), self.count.data_ptr(), u,
             self.packed.data_ptr(), s)
        bounds = [u * c // self.CHUNKS for c in range(self.CHUNKS + 1)]
        works = [dist.all_reduce(self.packed[bounds[c]:bounds[c + 1]], op=dist.ReduceOp.SUM, group=self.group,
                                 async_op=True) for c in range(self.CHUNKS)]
        if self.keep_reduced:
            for w in works:
                w.wait()
            self.reduced = (self.idx[:u].long().clone(), self.packed[:u].clone())
        for c in range(self.CHUNKS):
            works[c].wait()  # the compute stream waits for chunk c only
            call("gs_adam_packed", *adam_args, self.packed.data_ptr(), self.idx.data_ptr(), self.count.data_ptr(),
                 bounds[c], bounds[c + 1] - bounds[c], self.lr.data_ptr(), self.grads.data_ptr(),
                 self.touched.data_ptr(), stream_ptr())
        self.overflow.zero_()
