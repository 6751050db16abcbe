"""Mapping driver: mirror of R/mapper.py's optimisation loop over a device-resident engine.

`MapOptimizer` keeps every keyframe (target image + LiDAR K-list + camera) resident in HBM
and runs one map-optimisation iteration (R/mapper.py:246-263: forward -> mapping_loss ->
backward -> sparse_adam_step) as six C-ABI launches with no host synchronisation; the launch
sequence can be captured once into a CUDA graph and replayed per keyframe.  `optimize_map`
keeps the reference's signature and sampling (R/mapper.py:233-264).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call
from .errors import DataError
from .gaussians import GaussianMap, as_device_map, default_device, init_from_points, stream_ptr, struct_to_device
from .rasterizer import (BWD_FLAGS, LOSS_FLAGS, AdamState, Camera, DeviceView, Workspace, _bin_frame, camera_from,
                         default_lrs, engine_fwd_flags, forward, prime_workspace,
                         lr_columns)

NEAR_CLIP = 0.01


def kernels_per_iteration(tiles: int, chain_only: bool = False) -> int:
    """Our kernels per map-optimisation iteration: preprocess 4 (frame reset, projection +
    small-footprint cull, large-footprint bands, exact tiles), bin 3 (lazy lists: huge sort, huge
    transpose, tile scan), forward 3 (blend, bucket fill + sorted continuation for the tiles that
    need them), loss 3 (SSIM map + partials, SSIM adjoint + gradient assembly, LiDAR depth with
    the finalisation in its last block; the reflection tables are built once per workspace),
    backward 1 (the lazy forward clears the g2d rows), chain rule fused with Adam 1 (2
    with GSLIC_SPLIT_ADAM=1: chain + adam_list)."""
    del tiles
    import os
    split = os.environ.get("GSLIC_SPLIT_ADAM", "0") == "1"
    return 4 + 3 + 3 + 3 + 1 + (1 if chain_only or not split else 2)


@dataclass
class MappingConfig:
    """R/mapper.py:28-50 (the hot-path knobs: lam, xi, k_keyframes)."""
    lam: float = 0.2
    xi: float = 0.005
    k_keyframes: int = 100
    tau: float = 0.99
    n_p: int = 10
    eps1: float = 0.1
    eps2: float = 50.0
    keyframe_stride: int = 5
    grad_thresh: float = 1.0
    patch: int = 30
    refine_rounds: int = 0

    def __post_init__(self):
        if not 0.0 < self.tau < 1.0:
            raise ValueError("tau must lie in (0, 1)")
        if self.xi < 0:
            raise ValueError("xi must be non-negative")
        for name in ("lam", "k_keyframes", "n_p", "eps1", "eps2", "keyframe_stride", "grad_thresh", "patch"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")


@dataclass
class Keyframe:
    """R/mapper.py:53-66: a posed image plus its sparse LiDAR depth (and seed points)."""
    cam: Camera
    image: np.ndarray
    sparse_depth: np.ndarray
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    colors: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    stamp: float = 0.0


def _host_frame(image, h: int, w: int) -> torch.Tensor:
    """A keyframe image in pinned host memory: as 8 bits when every value is exactly k / 255 (a
    camera frame, R/io_formats.py:52-57 -- decoded on the device by gs_decode_u8 to the same fp32
    values), else as float32."""
    img = image.detach().double().cpu().numpy() if isinstance(image, torch.Tensor) else \
        np.asarray(image, dtype=np.float64)
    img = img.reshape(h, w, 3)
    q = np.round(img * 255.0)
    if np.all((q >= 0) & (q <= 255)) and np.array_equal(q / 255.0, img):
        return torch.as_tensor(q.astype(np.uint8)).pin_memory()
    return torch.as_tensor(img.astype(np.float32)).pin_memory()


class HostKeyframes:
    """Keyframes in pinned host memory -- the target image and the LiDAR returns as a K-list
    (pixel index, depth; compacted once here, as the device path caches it) -- streamed into
    NSLOT device slots: the upload of keyframe j+1 (copy stream) starts as soon as iteration
    j + 1 - NSLOT has released its slot, so it has NSLOT - 1 iterations to land.  `cur` is the
    engine's device gs_view that the captured iteration reads."""

    NSLOT = 3

    def __init__(self, keyframes, width: int, height: int, cur: torch.Tensor, device):
        h, w = int(height), int(width)
        self.cur, self.dev = cur, device
        self.img, self.idx, self.z = [], [], []
        for kf in keyframes:
            self.img.append(_host_frame(kf.image, h, w))
            sd = np.asarray(kf.sparse_depth, dtype=np.float32).reshape(-1) if kf.sparse_depth is not None else \
                np.zeros(h * w, np.float32)
            idx = np.flatnonzero(sd > 0).astype(np.int32)  # pixel order, as gs_lidar_compact
            self.idx.append(torch.as_tensor(idx).pin_memory())
            self.z.append(torch.as_tensor(sd[idx]).pin_memory())
        kmax = max(1, max(len(i) for i in self.idx))
        self.slots = [{"img": torch.empty((h, w, 3), device=device),
                       "u8": torch.empty((h, w, 3), dtype=torch.uint8, device=device),
                       "idx": torch.empty(kmax, dtype=torch.int32, device=device),
                       "z": torch.empty(kmax, device=device), "view": torch.empty_like(cur)}
                      for _ in range(self.NSLOT)]
        self.views = []  # per keyframe, per slot: the gs_view pointing at that slot's buffers
        for k, kf in enumerate(keyframes):
            per = []
            for sl in self.slots:
                v = _lib.GsView()
                v.cam = camera_from(kf.cam).struct()
                v.target, v.lidar_idx, v.lidar_z = sl["img"].data_ptr(), sl["idx"].data_ptr(), sl["z"].data_ptr()
                v.lidar_k = len(self.idx[k])
                per.append(torch.frombuffer(bytearray(bytes(memoryview(v).cast("B"))), dtype=torch.uint8).pin_memory())
            self.views.append(per)
        self.copy_stream = torch.cuda.Stream(device=device)
        self.slot_free = [None] * self.NSLOT
        nbytes = [self.img[k].numel() * self.img[k].element_size() + self.idx[k].numel() * 8 +
                  self.views[k][0].numel() for k in range(len(keyframes))]
        self.h2d_bytes = int(round(float(np.mean(nbytes))))

    def upload(self, j: int, k: int) -> torch.cuda.Event:
        """H2D of keyframe k into slot j % NSLOT on the copy stream, once the iteration that last
        read that slot has finished; returns the event marking the slot ready."""
        s = j % self.NSLOT
        sl, cs = self.slots[s], self.copy_stream
        with torch.cuda.stream(cs):
            if self.slot_free[s] is not None:
                cs.wait_event(self.slot_free[s])
            kk = self.idx[k].numel()
            if self.img[k].dtype == torch.uint8:  # 8-bit frame: a quarter of the bytes, exact decode
                sl["u8"].copy_(self.img[k], non_blocking=True)
                call("gs_decode_u8", sl["u8"].data_ptr(), sl["img"].data_ptr(), sl["img"].numel(), stream_ptr())
            else:
                sl["img"].copy_(self.img[k], non_blocking=True)
            if kk:
                sl["idx"][:kk].copy_(self.idx[k], non_blocking=True)
                sl["z"][:kk].copy_(self.z[k], non_blocking=True)
            sl["view"].copy_(self.views[k][s], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        return ev

    def replay_slot(self, k: int) -> int:
        """Keyframe k uploaded synchronously into a slot of its own (the re-run of an iteration
        whose streaming slot may have been refilled); returns the device gs_view pointer."""
        if not hasattr(self, "_replay"):
            sl = self.slots[0]
            self._replay = {key: torch.empty_like(t) for key, t in sl.items()}
            self._replay_views = []
            for kk in range(len(self.img)):
                v = _lib.GsView.from_buffer_copy(bytes(self.views[kk][0].numpy()))
                v.target, v.lidar_idx, v.lidar_z = (self._replay["img"].data_ptr(), self._replay["idx"].data_ptr(),
                                                    self._replay["z"].data_ptr())
                self._replay_views.append(torch.frombuffer(bytearray(bytes(memoryview(v).cast("B"))),
                                                           dtype=torch.uint8).pin_memory())
        r, kk = self._replay, self.idx[k].numel()
        if self.img[k].dtype == torch.uint8:
            r["u8"].copy_(self.img[k])
            call("gs_decode_u8", r["u8"].data_ptr(), r["img"].data_ptr(), r["img"].numel(), stream_ptr())
        else:
            r["img"].copy_(self.img[k])
        if kk:
            r["idx"][:kk].copy_(self.idx[k])
            r["z"][:kk].copy_(self.z[k])
        r["view"].copy_(self._replay_views[k])
        return r["view"].data_ptr()

    def stream(self, order, body, use_cur: bool = True) -> None:
        """For j, k in enumerate(order): keyframe k lands in a slot, then body(j, k, view_ptr) runs
        the iteration on the current stream (view_ptr: the slot's device gs_view; copied into
        `cur` first when use_cur); keyframe j+1 .. uploads meanwhile."""
        main = torch.cuda.current_stream()
        order = [int(k) for k in order]
        if not order:
            return
        self.copy_stream.wait_stream(main)  # uploads start after the work queued so far
        ahead = self.NSLOT - 1  # uploads in flight ahead of the iteration that runs
        ready = {}
        for j in range(min(ahead, len(order))):
            ready[j] = self.upload(j, order[j])
        for j, k in enumerate(order):
            if j + ahead < len(order):
                ready[j + ahead] = self.upload(j + ahead, order[j + ahead])
            ev = ready.pop(j)
            if not ev.query():  # uploads run ahead: usually landed already, no device-side wait
                main.wait_event(ev)
            view = self.slots[j % self.NSLOT]["view"]
            if use_cur:
                self.cur.copy_(view)
            body(j, k, view.data_ptr())
            free = torch.cuda.Event()
            free.record(main)
            self.slot_free[j % self.NSLOT] = free


class MapOptimizer:
    """Device-resident map-optimisation iterations over a fixed keyframe set."""

    def __init__(self, gmap: GaussianMap, keyframes, lrs: dict, lam: float = 0.2, xi: float = 0.005,
                 adam: AdamState | None = None, headroom: float = 1.3, views=None):
        self.g = as_device_map(gmap)
        if len(self.g) == 0:
            raise DataError("map not initialized")
        self.dev = self.g.device
        self.lam, self.xi = float(lam), float(xi)
        self.views = views if views is not None else [
            DeviceView(camera_from(kf.cam), kf.image, kf.sparse_depth, self.dev) for kf in keyframes]
        cams = [v.cam for v in self.views]
        self.W, self.H = int(cams[0].width), int(cams[0].height)
        if any((int(c.width), int(c.height)) != (self.W, self.H) for c in cams):
            raise DataError("all keyframes of one optimiser must share the image size")
        self.adam = adam if adam is not None else AdamState()
        self.adam.ensure(self.g)
        self.lr = lr_columns(lrs, self.dev)
        self.cur = torch.empty_like(self.views[0].buf)
        # entry capacity from a dry binning pass over every keyframe
        emax, tmax = 1, 1
        for v in self.views:
            _, cnt = _bin_frame(self.g, v, True)
            emax = max(emax, int(cnt[_lib.CNT_ENTRIES]))
            tmax = max(tmax, int(cnt[_lib.CNT_TOUCHED]))
        self.fwd_flags = engine_fwd_flags(tmax)
        self.headroom = headroom
        self.ws = self._workspace(int(emax * headroom) + 4096)
        self.graph = None
        self.graphs: dict = {}
        # per-step counters read back asynchronously: (event, pinned counters, how to re-run it)
        self._ring = [torch.zeros(8, dtype=torch.int32).pin_memory() for _ in range(self.RING)]
        self._pending: list = []
        self._steps = 0
        self.replayed = 0  # iterations re-run after an entry-capacity overflow
        self._dev_iter = 0  # GS_LOSS_ACCUMULATE iterations run on this workspace (its loss ring position)
        import os
        self.overlap_parts = int(os.environ.get("GSLIC_OVERLAP_PARTS", "0"))
        self._side = torch.cuda.Stream(device=self.dev)
        self._d2h = torch.cuda.Stream(device=self.dev)  # per-step read-backs (counters, losses)

    def _workspace(self, capacity: int) -> Workspace:
        """A zero-filled workspace whose loss reflection tables are built (one gs_loss on the
        blank images), so the captured iteration can skip that launch (GS_LOSS_TABLES_READY);
        a backward over its empty tiles then clears the depth / opacity gradient images that
        gs_loss wrote, the state the iteration keeps (GS_LOSS_DEPTH_GRADS_ZERO)."""
        ws = Workspace(len(self.g), self.W, self.H, capacity, self.dev)
        prime_workspace(ws, self.views[0].ptr, self.lam, self.xi)
        return ws

    # -- one iteration: R/mapper.py:249-256 --------------------------------------------
    def _launch(self, view_ptr: int | None = None) -> None:
        f, s = self.ws.fptr, stream_ptr()
        cur = self.cur.data_ptr() if view_ptr is None else view_ptr
        call("gs_preprocess_ex", f, self.g.data.data_ptr(), cur, _lib.GS_PP_LAZY_SH, s)
        call("gs_bin", f, _lib.GS_BIN_LAZY, s)
        call("gs_render_fwd_ex", f, self.fwd_flags, s)
        call("gs_loss_ex", f, cur, self.lam, self.xi, LOSS_FLAGS | _lib.GS_LOSS_ACCUMULATE, s)
        call("gs_render_bwd_ex", f, BWD_FLAGS, s)  # gs_render_fwd cleared the rows (lazy lists)
        self._chain_adam(cur)

    def _chain_adam(self, view_ptr: int | None = None) -> None:
        """Chain rule + sparse Adam.  overlap_parts > 1: the touched list is cut into chunks; the
        FP64 chain of chunk i+1 runs on this stream while the HBM-bound Adam stream of chunk i runs
        on a side stream (gs_chain_adam_part), so latency-bound math and bandwidth overlap."""
        f, s = self.ws.fptr, stream_ptr()
        cur = self.cur.data_ptr() if view_ptr is None else view_ptr
        args = (self.g.data.data_ptr(), self.adam.m_rows.data_ptr(), self.adam.v_rows.data_ptr(),
                self.adam.t_dev.data_ptr(), cur, self.lr.data_ptr())
        P = self.overlap_parts
        if P <= 1:
            call("gs_chain_adam", f, *args, s)
            return
        main = torch.cuda.current_stream()
        for i in range(P):
            call("gs_chain_adam_part", f, *args, 0, i, P, stream_ptr())
            ev = torch.cuda.Event()
            ev.record(main)
            self._side.wait_event(ev)
            with torch.cuda.stream(self._side):
                call("gs_chain_adam_part", f, *args, 1, i, P, stream_ptr())
        main.wait_stream(self._side)

    def capture(self) -> None:
        """Capture the launch sequence into CUDA graphs: one per device view (keyframes, host
        slots), each reading its own gs_view, so a step is a single replay with no view copy."""
        torch.cuda.current_stream().synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):  # capture records the launches; it executes nothing
            self._launch()
        self.graph = g
        self.graphs = {}

    def _graph_for(self, view_ptr: int):
        gr = self.graphs.get(view_ptr)
        if gr is None:
            torch.cuda.current_stream().synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                self._launch(view_ptr)
            self.graphs[view_ptr] = gr
        return gr

    RING = 8  # counter snapshots in flight (>= LAG + 2)
    LAG = 2  # steps between an iteration and the host's look at its counters (no per-step sync)

    def _run_view(self, view_ptr: int) -> None:
        if self.graph is not None:
            self._graph_for(view_ptr).replay()
        else:
            self._launch(view_ptr)

    def step(self, k: int) -> None:
        self._check(self.LAG)
        vp = self.views[k].ptr
        self._run_view(vp)
        self._record(lambda: self._run_view(vp))

    def _record(self, rerun, loss_slot: int | None = None) -> None:
        """After this iteration, read back (on the read-back stream, so the compute stream carries
        nothing but the graph replays) its counter snapshot -- written by the loss kernel into the
        workspace's device ring -- for the lagged capacity check, and with loss_slot its loss
        into pinned slot loss_slot (run_host)."""
        ring = self._ring[self._steps % self.RING]
        ev = torch.cuda.Event()
        ev.record()
        pos = self._dev_iter % _lib.GS_LOSS_RING
        d = self._d2h
        d.wait_event(ev)
        with torch.cuda.stream(d):
            ring.copy_(self._snap[pos], non_blocking=True)
            if loss_slot is not None:
                self._h_loss[loss_slot].copy_(self.ws.loss[8 + pos], non_blocking=True)
        done = torch.cuda.Event()
        done.record(d)
        self._pending.append((done, ring, rerun, loss_slot))
        self._steps += 1
        self._dev_iter += 1

    @property
    def _snap(self) -> torch.Tensor:
        """The workspace's counter snapshots (GS_LOSS_RING x 8 int32, gs_frame.loss)."""
        r = _lib.GS_LOSS_RING
        return self.ws.loss[8 + r:8 + 5 * r].view(torch.int32).view(r, 8)

    def _regrow(self, entries: int) -> None:
        torch.cuda.synchronize(self.dev)  # no kernel or copy still reads the old workspace
        old = self.ws
        self.ws = self._workspace(int(entries * self.headroom) + 4096)
        self.ws.loss[4:5].copy_(old.loss[4:5])  # the running loss sum moves along
        self._dev_iter = 0  # the new workspace's loss ring starts over
        if self.graph is not None:
            self.capture()  # (the per-view graphs are re-captured on first use)

    def _check(self, keep: int) -> None:
        """Counters of the iterations older than the last `keep` (finished in practice, so the
        event waits are free).  An iteration whose binning overflowed the entry capacity did
        nothing (background render, no gradient, no Adam step, loss not accumulated: the device
        kernels no-op on GS_CNT_OVERFLOW); the workspace is re-laid out and that iteration re-run
        at once -- after the `keep` iterations queued behind it, so the map sees it that much
        later (the only deviation from the reference's order, and only on overflow).  A step near
        capacity grows the workspace before it overflows."""
        while len(self._pending) > keep:
            ev, ring, rerun, loss_slot = self._pending.pop(0)
            ev.synchronize()
            over, entries = int(ring[_lib.CNT_OVERFLOW]), int(ring[_lib.CNT_ENTRIES])
            if over:
                self._regrow(entries)
                self.replayed += 1
                rerun()
                self._record(rerun, loss_slot)
            elif entries > 0.9 * self.ws.capacity:
                self._regrow(entries)

    def finish(self) -> None:
        """Check every queued iteration (re-running any that overflowed); returns when all of
        them have completed."""
        self._check(0)

    PHASES = ("preprocess", "bin", "render_fwd", "loss", "render_bwd", "chain_adam")

    def kernels_per_step(self) -> int:
        """Kernels of ours launched by one iteration."""
        return kernels_per_iteration(self.ws.tiles_x * self.ws.tiles_y)

    def profile_step(self, k: int) -> dict:
        """Eager iteration with CUDA events between the six C-ABI calls; returns ms per phase."""
        self.cur.copy_(self.views[k].buf)
        f, s, cur = self.ws.fptr, stream_ptr(), self.cur.data_ptr()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(self.PHASES) + 1)]
        ev[0].record()
        call("gs_preprocess_ex", f, self.g.data.data_ptr(), cur, _lib.GS_PP_LAZY_SH, s)
        ev[1].record()
        call("gs_bin", f, _lib.GS_BIN_LAZY, s)
        ev[2].record()
        call("gs_render_fwd_ex", f, self.fwd_flags, s)
        ev[3].record()
        call("gs_loss_ex", f, cur, self.lam, self.xi, LOSS_FLAGS | _lib.GS_LOSS_ACCUMULATE, s)
        ev[4].record()
        call("gs_render_bwd_ex", f, BWD_FLAGS, s)
        ev[5].record()
        self._chain_adam()
        ev[6].record()
        self._dev_iter += 1
        ev[6].synchronize()
        return {p: ev[i].elapsed_time(ev[i + 1]) for i, p in enumerate(self.PHASES)}

    # -- streaming keyframes from host memory (the e2e path) ---------------------------------
    def attach_host_keyframes(self, keyframes) -> None:
        """Keep keyframes in pinned host memory (HostKeyframes); run_host() uploads keyframe j+1
        on a copy stream while iteration j runs."""
        self.host = HostKeyframes(keyframes, self.W, self.H, self.cur, self.dev)
        self.h2d_bytes, self.d2h_bytes = self.host.h2d_bytes, 8
        self._h_loss = torch.zeros(self.LOSS_RING, dtype=torch.float64).pin_memory()
        self._host_steps = 0

    def run_host(self, order) -> None:
        """Map-optimisation iterations over host keyframes `order` (R/mapper.py:242-256 samples
        the keyframe order up front): keyframe j+1 is uploaded on a copy stream while iteration j
        runs; each iteration's loss is read back into pinned host memory (D2H)."""

        def body(j, k, view_ptr):
            self._check(self.LAG)
            self._run_view(view_ptr)
            h = self._host_steps % self.LOSS_RING
            self._host_steps += 1
            # an overflowed iteration is re-run from a dedicated slot (its streaming slot may have
            # been refilled by then) and its loss read again
            self._record(lambda: self._rerun_host(k, h), loss_slot=h)

        self.host.stream(order, body, use_cur=False)
        # the read-backs are part of the call: later work on this stream follows them
        torch.cuda.current_stream().wait_stream(self._d2h)

    LOSS_RING = 1024

    def _rerun_host(self, k: int, h: int) -> None:
        torch.cuda.synchronize(self.dev)
        self._run_view(self.host.replay_slot(k))

    def step_host(self, k: int, slot: int = 0) -> None:
        """One iteration on host keyframe k (no prefetch): run_host([k])."""
        self.run_host([k])

    def save_state(self) -> tuple:
        """Device copies of the optimised state (parameter rows, Adam m, v, t)."""
        a = self.adam
        return tuple(t.clone() for t in (self.g.data, a.m_rows, a.v_rows, a.t_dev))

    def restore_state(self, state: tuple) -> None:
        a = self.adam
        for dst, src in zip((self.g.data, a.m_rows, a.v_rows, a.t_dev), state):
            dst.copy_(src)

    def loss_sum(self, reset: bool = True) -> float:
        """Sum of the losses of the iterations since the last reset (ws.loss[4], accumulated on
        the device by the loss kernel)."""
        v = float(self.ws.loss[4].item())
        if reset:
            self.ws.loss[4:5].zero_()
        return v

    def counters(self) -> dict:
        c = self.ws.counters.cpu()
        return {"entries": int(c[1]), "touched": int(c[2]), "overflow": int(c[3]),
                "huge": int(c[_lib.GS_CNT_SLOTS + 3]), "bucketed_entries": int(c[_lib.GS_CNT_SLOTS + 2])}


_ENGINES: dict = {}
_ENGINES_LOCK = threading.Lock()


def _engine_for(gmap, keyframes, adam, lrs, cfg) -> MapOptimizer:
    # keyed on the identity of every keyframe (a keyframe replaced in place gets a new engine,
    # whose device views hold its image and camera), the map, its size and the Adam state
    key = (id(gmap), tuple(id(kf) for kf in keyframes), len(gmap), id(adam))
    with _ENGINES_LOCK:
        eng = _ENGINES.get(key)
    if eng is None or eng.g is not gmap:
        eng = MapOptimizer(gmap, keyframes, lrs, cfg.lam, cfg.xi, adam)
        with _ENGINES_LOCK:
            _ENGINES.clear()
            _ENGINES[key] = eng
    eng.lr = lr_columns(lrs, eng.dev)
    eng.lam, eng.xi = float(cfg.lam), float(cfg.xi)
    return eng


def release_engines() -> None:
    """Drop the cached optimize_map engine (its workspace and device keyframes)."""
    with _ENGINES_LOCK:
        _ENGINES.clear()


def _write_back(ref_map, rows: torch.Tensor, base: torch.Tensor) -> None:
    """Apply a device map's change since `base` to a reference-typed (numpy) map in place: the
    float64 difference of two fp32 rows is exact, so untouched rows are left bit-identical and
    touched ones move by exactly the device's step."""
    delta = rows[:, :59].double() - base[:, :59].double()
    idx = torch.nonzero(delta.abs().amax(dim=1) > 0, as_tuple=True)[0]
    d = delta[idx].cpu().numpy()
    ii = idx.cpu().numpy()
    from .gaussians import NAMES, SLICES
    for name in NAMES:
        a, b = SLICES[name]
        arr = getattr(ref_map, name)
        arr[ii] += d[:, a:b].reshape((len(ii),) + arr.shape[1:])


def _append(gmap, new: GaussianMap) -> None:
    """gmap.append(new) for a device map, or the same rows as a map of the caller's own type."""
    if isinstance(gmap, GaussianMap):
        gmap.append(new)
        return
    r = new.rows()[:, :59].double().cpu().numpy()
    n = len(r)
    gmap.append(type(gmap)(pos=r[:, 0:3], log_scale=r[:, 3:6], quat=r[:, 6:10], opacity_logit=r[:, 10],
                           sh_low=r[:, 11:14], sh_high=r[:, 14:59].reshape(n, 15, 3)))


def optimize_map(gmap, keyframes, cfg: MappingConfig, rng, adam: AdamState, lrs: dict,
                 timing: dict | None = None) -> float:
    """R/mapper.py:233-264: sample min(K, #kf) keyframes without replacement, shuffle, and run
    one descent step (fwd -> loss -> bwd -> sparse Adam) on each; returns the mean loss.  A
    reference-typed (numpy) map is optimised on a device copy and updated in place at the end."""
    if len(gmap) == 0:
        raise DataError("map not initialized")
    if not isinstance(gmap, GaussianMap):
        dev_map = as_device_map(gmap)
        base = dev_map.rows().clone()
        loss = optimize_map(dev_map, keyframes, cfg, rng, adam, lrs, timing)
        _write_back(gmap, dev_map.rows(), base)
        adam.host = True
        return loss
    m = min(cfg.k_keyframes, len(keyframes))
    order = rng.choice(len(keyframes), size=m, replace=False)
    rng.shuffle(order)
    eng = _engine_for(gmap, keyframes, adam, lrs, cfg)
    eng.loss_sum(reset=True)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    for i in order:
        eng.step(int(i))
    eng.finish()  # every iteration checked (and re-run on an entry-capacity overflow)
    end.record()
    total = eng.loss_sum()
    if timing is not None:
        end.synchronize()
        timing["iter"] = timing.get("iter", 0.0) + start.elapsed_time(end) / 1e3
        timing["steps"] = timing.get("steps", 0) + m
    return total / max(m, 1)


# ---------------------------------------------------------------------------
# map growth (R/mapper.py:69-107, 209-230) -- device versions of the keyframe helpers


def _points_dev(points, device) -> torch.Tensor:
    return torch.as_tensor(points if isinstance(points, torch.Tensor) else np.asarray(points, dtype=np.float32),
                           dtype=torch.float32, device=device).reshape(-1, 3).contiguous()


def _cam_dev(cam, device) -> torch.Tensor:
    c = camera_from(cam)
    return struct_to_device(c.struct(), device)


def _project(points_w, cam, image=None, opacity=None, tau: float = 0.0):
    """gs_project_points: (u, v, ui, vi, z, flags, colors) device tensors."""
    cam = camera_from(cam)
    dev = points_w.device if isinstance(points_w, torch.Tensor) and points_w.is_cuda else default_device()
    pts = _points_dev(points_w, dev)
    m = len(pts)
    u, v, z = (torch.empty(m, device=dev) for _ in range(3))
    ui, vi = (torch.empty(m, dtype=torch.int32, device=dev) for _ in range(2))
    flags = torch.empty(m, dtype=torch.uint8, device=dev)
    img = None if image is None else torch.as_tensor(image, dtype=torch.float32, device=dev).contiguous()
    op = None if opacity is None else torch.as_tensor(opacity, dtype=torch.float32, device=dev).contiguous()
    colors = torch.empty((m, 3), device=dev) if img is not None else None
    camd = _cam_dev(cam, dev)
    call("gs_project_points", pts.data_ptr(), m, camd.data_ptr(), img.data_ptr() if img is not None else None,
         op.data_ptr() if op is not None else None, float(tau), u.data_ptr(), v.data_ptr(), ui.data_ptr(),
         vi.data_ptr(), z.data_ptr(), flags.data_ptr(), colors.data_ptr() if colors is not None else None,
         stream_ptr())
    return u, v, ui, vi, z, flags, colors, pts


def project_points(points_w, cam: Camera):
    """R/mapper.py:69-81 (gs_project_points): pixel coords, depths and an inside-image mask."""
    u, v, ui, vi, z, flags, _, _ = _project(points_w, cam)
    return u, v, ui.long(), vi.long(), z, (flags & 1).bool()


def bilinear_color(image, u, v):
    """R/mapper.py:84-98 through gs_project_points is keyed on points; this helper takes pixel
    coordinates directly (same arithmetic, torch, float64) for API parity."""
    img = torch.as_tensor(image, dtype=torch.float64)
    h, w = img.shape[:2]
    x = torch.clamp(torch.as_tensor(u, dtype=torch.float64, device=img.device), 0.0, w - 1.0)
    y = torch.clamp(torch.as_tensor(v, dtype=torch.float64, device=img.device), 0.0, h - 1.0)
    x0 = torch.clamp(torch.floor(x).long(), 0, max(w - 2, 0))
    y0 = torch.clamp(torch.floor(y).long(), 0, max(h - 2, 0))
    fx, fy = (x - x0)[:, None], (y - y0)[:, None]
    x1, y1 = torch.clamp(x0 + 1, max=w - 1), torch.clamp(y0 + 1, max=h - 1)
    top = img[y0, x0] * (1 - fx) + img[y0, x1] * fx
    bot = img[y1, x0] * (1 - fx) + img[y1, x1] * fx
    return top * (1 - fy) + bot * fy


def zbuffer_project(points_w, cam: Camera) -> torch.Tensor:
    """R/mapper.py:101-107 (gs_zbuffer): dense sparse-depth map, nearest point per pixel, 0 where
    empty -- the supervision the LiDAR K-list is compacted from."""
    cam = camera_from(cam)
    dev = points_w.device if isinstance(points_w, torch.Tensor) and points_w.is_cuda else default_device()
    pts = _points_dev(points_w, dev)
    h, w = int(cam.height), int(cam.width)
    zbuf = torch.empty(h * w, dtype=torch.int32, device=dev)
    depth = torch.empty((h, w), device=dev)
    camd = _cam_dev(cam, dev)
    call("gs_zbuffer", pts.data_ptr(), len(pts), camd.data_ptr(), w, h, zbuf.data_ptr(), depth.data_ptr(),
         stream_ptr())
    return depth


def group_mapping_data(frame_index: int, clouds, image, cam: Camera, cfg: MappingConfig, rng):
    """R/mapper.py:110-131 on the device: z-buffered sparse depth of the merged clouds, random 1-in-
    n_p decimation (host rng, the reference's draw), colours by bilinear lookup of the image."""
    if frame_index % cfg.keyframe_stride != 0:
        return None
    dev = default_device()
    parts = [_points_dev(c, dev) for c in clouds] if clouds else []
    merged = torch.cat(parts) if parts else torch.zeros((0, 3), device=dev)
    sparse = zbuffer_project(merged, cam)
    n = len(merged)
    keep = rng.permutation(n)[:max(n // cfg.n_p, 1 if n else 0)]
    dec = merged[torch.as_tensor(keep, dtype=torch.long, device=dev)]
    img = torch.as_tensor(image, dtype=torch.float32, device=dev)
    _, _, _, _, _, flags, colors, pts = _project(dec, cam, image=img)
    inside = (flags & 1).bool()
    return Keyframe(cam=camera_from(cam), image=img, sparse_depth=sparse, points=pts[inside],
                    colors=colors[inside])


def _init_rows(points, colors, depths, focal: float, device) -> GaussianMap:
    return init_from_points(points, colors, depths, focal, device=device)


def init_map(gmap: GaussianMap, kf: Keyframe) -> int:
    """R/mapper.py:209-215: one Gaussian per keyframe point (depth = camera z)."""
    if len(gmap):
        raise DataError("map already initialized")
    _, _, _, _, z, _, _, pts = _project(kf.points, kf.cam)
    _append(gmap, _init_rows(pts, kf.colors, z, camera_from(kf.cam).fx, pts.device))
    return len(pts)


def expand_map(gmap: GaussianMap, kf: Keyframe, tau: float) -> int:
    """R/mapper.py:218-230: add Gaussians only where the rendered opacity is below tau (the test
    fused into gs_project_points)."""
    if len(gmap) == 0:
        raise DataError("map not initialized")
    opac = forward(gmap, kf.cam).opacity
    _, _, _, _, z, flags, _, pts = _project(kf.points, kf.cam, opacity=opac, tau=tau)
    fresh = (flags & 2).bool()
    nf = int(fresh.sum())
    if nf == 0:
        return 0
    cols = torch.as_tensor(kf.colors, dtype=torch.float32, device=pts.device).reshape(-1, 3)
    _append(gmap, _init_rows(pts[fresh], cols[fresh], z[fresh], camera_from(kf.cam).fx, pts.device))
    return nf


class Mapper:
    """R/mapper.py:267-316: keyframe-driven map owner with copy-on-publish snapshots."""

    def __init__(self, cfg: MappingConfig | None = None, seed: int = 0, device=None):
        self.cfg = cfg or MappingConfig()
        self.seed = seed
        self.gmap = GaussianMap(device=device)
        self.keyframes: list = []
        self.adam = AdamState()
        self.lrs = None
        self.losses: list = []
        self.timing: dict = {}
        self._lock = threading.Lock()
        self._published = self.gmap.snapshot()

    def submit(self, kf: Keyframe) -> int:
        if len(self.gmap) == 0:
            added = init_map(self.gmap, kf)
            pts = kf.points.detach().double().cpu().numpy() if isinstance(kf.points, torch.Tensor) else \
                np.asarray(kf.points, dtype=np.float64)
            pts = pts.reshape(-1, 3)
            extent = float(np.linalg.norm(pts - pts.mean(axis=0), axis=1).max()) if len(pts) else 1.0
            self.lrs = default_lrs(max(extent, 1e-6))
        else:
            added = expand_map(self.gmap, kf, self.cfg.tau)
        self.keyframes.append(kf)
        rng = np.random.default_rng([self.seed, len(self.keyframes)])
        self.losses.append(optimize_map(self.gmap, self.keyframes, self.cfg, rng, self.adam, self.lrs, self.timing))
        with self._lock:
            self._published = self.gmap.snapshot()
        return added

    def refine(self, rounds: int) -> None:
        for k in range(rounds):
            rng = np.random.default_rng([self.seed, 1 << 20, k])
            self.losses.append(optimize_map(self.gmap, self.keyframes, self.cfg, rng, self.adam, self.lrs,
                                            self.timing))
        with self._lock:
            self._published = self.gmap.snapshot()

    def snapshot(self) -> GaussianMap:
        with self._lock:
            return self._published


def mapping_loop(keyframe_queue, mapper: Mapper) -> None:
    """R/mapper.py:319-334: drain a queue of keyframes; None closes it and triggers refinement
    (max(cfg.refine_rounds, 1) rounds).  Calls task_done after each item when the queue supports
    it, so a producer can rendezvous on queue.join()."""
    done = getattr(keyframe_queue, "task_done", lambda: None)
    while True:
        kf = keyframe_queue.get()
        if kf is None:
            done()
            break
        mapper.submit(kf)
        done()
    if mapper.keyframes:
        mapper.refine(max(mapper.cfg.refine_rounds, 1))
