#!/usr/bin/env python
"""Benchmark of the Gaussian map-optimisation iteration on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

Default workload (N=1): `S2r-1M-1280x720-32line` -- 1,048,576 Gaussians seeded on the surfaces
of a ray-cast room (SLAM-like, SURVEY.md 8d S2 recipe with this repo's own room generator),
1280x720 keyframes with 32-line LiDAR depth supervision, 4 keyframes cycled.  One step = one
map-optimisation iteration of R/mapper.py:249-256 (forward -> mapping_loss -> backward ->
sparse Adam) with reference semantics (Adam after every keyframe).

N > 1 (torchrun, one rank per GPU, NCCL): a 32-keyframe batch per step split 32/N per GPU over
a replicated map; per-view gradients are accumulated, allreduced with NCCL (touched mask fused
into the same buffer) and one sparse Adam step is applied on every rank.

`--impl reference` times the reference's own CPU algorithm (the float64 C restatement in
oracle/, all host cores) on the same workload and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "map-opt iters/sec (fwd+bwd+Adam) @1M Gaussians 1280x720; render FPS; % HBM roofline"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

CONFIGS = {
    # name: (scene kind, n, width, height, lidar, keyframes, mode)
    "S2r-1M-1280x720-32line": ("room", 1 << 20, 1280, 720, 32, 4, "train"),
    "S2r-500k-1280x720-32line": ("room", 1 << 19, 1280, 720, 32, 4, "train"),
    "S1-1M-1280x720": ("s1", 1 << 20, 1280, 720, 30000, 1, "train"),
    "S1-10k-320x240": ("s1", 10000, 320, 240, 5000, 1, "train"),
    "S2r-2M-1920x1080-render": ("room", 1 << 21, 1920, 1080, 32, 4, "render"),
    # tracking (R/odometry.py:305-336, 30 photometric pose iterations per frame), frames/s
    "S2r-1M-1280x720-track": ("room", 1 << 20, 1280, 720, 32, 1, "track"),
    # BASELINE config 5: LiDAR density sweep at 1M Gaussians, 1280x720
    "S2r-1M-1280x720-16line": ("room", 1 << 20, 1280, 720, 16, 4, "train"),
    "S2r-1M-1280x720-64line": ("room", 1 << 20, 1280, 720, 64, 4, "train"),
    "S2r-1M-1280x720-128line": ("room", 1 << 20, 1280, 720, 128, 4, "train"),
    "S2r-1M-1280x720-livox5k": ("room", 1 << 20, 1280, 720, "rosette:5000", 4, "train"),
    "S2r-1M-1280x720-livox200k": ("room", 1 << 20, 1280, 720, "rosette:200000", 4, "train"),
}
DEFAULT = "S2r-1M-1280x720-32line"
SEGMENT = 100  # iterations per timed segment (the map is restored between segments, untimed)
# share of each phase's time taken by its largest kernel (warm graph-replay ncu list, r01d)
TOP_KERNEL_SHARE = {"preprocess": 0.60, "render_fwd": 0.85, "loss": 0.88, "render_bwd": 0.96, "chain_adam": 1.0}
TOP_KERNEL = {"preprocess": "preprocess_kernel", "render_fwd": "render_fwd_kernel", "loss": "ssim_fwd_kernel + ssim_bwd_kernel",
              "render_bwd": "render_bwd_kernel", "chain_adam": "chain_kernel (fused chain rule + sparse Adam)"}


def peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return dict(PEAKS_FALLBACK), "fallback"


def fp32_peak() -> tuple[float, str]:
    """Measured FP32 issue peak (lane instructions / s) of the FFMA microbenchmark
    (profiles/r02_fp32_peak.json, tools/micro/ffma2.cu); the theoretical figure otherwise."""
    p = os.path.join(ROOT, "profiles", "r02_fp32_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["fp32_lane_instr_per_s"]), "profiles/r02_fp32_peak.json (FFMA microbenchmark)"
    return 148 * 128 * 1.965e9, "theoretical 148 SM x 128 lanes x 1.965 GHz"


def make_scene(name: str, rank: int = 0, world: int = 1, views_override=None):
    from paper_2507_04004_b200 import scenes
    kind, n, w, h, lidar, nkf, mode = CONFIGS[name]
    if kind == "s1":
        return scenes.scene_s1(n, w, h, k_lidar=lidar)
    views = views_override if views_override is not None else tuple(range(0, 32, 32 // nkf))[:nkf]
    sc = scenes.scene_room(n, w, h, lidar=lidar, render_views=views)
    # keyframe images are 8-bit camera frames (the reference loads PNGs, R/io_formats.py:52-57):
    # quantise the ray-traced targets to k / 255
    sc.targets = [np.round(np.clip(t, 0.0, 1.0) * 255.0) / 255.0 for t in sc.targets]
    return sc


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every ~2 ms from a thread (so even a 10 ms region gets samples), nvidia-smi -lms 100 as the
    fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, cuda_index: int):
        self.idx = cuda_index
        self.samples = []  # (sm MHz, reason bitmask)
        self.max_mhz = None
        self.source = None
        self._stop = threading.Event()
        self._go = threading.Event()
        self.t0 = self.t1 = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.idx)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001 -- fall back to the CUDA index
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.idx)

    def _poll(self, nv, h):
        while not self._stop.is_set():
            if self._go.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), int(rs)))
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._mask = {name: getattr(nv, attr) for name, attr in self.REASONS if hasattr(nv, attr)}
            self.source = "nvml, 2 ms polling during the timed region"
            self.thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001 -- no NVML: unsampled
            self.thread = None
        return self

    def start(self) -> None:
        """Mark the start of the timed region (call right before it)."""
        self.t0 = time.perf_counter()
        self._go.set()

    def stop(self) -> None:
        self._go.clear()
        self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        window = None if self.t0 is None or self.t1 is None else round((self.t1 - self.t0) * 1e3, 1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "window_ms": window}
        sm = [s for s, _ in self.samples]
        reasons = sorted({name for _, r in self.samples for name, m in self._mask.items() if r & m})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "window_ms": window, "source": self.source}


# ---------------------------------------------------------------------------
# algorithmic bytes


def algorithmic_bytes(eng, scene_cam) -> dict:
    """Compulsory HBM bytes per launch of each phase, from the iteration's own statistics."""
    import torch
    ws = eng.ws
    n = len(eng.g)
    cnt = ws.counters[:20].cpu().numpy()
    n_t = int(cnt[2])
    E = int(cnt[1])
    huge_n = min(int(cnt[19]), 4096)  # GS_CNT_HUGE_N (capped at GS_HUGE_CAP)
    P = eng.W * eng.H
    nc = ws.n_contrib
    tx, ty = ws.tiles_x, ws.tiles_y
    pad = torch.zeros((ty * 16, tx * 16), dtype=torch.int32, device=nc.device)
    pad[:eng.H, :eng.W] = nc
    tile_max = pad.view(ty, 16, tx, 16).amax(dim=(1, 3))
    proc = int(tile_max.sum().item())  # entries the blend must read (per tile, up to max n_contrib)
    # per-Gaussian statistics from the reference-shaped forward of the same view (the engine's
    # preprocess does not write the records of Gaussians it cannot draw)
    from paper_2507_04004_b200 import rasterizer as R
    full = R.forward(eng.g, eng.views[0].cam).ctx["workspace"]
    near = int((full.splat2d[:, 6] > 0.01).sum().item())
    valid = int(full.valid.sum().item())
    blend = int(full.touched.sum().item())
    K = int(eng.views[0].lidar_z.numel()) if eng.views[0].sparse is not None else 0
    # FP32 work (lane instructions): blend ~17 + 1 MUFU per (entry, pixel) pair
    # forward, ~50 + 2 MUFU backward; SSIM 4 moments x 11 taps x 2 passes + 3 adjoint images x 11
    # x 2 + ~26 for the SSIM map per pixel-channel; preprocess ~300 per Gaussian in front of the
    # camera; chain rule ~900 + Adam 10 per parameter per touched Gaussian
    pairs = int(nc.sum().item())
    fp32 = {"render_fwd": 18 * pairs, "render_bwd": 52 * pairs, "loss": 3 * P * (88 + 66 + 26),
            "preprocess": 300 * near, "chain_adam": n_t * (900 + 10 * 59)}
    return {
        "_fp32": fp32,
        # compulsory bytes of the preprocess: the position of every Gaussian (12 B), the rest of
        # the geometry of those in front of the camera (32 B), the SH tail of the drawable ones
        # (180 B) and their 76-B records (splat 48, rect 16, kept 4, cull bits 8).  (The kernel
        # reads whole 64-B geometry chunks: ncu traffic > this figure by that granularity.)
        "preprocess": 12 * n + 32 * near + 180 * blend + 76 * blend,
        "render_fwd": 52 * proc + 28 * P + 8 * tx * ty,
        "render_bwd": 28 * P + (52 + 40) * proc + 48 * n_t + 8 * tx * ty,
        # fused chain + Adam, SURVEY.md 8d's 1,465 B per touched Gaussian: params, m and v read
        # and written (236 B each way), the screen-space gradients read (40 B), the step counter
        # read and written (the fixed-point rows' 160-B read + 160-B clear are implementation
        # overhead, in "traffic")
        "chain_adam": 1465 * n_t,
        "loss": 36 * P + 8 * P,
        # lazy binning (the engine): per-tile counts read, offsets / flags written (20 B per
        # tile), the screen-covering Gaussians' depth keys sorted (16 B each) and their per-tile
        # bitmaps transposed (read + write).  The small Gaussians' entries are not materialised
        # here: the forward fills the buckets of the tiles that outlive the screen-covering run.
        "bin": 20 * tx * ty + 16 * huge_n + 2 * huge_n * ((tx * ty + 31) // 32) * 4,
        "_stats": {"n": n, "n_valid": valid, "n_touched": n_t, "entries": E, "blend_entries": proc, "pixels": P,
                   "blend_pairs": pairs},
    }


def run_ours(args) -> dict:
    import torch
    import torch.distributed as dist

    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1 or args.batch:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.config
    kind, n_g, W, H, lidar, nkf, mode = CONFIGS[name]
    if world > 1 or args.batch:
        return run_ours_dp(args, rank, world, local)
    sc = make_scene(name)
    g = GaussianMap.from_rows(sc.rows)
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    pk, pk_kind = peaks()
    if mode == "render":
        return run_render(args, g, kfs, pk, pk_kind, name)
    if mode == "track":
        return run_track(args, g, kfs, name)
    lrs = R.default_lrs(3.0)
    eng = M.MapOptimizer(g, kfs, lrs)
    eng.capture()
    nv = len(kfs)
    initial = eng.save_state()

    def timed(block_fn, clk=None):
        """K steps timed with CUDA events in segments of <= SEGMENT iterations; between
        segments (untimed) the map and Adam state are restored to the scene's initial state, so
        the workload is the named scene + < SEGMENT iterations of optimisation whatever K is.
        block_fn(first, count) runs iterations first .. first + count - 1."""
        eng.restore_state(initial)
        block_fn(0, args.warmup)
        eng.restore_state(initial)
        torch.cuda.synchronize()
        total_ms, wall_s, done = 0.0, 0.0, 0
        if clk is not None:
            clk.start()
        while done < args.steps:
            seg = min(SEGMENT, args.steps - done)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s_.record()
            block_fn(done, seg)
            e_.record()
            e_.synchronize()
            wall_s += time.perf_counter() - t0
            total_ms += s_.elapsed_time(e_)
            done += seg
            eng.restore_state(initial)
        if clk is not None:
            clk.stop()
        return total_ms / args.steps, wall_s * 1e3 / args.steps

    def graph_block(first, count):
        for i in range(first, first + count):
            eng.step(i % nv)

    with ClockSampler(local) as clk:
        ms, _ = timed(graph_block, clk)
    value = 1000.0 / ms
    loss = eng.loss_sum() / (args.steps + args.warmup)
    # e2e: host keyframes through the public streaming API (H2D inside the timed region)
    eng.attach_host_keyframes(kfs)
    e2e_ms, wall_ms = timed(lambda first, count: eng.run_host([i % nv for i in range(first, first + count)]))
    # per-phase profile (eager, events between the C-ABI calls) for the roofline
    prof = {p: [] for p in M.MapOptimizer.PHASES}
    for i in range(max(10, min(args.steps, 30))):
        for p, v in eng.profile_step(i % nv).items():
            prof[p].append(v)
    phase_ms = {p: float(np.median(v)) for p, v in prof.items()}
    bytes_ = algorithmic_bytes(eng, kfs[0].cam)
    # the roofline is quoted for the dominant KERNEL: each phase's time times the share of its
    # largest kernel in the warm ncu launch list (profiles/*_graph_launches.md); the fused
    # chain+Adam phase is a single launch
    dom = max((p for p in phase_ms if p != "bin"), key=lambda p: phase_ms[p] * TOP_KERNEL_SHARE.get(p, 1.0))
    dom_all = max(phase_ms, key=lambda p: phase_ms[p])
    hbm = float(pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    f32peak, f32src = fp32_peak()
    achieved = bytes_[dom] / (phase_ms[dom] * 1e-3) / 1e9
    # per phase: both rooflines -- HBM (algorithmic bytes / time vs the measured copy bandwidth)
    # and FP32 issue (algorithmic FP32 lane instructions / time vs the measured FFMA rate)
    phases = {}
    for p in phase_ms:
        sec = phase_ms[p] * 1e-3
        e = {"ms": round(phase_ms[p], 4), "share": round(phase_ms[p] / sum(phase_ms.values()), 4),
             "alg_bytes": int(bytes_[p]), "gbs": round(bytes_[p] / sec / 1e9, 1),
             "hbm_frac": round(bytes_[p] / sec / 1e9 / hbm, 4)}
        if p in bytes_["_fp32"]:
            e["fp32_instr"] = int(bytes_["_fp32"][p])
            e["fp32_frac"] = round(bytes_["_fp32"][p] / sec / f32peak, 4)
        e["bound"] = "fp32" if e.get("fp32_frac", 0.0) > e["hbm_frac"] else "hbm"
        phases[p] = e
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(dom)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "it/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: S2r room scene (seed 7), Gaussians seeded on ray-cast surfaces from 32 views, "
                "targets (8-bit, like camera frames) and LiDAR ray-traced; random-free deterministic generator",
        "config": bench_config(name, nv),
        "notes": {"l2": "inputs larger than L2 (params + Adam moments = 768 MB per step)",
                  "cuda_graph": True, "mean_loss": round(loss, 6),
                  "timing": f"CUDA events over segments of {SEGMENT} iterations; map + Adam state restored "
                            "to the initial scene between segments (untimed)"},
        "e2e": {"value": round(1000.0 / e2e_ms, 2), "unit": "it/s", "h2d_bytes_per_step": int(eng.h2d_bytes),
                "d2h_bytes_per_step": int(eng.d2h_bytes), "wall_ms_per_step": round(wall_ms, 4),
                "path": "MapOptimizer.run_host: pinned host keyframe (8-bit target frame + LiDAR K-list) -> H2D "
                        "on a copy stream, multi-buffered ahead of the iterations, exact fp32 decode on the "
                        "device -> iteration -> D2H loss"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})",
                     "bytes": "SURVEY.md 8d: 1,465 B per touched Gaussian" if dom == "chain_adam" else "DESIGN.md 3",
                     "dominant_phase_overall": dom_all, "kernel_name": TOP_KERNEL.get(dom, dom),
                     "fp32_peak": f32peak, "fp32_peak_source": f32src},
        "phases": phases,
        "stats": bytes_["_stats"],
        "gpu_launches": int(eng.kernels_per_step() * args.steps),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sc, args.cpu_budget)
    return out


def bench_config(name: str, keyframes: int | None = None, batch: int | None = None, world: int = 1) -> dict:
    """The workload description both arms print (ours and --impl reference)."""
    kind, n_g, W, H, lidar, nkf, mode = CONFIGS[name]
    cfg = {"workload": name, "gaussians": int(n_g), "width": W, "height": H, "lidar": lidar,
           "keyframes": int(keyframes if keyframes is not None else nkf), "mode": mode}
    if batch:
        cfg["semantics"] = f"batch-{batch}: gradient sum + touched union + one sparse Adam per batch"
        cfg["parallelism"] = f"dp{world}"
    elif mode == "train":
        cfg["semantics"] = "per-keyframe sparse Adam (R/mapper.py:246-257)"
    return cfg


def run_render(args, g, kfs, pk, pk_kind, name) -> dict:
    """Forward-only novel-view rendering (BASELINE config 4, render FPS)."""
    import torch

    from paper_2507_04004_b200 import _lib
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import stream_ptr
    views = [R.DeviceView(kf.cam) for kf in kfs]
    ws, _ = R._bin_frame(g, views[0], True)
    emax = 0
    for v in views:
        _, cnt = R._bin_frame(g, v, True)
        emax = max(emax, int(cnt[_lib.CNT_ENTRIES]))
    ws = R.Workspace(len(g), kfs[0].cam.width, kfs[0].cam.height, int(emax * 1.3) + 4096, g.device)
    def launch(view_ptr):
        _lib.call("gs_preprocess_ex", ws.fptr, g.data.data_ptr(), view_ptr, _lib.GS_PP_LAZY_SH, stream_ptr())
        _lib.call("gs_bin", ws.fptr, _lib.GS_BIN_LAZY, stream_ptr())
        _lib.call("gs_render_fwd", ws.fptr, 1, stream_ptr())

    launch(views[0].ptr)
    torch.cuda.synchronize()
    graphs = []  # one graph per view (each reads its own device gs_view: no per-frame copy)
    for v in views:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            launch(v.ptr)
        graphs.append(gr)
    for i in range(args.warmup):
        graphs[i % len(views)].replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        clk.start()
        s.record()
        for i in range(args.steps):
            graphs[i % len(views)].replay()
        e.record()
        e.synchronize()
        clk.stop()
    ms = s.elapsed_time(e) / args.steps
    cnt = ws.counters.cpu().numpy()
    stats = {"entries": int(cnt[_lib.CNT_ENTRIES]), "touched": int(cnt[_lib.CNT_TOUCHED]),
             "screen_covering": int(cnt[_lib.GS_CNT_SLOTS + 3]), "pixels": int(ws.width * ws.height)}
    return {"metric": METRIC, "value": round(1000.0 / ms, 2), "unit": "FPS", "stats": stats, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic S2r room scene",
            "config": bench_config(name, len(kfs)),
            "clocks": clk.summary()}


def run_track(args, g, kfs, name) -> dict:
    """Photometric pose refinement (R/odometry.py:305-336): one step = one frame = 30 iterations
    from a perturbed pose against the keyframe image, graph-replayed."""
    import torch

    from paper_2507_04004_b200 import odometry as OD
    from paper_2507_04004_b200.scenes import exp_so3
    kf = kfs[0]
    cam = kf.cam
    rng = np.random.default_rng(5)
    rot0 = exp_so3(0.005 * rng.standard_normal(3)) @ np.asarray(cam.rot_cw)
    t0 = np.asarray(cam.trans_cw) + 0.01 * rng.standard_normal(3)
    ref = OD.PoseRefiner(g, kf.image, cam.with_pose(rot0, t0))
    ref.capture()
    iters = 30

    def frame():
        ref.reset(rot0, t0)
        ref.run(iters)

    for _ in range(args.warmup):
        frame()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        clk.start()
        s.record()
        for _ in range(args.steps):
            frame()
        e.record()
        e.synchronize()
        clk.stop()
    ms = s.elapsed_time(e) / args.steps
    rot, trans, loss = ref.result()
    return {"metric": METRIC, "value": round(1000.0 / ms, 2), "unit": "frames/s (30 pose iterations)",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic S2r room scene", "config": bench_config(name, 1),
            "final_loss": round(loss, 6), "pose_error_m": float(np.linalg.norm(trans - np.asarray(cam.trans_cw))),
            "clocks": clk.summary()}


def run_ours_dp(args, rank, world, local) -> dict:
    """Keyframe-batch data parallelism: 32 views per step, 32/N per rank (each
    rank's view loop one CUDA graph), the touched union compacted on the device, its gradient rows
    allreduced with NCCL in chunks whose sparse Adam steps overlap the remaining chunks' transfer.
    One step = one batch; `value` counts views (map-optimisation iterations) per second of the
    whole job, so N = 1 (`--batch`) and N > 1 are the same unit and semantics."""
    import torch
    import torch.distributed as dist

    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import parallel as PAR
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    batch = 32
    mine = tuple(range(rank, batch, world))
    sc = make_scene(args.config, views_override=mine)
    g = GaussianMap.from_rows(sc.rows)
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    eng = PAR.BatchMapOptimizer(g, kfs, R.default_lrs(3.0))
    ids = list(range(len(kfs)))
    initial = eng.save_state()
    seg = max(1, SEGMENT // batch)  # batches per timed segment (~100 iterations), state restored between

    def timed(step_fn, clk=None):
        eng.restore_state(initial)
        for _ in range(args.warmup):
            step_fn()
        eng.restore_state(initial)
        torch.cuda.synchronize()
        dist.barrier()
        total, done = 0.0, 0
        if clk is not None:
            clk.start()
        while done < args.steps:
            n = min(seg, args.steps - done)
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            dist.barrier()
            s_.record()
            for _ in range(n):
                step_fn()
            e_.record()
            e_.synchronize()
            total += s_.elapsed_time(e_)
            done += n
            eng.restore_state(initial)
        if clk is not None:
            clk.stop()
        ms = torch.tensor([total / args.steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # the job's time is the slowest rank's
        return float(ms.item())

    with ClockSampler(local) as clk:
        ms = timed(lambda: eng.step(ids), clk)
    eng.attach_host_keyframes(kfs)
    e2e_ms = timed(lambda: eng.step_host(ids))
    value = batch * 1000.0 / ms
    out = {"metric": METRIC, "value": round(value, 2), "unit": "it/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic S2r room scene (seed 7)",
           "config": bench_config(args.config, batch, batch=batch, world=world),
           "notes": {"per_rank_views": len(mine), "union_rows_last_batch": eng.union,
                     "reduction": "single rank: device compaction of the touched union, one sparse Adam straight "
                                  "from the accumulated gradient rows" if world == 1 else
                                  ("touched OR (n bytes) + device compaction + one kernel per rank: reduce-scatter "
                                   "of the union's rows over peer memory (CUDA IPC, NVLink) fused with the all-gather "
                                   "and the sparse Adam (gs_p2p_reduce_adam)") if eng.p2p is not None else
                                  ("touched OR (n bytes) + device compaction + NCCL allreduce of the union's "
                                   f"rows in {PAR.BatchMapOptimizer.CHUNKS} chunks, Adam per chunk"),
                     "timing": f"segments of {seg} batches, map + Adam state restored between (untimed); "
                               "max over ranks"},
           "e2e": {"value": round(batch * 1000.0 / e2e_ms, 2), "unit": "it/s",
                   "h2d_bytes_per_step": int(eng.h2d_bytes_per_view * len(ids) * world), "d2h_bytes_per_step": 8 * world,
                   "path": "BatchMapOptimizer.step_host: pinned host keyframes streamed per view (copy stream, "
                           "multi-buffered) -> accumulate -> allreduce -> Adam -> D2H batch loss"},
           "gpu_launches": int(eng.kernels_per_step() * args.steps), "clocks": clk.summary()}
    dist.barrier()
    return out


def run_plumbing(args) -> dict:
    """GSLIC_BENCH_PLUMBING=1 (tests/test_bench_launch.py, CPU): the multi-rank launch path of
    this script -- self-spawn through torchrun, rendezvous on 127.0.0.1, barrier-bracketed timing,
    max over ranks, one JSON line from rank 0 -- with a gloo allreduce of gradient rows standing
    in for the GPU step.  Never a benchmark number."""
    import torch
    import torch.distributed as dist

    from paper_2507_04004_b200 import parallel as PAR
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dist.init_process_group("gloo")
    n = 4096
    gen = torch.Generator().manual_seed(rank)
    base = torch.randn(n, 64, generator=gen)
    flags = (torch.rand(n, generator=gen) < 0.3).to(torch.uint8)

    def step():
        PAR.allreduce_grads_sparse(base.clone(), flags.clone())

    for _ in range(args.warmup):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dist.barrier()
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / args.steps])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    union = flags.clone()
    dist.all_reduce(union, op=dist.ReduceOp.MAX)
    out = {"metric": METRIC, "value": None, "unit": "it/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(float(ms.item()), 4), "plumbing": True,
           "union_rows": int(union.sum().item()), "config": bench_config(args.config, 32, batch=32, world=world)}
    dist.barrier()
    dist.destroy_process_group()
    return out


def cpu_baseline(sc, budget_s: float) -> dict:
    """The oracle (float64 C restatement of the reference, all host cores) on a bounded sample:
    as many full iterations of the same workload as fit the budget (>= 1 after a warm-up)."""
    import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    rows = sc.rows.astype(np.float32).astype(np.float64)
    st = O.AdamState()
    lrs = O.default_lrs(3.0)
    c = sc.cams[0]
    cam = O.Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"], c["trans_cw"])
    O.map_iteration_rows(rows, cam, sc.targets[0], sc.sparse_depths[0], st, lrs)  # warm-up
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        O.map_iteration_rows(rows, cam, sc.targets[0], sc.sparse_depths[0], st, lrs)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all + times[-1] > budget_s or len(times) >= 10:
            break
    med = float(np.median(times))
    return {"value": round(1.0 / med, 4), "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{len(times)} full iterations (after 1 warm-up) of the same workload, median "
                      f"{med:.3f} s/iter, oracle/gs_oracle.c float64 with {threads} OpenMP threads"}


def run_reference(args) -> dict | None:
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if rank != 0:
        return None
    sc = make_scene(args.config)
    import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    rows = sc.rows.astype(np.float32).astype(np.float64)
    st = O.AdamState()
    lrs = O.default_lrs(3.0)
    cams = [O.Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"], c["trans_cw"])
            for c in sc.cams]
    nv = len(cams)
    budget = float(args.ref_budget)
    kind, n_g, W, H, lidar, nkf, mode = CONFIGS[args.config]
    g = O.GaussianMap.from_rows(rows)

    def one(i):  # one step of the reference algorithm for this config's mode
        k = i % nv
        if mode == "render":  # R/rasterizer.py:442 forward only
            O.forward(g, cams[k])
        elif mode == "track":  # R/odometry.py:305-336: 30 x (forward, tracking loss, pose backward)
            for _ in range(30):
                out = O.forward(g, cams[k])
                _, gc = O.photometric_loss(out.color, sc.targets[k], 0.5)
                O.backward(g, out, gc, with_pose=True)
        else:  # R/mapper.py:249-256
            O.map_iteration_rows(rows, cams[k], sc.targets[k], sc.sparse_depths[k], st, lrs)

    unit = {"render": "FPS", "track": "frames/s (30 pose iterations)"}.get(mode, "it/s")
    t_start = time.perf_counter()
    warm = 0
    for i in range(args.warmup):
        one(i)
        warm += 1
        if time.perf_counter() - t_start > budget / 3:
            break
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        one(i)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget:
            break
    ms = 1e3 * float(np.mean(times))
    value = 1000.0 / ms
    return {"metric": METRIC, "value": round(value, 4), "unit": unit, "n_gpus": args.gpus, "steps": len(times),
            "warmup": warm, "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic S2r room scene (seed 7), same generator as the GPU arm",
            "config": bench_config(args.config, 32 if args.gpus > 1 or args.batch else None,
                                   batch=32 if args.gpus > 1 or args.batch else None, world=args.gpus),
            "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": threads, "kind": "port",
                             "sample": f"{len(times)} full steps (capped by a {budget:.0f} s budget) of the "
                                       f"workload; oracle/gs_oracle.c float64, {threads} OpenMP threads"},
            "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=DEFAULT)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", action="store_true",
                    help="N=1 run of the multi-GPU semantics (32-keyframe batch, one Adam per batch)")
    ap.add_argument("--cpu-budget", type=float, default=25.0)
    ap.add_argument("--ref-budget", type=float, default=150.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # N GPUs requested without a launcher: become torchrun with one rank per GPU (rank 0
        # prints the JSON line; rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    # stdout carries exactly one JSON line: everything else the process (or a library -- NCCL
    # prints its version banner to stdout on communicator set-up) writes to fd 1 goes to stderr
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    plumbing = os.environ.get("GSLIC_BENCH_PLUMBING") == "1"
    if args.impl == "reference":
        out = run_reference(args)
    elif plumbing:
        out = run_plumbing(args)
    else:
        out = run_ours(args)
    if out is not None and int(os.environ.get("RANK", 0)) == 0:
        json_out.write(json.dumps(out) + "\n")
        json_out.flush()
    if (int(os.environ.get("WORLD_SIZE", 1)) > 1 or args.batch) and args.impl == "ours" and not plumbing:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
