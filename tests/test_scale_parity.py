"""Parity at the BASELINE configurations, on the path the bench times.

One iteration of the graph-captured engine (`MapOptimizer`: lazy tile lists, lazy SH reads, fused
chain rule + sparse Adam -- exactly what bench.py replays) against the float64 oracle iteration
(R/mapper.py:249-256) on the same fp32 parameter rows, at the sizes BASELINE.json names:

* S2r-1M-1280x720-32line (the headline; its first keyframe, 8-bit target as in the bench) and the
  LiDAR density sweep (16 / 64 / 128 lines, Livox-style 5k / 200k rosettes);
* S1-10k-320x240, the configuration the CPU reference runs;
* S2r-2M-1920x1080 forward-only render (images).

Bars (BASELINE.json north_star): images max-abs 1e-4; loss 1e-3 relative; parameter gradients
1e-3 normwise per group -- read off the engine's first Adam moments, m = 0.1 g; touched set exact
(read off the per-Gaussian step counters); the Adam step itself (lr * sign(g) on the first step).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GROUPS = {"pos": (0, 3), "log_scale": (3, 6), "quat": (6, 10), "opacity_logit": (10, 11), "sh_low": (11, 14),
          "sh_high": (14, 59)}


def normwise(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)) if b.size else 0.0


def _scene(kind, n, w, h, lidar, view=0):
    from paper_2507_04004_b200 import scenes
    if kind == "s1":
        return scenes.scene_s1(n, w, h, k_lidar=lidar)
    sc = scenes.scene_room(n, w, h, lidar=lidar, render_views=(view,))
    sc.targets = [np.round(np.clip(t, 0.0, 1.0) * 255.0) / 255.0 for t in sc.targets]  # bench: 8-bit frames
    return sc


def _ocam(c):
    r32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731  (gs_camera is fp32)
    return O.Camera(int(c["width"]), int(c["height"]), float(np.float32(c["fx"])), float(np.float32(c["fy"])),
                    float(np.float32(c["cx"])), float(np.float32(c["cy"])), r32(c["rot_cw"]), r32(c["trans_cw"]))


CASES = [("S2r-1M-1280x720-32line", "room", 1 << 20, 1280, 720, 32),
         # the bench's fourth keyframe: ~2.4k screen-covering Gaussians, more depth-ordered mask
         # words per tile (> 64) than a 64-thread backward CTA has threads
         ("S2r-1M-1280x720-32line-view3", "room3", 1 << 20, 1280, 720, 32),
         ("S1-10k-320x240", "s1", 10000, 320, 240, 5000),
         ("S2r-1M-1280x720-16line", "room", 1 << 20, 1280, 720, 16),
         ("S2r-1M-1280x720-64line", "room", 1 << 20, 1280, 720, 64),
         ("S2r-1M-1280x720-128line", "room", 1 << 20, 1280, 720, 128),
         ("S2r-1M-1280x720-livox5k", "room", 1 << 20, 1280, 720, "rosette:5000"),
         ("S2r-1M-1280x720-livox200k", "room", 1 << 20, 1280, 720, "rosette:200000")]


@pytest.mark.parametrize("name,kind,n,w,h,lidar", CASES, ids=[c[0] for c in CASES])
def test_engine_iteration_matches_oracle(name, kind, n, w, h, lidar):
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = _scene("room" if kind == "room3" else kind, n, w, h, lidar, view=3 if kind == "room3" else 0)
    rows32 = sc.rows.astype(np.float32).astype(np.float64)
    g = GaussianMap.from_rows(sc.rows)
    lrs = R.default_lrs(3.0)
    kf = M.Keyframe(R.camera_from(sc.cams[0]), sc.targets[0], sc.sparse_depths[0])
    eng = M.MapOptimizer(g, [kf], lrs)
    eng.capture()
    eng.step(0)
    torch.cuda.synchronize()
    ref = O.iteration_detail(rows32.copy(), _ocam(sc.cams[0]), sc.targets[0], sc.sparse_depths[0], with_images=True)
    ws = eng.ws
    if kind == "room3":  # the case exists for its many screen-covering Gaussians
        assert int(ws.counters.cpu()[19]) > 2048  # GS_CNT_HUGE_N: > 64 mask words per tile
    # forward images of the timed path (lazy lists) against the float64 blend
    for k, a in (("color", ws.color), ("depth", ws.depth), ("opacity", ws.opacity), ("transmittance", ws.trans)):
        r = ref[k]
        err = float(np.max(np.abs(a.double().cpu().numpy() - r)))
        assert err < 1e-4 * (max(1.0, float(np.abs(r).max())) if k == "depth" else 1.0), (k, err)
    assert abs(float(ws.loss[0].item()) - ref["loss"]) < 1e-3 * abs(ref["loss"])
    # touched = the Gaussians whose step counter advanced (exact)
    t = eng.adam.t[:n].cpu().numpy()
    assert np.array_equal(t > 0, ref["touched"]) and set(np.unique(t)) <= {0, 1}
    # parameter gradients: the first moment is m = 0.1 g (fp32)
    gm = eng.adam.m_rows[:n, :59].double().cpu().numpy() / 0.1
    for k, (a, b) in GROUPS.items():
        err = normwise(gm[:, a:b], ref["grads"][:, a:b])
        assert err < 1e-3, (k, err)
    # the Adam step: lr * sign(g) (first step, R/rasterizer.py:715-725) wherever the gradient is
    # resolved (|g| above 1e-3 of its group's largest); never more than lr anywhere
    delta = g.rows()[:n, :59].double().cpu().numpy() - rows32[:, :59]
    lr = O.lr_columns(lrs)[:59]
    assert np.all(np.abs(delta) <= lr[None, :] * (1 + 1e-3) + 1e-6)
    for k, (a, b) in GROUPS.items():
        gr = ref["grads"][:, a:b]
        sig = np.abs(gr) > 1e-3 * np.abs(gr).max()
        assert np.array_equal(np.sign(delta[:, a:b][sig]), -np.sign(gr[sig])), k


def test_render_2m_1080p_matches_oracle():
    """BASELINE config 4 (forward-only render FPS at 2M Gaussians, 1920x1080): images against the
    float64 blend of the same fp32 rows."""
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = _scene("room", 1 << 21, 1920, 1080, 32)
    g = GaussianMap.from_rows(sc.rows)
    out = R.forward(g, R.camera_from(sc.cams[0]))
    og = O.GaussianMap.from_rows(sc.rows.astype(np.float32).astype(np.float64))
    ref = O.forward(og, _ocam(sc.cams[0]))
    for k in ("color", "depth", "opacity", "transmittance"):
        a, r = getattr(out, k).double().cpu().numpy(), getattr(ref, k)
        err = float(np.max(np.abs(a - r)))
        assert err < 1e-4 * (max(1.0, float(np.abs(r).max())) if k == "depth" else 1.0), (k, err)
    assert np.mean(out.n_contrib.cpu().numpy() != ref.n_contrib) < 1e-5
