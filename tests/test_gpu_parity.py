"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the reference's
golden vectors.

Bars (BASELINE.json north_star):
  * bit-exact: tile keys / sort order (entry_splat), tile ranges, touched mask -- against the
    fp32 CPU restatement fed the GPU's own fp32 2D splats (oracle.bin_f32);
  * rendered RGB / depth / alpha: max-abs 1e-4 against the float64 reference;
  * loss and parameter gradients: 1e-3 relative (norm-wise per parameter group).
"""
import glob
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SCENES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz"))
                if "entry_splat" in np.load(p).files)  # the forward/backward scenes
GROUPS = {"pos": (0, 3), "log_scale": (3, 6), "quat": (6, 10), "opacity_logit": (10, 11), "sh_low": (11, 14),
          "sh_high": (14, 59)}
IMG_TOL = 1e-4
REL_TOL = 1e-3
G2D_TOL = REL_TOL  # screen-space (intermediate) gradients: the same 1e-3 bar


def _np(t):
    return t.detach().double().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def normwise(a, b, floor=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), floor)) if b.size else 0.0


def load(name):
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    z = np.load(os.path.join(GOLD, name + ".npz"))
    cam = R.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    return z, cam, GaussianMap.from_rows(z["rows"])


def gpu_splats(out):
    p = out.ctx["proj"]
    return (_np(p["mean2d"]).astype(np.float32), _np(p["conic"]).astype(np.float32),
            _np(p["cov2d"]).reshape(-1, 4)[:, [0, 1, 3]].astype(np.float32), _np(out.ctx["opac"]).astype(np.float32),
            _np(p["depth"]).astype(np.float32), _np(p["valid"]).astype(bool))


@pytest.mark.parametrize("name", SCENES)
def test_binning_bit_exact_vs_fp32_oracle(name):
    from paper_2507_04004_b200 import rasterizer as R
    z, cam, g = load(name)
    for cull in (True, False):
        out = R.forward(g, cam, cull=cull)
        m, c, cv, o, d, v = gpu_splats(out)
        ent, offs, touched = O.bin_f32(m, c, cv, o, d, v, cam.width, cam.height, cull)
        assert np.array_equal(_np(out.ctx["entry_splat"]).astype(np.int64), ent.astype(np.int64))
        assert np.array_equal(_np(out.ctx["tile_offsets"]).astype(np.int64), offs.astype(np.int64))
        if cull:
            ws = out.ctx["workspace"]
            assert np.array_equal(_np(ws.touched).astype(bool), touched)


@pytest.mark.parametrize("name", SCENES)
def test_forward_matches_reference(name):
    from paper_2507_04004_b200 import rasterizer as R
    z, cam, g = load(name)
    out = R.forward(g, cam)
    # tile lists equal the float64 reference's (no near-threshold pair in these scenes)
    assert np.array_equal(_np(out.ctx["entry_splat"]).astype(np.int64), z["entry_splat"])
    assert np.array_equal(_np(out.ctx["tile_offsets"]).astype(np.int64), z["tile_offsets"])
    for k, ref in (("color", z["color"]), ("depth", z["depth"]), ("opacity", z["opacity"]),
                   ("transmittance", z["transmittance"])):
        err = np.max(np.abs(_np(getattr(out, k)) - ref))
        assert err < IMG_TOL * max(1.0, float(np.abs(ref).max()) if k == "depth" else 1.0), (k, err)
    assert np.array_equal(_np(out.n_contrib), z["n_contrib"])
    assert np.array_equal(_np(out.ctx["proj"]["valid"]).astype(bool), z["valid"])
    # mean2d of every valid Gaussian against the oracle projection of the same fp32 parameters
    # and fp32 camera (the device's map and gs_camera are fp32; just past the 0.01 m clip plane
    # fx / z ~ 1e5 turns their 6e-8 rounding into ~1e-5 relative, so the float64 golden is the
    # bar beyond 0.1 m)
    vm = z["valid"]
    r32 = lambda a: np.asarray(a).astype(np.float32).astype(np.float64)  # noqa: E731
    oproj = O.project(O.GaussianMap.from_rows(r32(z["rows"])), r32(z["rot_cw"]), r32(z["trans_cw"]),
                      tuple(float(np.float32(z[k])) for k in ("fx", "fy", "cx", "cy")))
    m32 = oproj["mean2d"][vm]
    assert np.max(np.abs(_np(out.ctx["proj"]["mean2d"])[vm] - m32) / np.maximum(1.0, np.abs(m32))) < 1e-6
    far = z["valid"] & (z["pdepth"] > 0.1)
    mref = z["mean2d"][far]
    assert np.max(np.abs(_np(out.ctx["proj"]["mean2d"])[far] - mref) / np.maximum(1.0, np.abs(mref))) < 1e-5
    nearv = z["pdepth"] > 0.01  # colours of Gaussians behind the camera are never used
    assert normwise(_np(out.ctx["colors"])[nearv], z["colors"][nearv]) < 1e-5
    full = R.forward(g, cam, cull=False)
    assert np.max(np.abs(_np(full.color) - z["full_color"])) < IMG_TOL


@pytest.mark.parametrize("name", SCENES)
def test_loss_and_gradients_match_reference(name):
    from paper_2507_04004_b200 import losses as L
    from paper_2507_04004_b200 import rasterizer as R
    z, cam, g = load(name)
    out = R.forward(g, cam)
    loss, gc, gd, go = L.mapping_loss(out.color, out.depth, out.opacity, z["target"], z["sparse_depth"],
                                      float(z["lam"]), float(z["xi"]))
    assert abs(loss - float(z["loss"])) < REL_TOL * abs(float(z["loss"]))
    assert normwise(_np(gc), z["g_color"]) < REL_TOL
    assert normwise(_np(gd), z["g_depth"]) < REL_TOL
    assert normwise(_np(go), z["g_opac"]) < REL_TOL
    # screen-space gradients from the reference's own image gradients
    g2d = R.backward_2d(out, z["g_color"], z["g_depth"], z["g_opac"])
    for k, a in zip(("mean2d", "conic", "op", "color", "depth"), g2d[:5]):
        assert normwise(_np(a), z["g2d_" + k]) < G2D_TOL, k
    assert np.array_equal(_np(g2d[5]).astype(bool), z["touched"])
    rng = np.random.default_rng(99)
    rgc = rng.standard_normal(z["color"].shape)
    rgd = rng.standard_normal(z["depth"].shape)
    rgo = rng.standard_normal(z["opacity"].shape)
    r2d = R.backward_2d(out, rgc, rgd, rgo)
    for k, a in zip(("mean2d", "conic", "op", "color", "depth"), r2d[:5]):
        assert normwise(_np(a), z["r2d_" + k]) < G2D_TOL, k
    grads, touched, _ = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
    assert np.array_equal(_np(touched).astype(bool), z["touched"])
    gr = _np(grads["_rows"])[:, :59]
    # every Gaussian, including those just past the 0.01 m clip plane (room4096: 1,818 of 4,096
    # within 5 cm, whose mean and conic paths cancel ~1e4-fold in the chain rule; the factored
    # conic record and the FP64 geometric reduction keep them at ~1e-4)
    for k, (a, b) in GROUPS.items():
        err = normwise(gr[:, a:b], z["grads"][:, a:b])
        assert err < REL_TOL, (k, err)


def test_losses_match_reference_golden():
    from paper_2507_04004_b200 import losses as L
    z = np.load(os.path.join(GOLD, "losses.npz"))
    v, g = L.photometric_loss(z["a"], z["b"], 0.2)
    assert abs(v - float(z["val"])) < 1e-5 * abs(float(z["val"]))
    assert normwise(_np(g), z["grad"]) < REL_TOL
    dv, dg = L.dssim_and_grad(z["a"], z["b"])
    assert abs(dv - float(z["dval"])) < 1e-5
    assert normwise(_np(dg), z["dgrad"]) < REL_TOL
    for pre in ("t", "o"):  # 3x5 and 1x7 images: multi-bounce mirror padding
        a = z["tiny_a"] if pre == "t" else z["one_a"]
        b = z["tiny_b"] if pre == "t" else z["one_b"]
        v, g = L.photometric_loss(a, b, 0.2)
        assert abs(v - float(z[pre + "val"])) < 1e-5
        assert normwise(_np(g), z[pre + "grad"]) < REL_TOL
    v, gd, go = L.depth_ratio_loss(z["depth"], z["opac"], z["sparse"])
    assert abs(v - float(z["dv"])) < REL_TOL * abs(float(z["dv"]))
    assert normwise(_np(gd), z["dgd"]) < REL_TOL
    assert normwise(_np(go), z["dgo"]) < REL_TOL
    # known answers (T/test_losses.py:105-166)
    depth = np.zeros((4, 4)); opac = np.zeros((4, 4)); sparse = np.zeros((4, 4))
    depth[1, 2], opac[1, 2], sparse[1, 2] = 1.5, 0.5, 2.0
    v, gd, go = L.depth_ratio_loss(depth, opac, sparse)
    assert abs(v - 1.0) < 1e-6
    assert np.count_nonzero(_np(gd)) == 1
    v, gd, go = L.depth_ratio_loss(np.ones((3, 3)), np.zeros((3, 3)), np.ones((3, 3)))
    assert np.isfinite(v) and not _np(go).any()


def test_adam_matches_oracle_and_reference_semantics():
    import torch
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    rng = np.random.default_rng(3)
    rows = rng.standard_normal((12, 59))
    g = GaussianMap.from_rows(rows)
    st = R.AdamState()
    lrs = R.default_lrs(2.0)
    orows = rows.astype(np.float32).astype(np.float64)
    ost = O.AdamState()
    touched = np.array([True, False, True, True, False, True, True, True, False, True, True, True])
    for _ in range(5):
        gr = rng.standard_normal((12, 59)).astype(np.float32)
        grows = torch.zeros((12, 64), device="cuda")
        grows[:, :59] = torch.as_tensor(gr, device="cuda")
        before = g.rows().clone()
        R.sparse_adam_step(g, R.rows_to_grads(grows), touched, st, lrs)
        O.adam_rows(orows, gr.astype(np.float64), touched, ost, lrs)
        after = g.rows()
        assert torch.equal(after[~torch.as_tensor(touched, device="cuda")],
                           before[~torch.as_tensor(touched, device="cuda")])
    assert normwise(_np(g.rows())[:, :59] - rows, orows - rows) < 1e-4
    assert np.array_equal(_np(st.t).astype(np.int64), ost.t)
    # first step magnitude = lr (T/test_rasterizer.py:350-359)
    g1 = GaussianMap.from_rows(np.zeros((1, 59)))  # p = 0 so p - lr is exact in fp32
    s1 = R.AdamState()
    b = g1.rows().clone()
    ones = torch.zeros((1, 64), device="cuda")
    ones[:, :59] = 1.0
    R.sparse_adam_step(g1, R.rows_to_grads(ones), np.array([True]), s1, R.default_lrs(1.0))
    step = _np(b - g1.rows())[0, :59]
    assert np.allclose(step, O.lr_columns(R.default_lrs(1.0)), rtol=1e-6)


def test_render_known_answers():
    import torch
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    # single splat identity (T/test_rasterizer.py:91-104)
    sc = scenes.make_scene(11, n=1, max_op=0.6)
    cam = R.camera_from(sc.cams[0])
    out = R.forward(GaussianMap.from_rows(sc.rows), cam)
    m = _np(out.ctx["proj"]["mean2d"])[0]
    cn = _np(out.ctx["proj"]["conic"])[0]
    op = _np(out.ctx["opac"])[0]
    col = _np(out.ctx["colors"])[0]
    px, py = int(round(m[0])), int(round(m[1]))
    d = np.array([px, py]) - m
    q = cn[0] * d[0] ** 2 + 2 * cn[1] * d[0] * d[1] + cn[2] * d[1] ** 2
    alpha = min(op * np.exp(-0.5 * q), 0.99)
    assert np.allclose(_np(out.color)[py, px], alpha * col, atol=1e-6)
    assert abs(_np(out.opacity)[py, px] - alpha) < 1e-6
    # empty map renders background
    empty = GaussianMap.from_rows(np.zeros((0, 59)))
    out = R.forward(empty, cam)
    assert not _np(out.color).any() and not _np(out.opacity).any()
    # energy conservation and permutation invariance (bit-identical) and determinism
    for seed in range(3):
        sc = scenes.make_scene(seed, n=120, max_op=0.97)
        cam = R.camera_from(sc.cams[0])
        g = GaussianMap.from_rows(sc.rows)
        out = R.forward(g, cam)
        o = _np(out.opacity)
        assert np.all(o >= 0) and np.all(o <= 1)
        assert np.allclose(o + _np(out.transmittance), 1.0, atol=1e-6)
        perm = np.random.default_rng(5).permutation(120)
        out2 = R.forward(GaussianMap.from_rows(sc.rows[perm]), cam)
        assert torch.equal(out.color, out2.color) and torch.equal(out.depth, out2.depth)
        out3 = R.forward(g, cam)
        assert torch.equal(out.color, out3.color)
    # splats below 1/255 opacity are culled everywhere (T/test_rasterizer.py:182-187)
    sc = scenes.make_scene(19, n=10)
    sc.rows[:, 10] = np.log((1 / 300) / (1 - 1 / 300))
    out = R.forward(GaussianMap.from_rows(sc.rows), R.camera_from(sc.cams[0]))
    assert out.ctx["entry_splat"].numel() == 0 and not _np(out.color).any()


def test_cull_matches_bruteforce():
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.make_scene(17, n=80, width=64, height=48, max_op=0.97)
    cam = R.camera_from(sc.cams[0])
    out = R.forward(GaussianMap.from_rows(sc.rows), cam)
    m, c, cv, o, d, v = gpu_splats(out)
    got = set()
    ent, offs = _np(out.ctx["entry_splat"]).astype(int), _np(out.ctx["tile_offsets"]).astype(int)
    for t in range(len(offs) - 1):
        for e in range(offs[t], offs[t + 1]):
            got.add((int(ent[e]), t))
    tiles_x = (cam.width + 15) // 16
    want = set()
    for gi in np.flatnonzero(v):
        for ty in range((cam.height + 15) // 16):
            for tx in range(tiles_x):
                ys, xs = np.mgrid[ty * 16:min(ty * 16 + 16, cam.height), tx * 16:min(tx * 16 + 16, cam.width)]
                dx, dy = xs - float(m[gi, 0]), ys - float(m[gi, 1])
                qq = c[gi, 0] * dx * dx + 2 * c[gi, 1] * dx * dy + c[gi, 2] * dy * dy
                if np.max(np.minimum(o[gi] * np.exp(-0.5 * qq), 0.99)) >= 1.0 / 255.0:
                    want.add((int(gi), ty * tiles_x + tx))
    assert got == want


def test_mapping_iterations_match_oracle():
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(4096, 128, 72, lidar=16, render_views=(0, 1, 2))
    g = GaussianMap.from_rows(sc.rows)
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    lrs = R.default_lrs(3.0)
    eng = M.MapOptimizer(g, kfs, lrs)
    og = O.GaussianMap.from_rows(sc.rows.astype(np.float32).astype(np.float64))
    ost = O.AdamState()
    ocams = [O.Camera(**{k: c[k] for k in ("width", "height", "fx", "fy", "cx", "cy", "rot_cw", "trans_cw")})
             for c in sc.cams]
    for it in range(6):
        k = it % 3
        eng.step(k)
        gl = eng.loss_sum()
        ol = O.map_iteration(og, ocams[k], sc.targets[k], sc.sparse_depths[k], ost, lrs)
        assert abs(gl - ol) < REL_TOL * abs(ol), (it, gl, ol)
        # the engine keeps the depth / opacity gradient images zero between iterations (the
        # backward clears the LiDAR pixels the loss wrote: GS_BWD_CLEAR_DEPTH_GRADS)
        assert not bool(eng.ws.g_depth.any()) and not bool(eng.ws.g_opac.any()), it
    delta_gpu = _np(g.rows())[:, :59] - sc.rows
    delta_ref = og.rows() - sc.rows
    assert normwise(delta_gpu, delta_ref) < REL_TOL
    # graph-captured replay runs the same iteration
    eng.capture()
    eng.step(0)
    assert np.isfinite(eng.loss_sum())


@pytest.mark.parametrize("n,w,h", [(1 << 20, 1280, 720), (1 << 21, 1920, 1080)])
def test_full_size_properties(n, w, h):
    """S2r at BASELINE sizes (1M Gaussians at 1280x720; 2M at 1920x1080, the render-FPS config):
    bit-exact binning against the fp32 oracle, O + T = 1, touched == ids present in the entry
    list."""
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(n, w, h, lidar=32)
    cam = R.camera_from(sc.cams[0])
    g = GaussianMap.from_rows(sc.rows)
    out = R.forward(g, cam)
    m, c, cv, o, d, v = gpu_splats(out)
    ent, offs, touched = O.bin_f32(m, c, cv, o, d, v, cam.width, cam.height, True)
    assert np.array_equal(_np(out.ctx["entry_splat"]).astype(np.int64), ent.astype(np.int64))
    assert np.array_equal(_np(out.ctx["tile_offsets"]).astype(np.int64), offs.astype(np.int64))
    tg = _np(out.ctx["workspace"].touched).astype(bool)
    assert np.array_equal(tg, touched)
    present = np.zeros(len(tg), bool)
    present[ent] = True
    assert np.array_equal(present, tg)
    assert np.allclose(_np(out.opacity) + _np(out.transmittance), 1.0, atol=1e-6)
    nc = _np(out.n_contrib)
    counts = np.diff(offs)
    tiles_x = (cam.width + 15) // 16
    ty, tx = np.mgrid[0:cam.height, 0:cam.width] // 16
    assert np.all(nc <= counts[ty * tiles_x + tx])
    # g2d rows are indexed by touched slot: slot(touched_list[k]) == k for every k < nt, both for
    # the reference-shaped path and the engine's (lazy lists, large-footprint publishes)
    for ws in (out.ctx["workspace"], _lazy_forward(g, cam)):
        _check_touched_slots(ws)


def _check_touched_slots(ws):
    import torch
    from paper_2507_04004_b200 import _lib
    nt = int(ws.counters[_lib.CNT_TOUCHED].item())
    tl = ws.view("touched_list", "i32", (max(ws.n, 1),))[:nt].long()
    assert nt > 0 and len(torch.unique(tl)) == nt
    slot = ws.splat2d[:, 14].contiguous().view(torch.int32).long()
    assert torch.equal(slot[tl], torch.arange(nt, device=tl.device))


def _lazy_forward(g, cam):
    """The engine's binning (gs_bin(GS_BIN_LAZY): lists materialised on demand) + forward."""
    import torch
    from paper_2507_04004_b200 import _lib
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import stream_ptr
    view = R.DeviceView(cam, device=g.device)
    ws, _ = R._bin_frame(g, view, True)  # sizes the workspace
    _lib.call("gs_preprocess_ex", ws.fptr, g.data.data_ptr(), view.ptr, _lib.GS_PP_LAZY_SH, stream_ptr())
    _lib.call("gs_bin", ws.fptr, _lib.GS_BIN_LAZY, stream_ptr())
    _lib.call("gs_render_fwd", ws.fptr, 1, stream_ptr())
    torch.cuda.synchronize()
    return ws


def _interleaved_scene():
    """Screen-covering Gaussians behind and in front of small ones: the lazy lists must merge."""
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_s1(4000, 640, 480, k_lidar=500)
    rows = sc.rows.copy()
    cam = R.camera_from(sc.cams[0])
    rng = np.random.default_rng(5)
    k = 40
    big = rows[rng.choice(len(rows), k, replace=False)].copy()
    big[:, 3:6] += np.log(80.0)  # 80x larger: hundreds of candidate tiles each
    big[:, 10] = -2.0            # faint, so the blend does not stop on them
    return GaussianMap.from_rows(np.concatenate([rows, big])), cam


@pytest.mark.parametrize("which", ["room", "interleaved"])
def test_lazy_lists_match_materialised(which):
    """gs_bin(GS_BIN_LAZY) + forward + backward == the materialised lists, bit for bit."""
    import torch
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    if which == "room":
        sc = scenes.scene_room(1 << 17, 640, 360, lidar=16)
        g, cam = GaussianMap.from_rows(sc.rows), R.camera_from(sc.cams[0])
    else:
        g, cam = _interleaved_scene()
    out = R.forward(g, cam)
    ref = [t.clone() for t in (out.color, out.depth, out.opacity, out.transmittance, out.n_contrib)]
    ws = _lazy_forward(g, cam)
    got = (ws.color, ws.depth, ws.opacity, ws.trans, ws.n_contrib)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
    cnt = ws.counters.cpu().numpy()
    T = ws.tiles_x * ws.tiles_y
    flags = ws.view("tile_scratch", "i32", (5 * (T + 1),))[3 * (T + 1):4 * (T + 1) - 1].cpu().numpy()
    if which == "interleaved":
        assert cnt[16 + 3] > 0  # screen-covering Gaussians present
        assert (flags == 1).any()  # some tile's bucket interleaves with them: merged list
    # the backward over the lazy lists matches the materialised lists' bit for bit
    rng = np.random.default_rng(0)
    h, w = int(cam.height), int(cam.width)
    gc = torch.as_tensor(rng.standard_normal((h, w, 3)), dtype=torch.float32, device="cuda")
    gd = torch.as_tensor(rng.standard_normal((h, w)), dtype=torch.float32, device="cuda")
    go = torch.as_tensor(rng.standard_normal((h, w)), dtype=torch.float32, device="cuda")
    ref2d = R.backward_2d(out, gc, gd, go)
    from paper_2507_04004_b200 import _lib
    from paper_2507_04004_b200.gaussians import stream_ptr
    ws.g_color.copy_(gc)
    ws.g_depth.copy_(gd)
    ws.g_opac.copy_(go)
    _lib.call("gs_render_bwd", ws.fptr, stream_ptr())
    torch.cuda.synchronize()
    g2d = ws.g2d.cpu().numpy()
    touched = ws.touched.bool().cpu().numpy()
    for k, ref in enumerate(ref2d[:5]):
        cols = {0: [0, 1], 1: [2, 3, 4], 2: [5], 3: [6, 7, 8], 4: [9]}[k]
        a = _np(ref).reshape(len(touched), -1)[touched]
        b = g2d[touched][:, cols].reshape(a.shape)
        assert np.array_equal(b, a), k


@pytest.mark.parametrize("name", SCENES)
def test_pose_gradient_matches_reference(name):
    """backward(with_pose=True) through gs_chain_pose: the 6-dof pose gradient of
    R/rasterizer.py:646-657 (golden from the reference), attribute gradients unchanged, and the
    tracker's pose-only call (grads not materialised) agrees bit for bit."""
    import torch
    from paper_2507_04004_b200 import rasterizer as R
    p = np.load(os.path.join(GOLD, "pose.npz"))
    z, cam, g = load(name)
    out = R.forward(g, cam)
    grads, touched, pose = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"], with_pose=True)
    # the pose chain itself, isolated from the blend: the oracle fed the screen-space gradients
    # this very backward accumulated (still in the workspace) and the fp32 parameters
    ws = out.ctx["workspace"]
    g2 = _np(ws.g2d)[:, :10]
    ocam = O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, np.asarray(cam.rot_cw, np.float32),
                    np.asarray(cam.trans_cw, np.float32))
    _, opose = O.chain(z["rows"].astype(np.float32).astype(np.float64), ocam, g2, _np(touched).astype(bool),
                       with_pose=True)
    assert normwise(_np(pose), opose) < 1e-4, (_np(pose), opose)
    ref = p[f"{name}_pose"]
    assert normwise(_np(pose), ref) < REL_TOL, (_np(pose), ref)
    assert np.array_equal(_np(touched).astype(bool), z["touched"])
    # bit-identical run to run (fixed-point accumulation; T/test_rasterizer.py:153-162)
    g1, _, pose1 = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"], with_pose=True)
    assert torch.equal(g1["_rows"], grads["_rows"]) and torch.equal(pose1, pose)
    only = R.pose_backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
    assert torch.equal(only, pose)
    # without the pose: the same screen-space gradients through the non-pose chain instantiation
    # (its FP64 chain is compiled separately, so rounding may differ in the last bits)
    g0, _, none = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
    assert none is None
    assert normwise(_np(g0["_rows"]), _np(grads["_rows"])) < 1e-6


@pytest.mark.parametrize("seed", [0, 1])
def test_pose_gradient_fd_scenes(seed):
    """The reference's finite-difference scenes (T/test_rasterizer.py:261-280): cull=False,
    early_stop=False, random image weights."""
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    p = np.load(os.path.join(GOLD, "pose.npz"))
    key = f"fd{seed}"
    c = p[f"{key}_cam"]
    cam = R.Camera(int(c[0]), int(c[1]), float(c[2]), float(c[3]), float(c[4]), float(c[5]), p[f"{key}_rot"],
                   p[f"{key}_trans"])
    g = GaussianMap.from_rows(p[f"{key}_rows"])
    out = R.forward(g, cam, cull=False, early_stop=False)
    grads, _, pose = R.backward(g, out, p[f"{key}_wc"], p[f"{key}_wd"], p[f"{key}_wo"], with_pose=True)
    assert normwise(_np(pose), p[f"{key}_pose"]) < REL_TOL
    assert normwise(_np(grads["_rows"])[:, :59], p[f"{key}_grads"]) < REL_TOL


@pytest.mark.parametrize("frames", ["float", "8bit"])
def test_host_streaming_matches_device_keyframes(frames):
    """MapOptimizer.run_host (pinned host keyframes, K-list compacted on the host, H2D multi-
    buffered on a copy stream; 8-bit frames decoded on the device) runs the same iterations as
    device-resident keyframes."""
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(8192, 160, 96, lidar=16, render_views=(0, 1, 2))
    if frames == "8bit":
        sc.targets = [np.round(np.clip(t, 0, 1) * 255.0) / 255.0 for t in sc.targets]
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    order = [0, 2, 1, 1, 0, 2, 2]
    a = M.MapOptimizer(GaussianMap.from_rows(sc.rows), kfs, R.default_lrs(3.0))
    a.capture()
    la = []
    for k in order:
        a.step(k)
        la.append(a.loss_sum())
    b = M.MapOptimizer(GaussianMap.from_rows(sc.rows), kfs, R.default_lrs(3.0))
    b.capture()
    b.attach_host_keyframes(kfs)
    assert (b.host.img[0].dtype == torch.uint8) == (frames == "8bit")
    b.run_host(order)
    torch.cuda.synchronize()
    lb = b._h_loss[:len(order)].numpy()
    assert la[0] == lb[0]  # the forward and loss are deterministic
    assert np.max(np.abs(np.array(la) - lb) / np.abs(np.array(la))) < 1e-5
    assert normwise(_np(b.g.rows()), _np(a.g.rows())) < 1e-4


@pytest.mark.parametrize("lidar", [16, 64, 128, "rosette:5000", "rosette:200000"])
def test_lidar_density_sweep(lidar):
    """BASELINE config 5: 16/64/128-line and Livox-style rosette LiDAR at 1280x720 (K from ~5k
    to ~164k pixels).  The depth term evaluated on the device K-list equals the reference's dense
    depth_ratio_loss (R/losses.py:133-154) on the same rendered depth / opacity."""
    from paper_2507_04004_b200 import losses as L
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(1 << 17, 1280, 720, lidar=lidar)
    cam = R.camera_from(sc.cams[0])
    g = GaussianMap.from_rows(sc.rows)
    out = R.forward(g, cam)
    sd = sc.sparse_depths[0]
    k = int((sd > 0).sum())
    assert k > 1000
    xi = 0.005
    loss, gc, gd, go = L.mapping_loss(out.color, out.depth, out.opacity, sc.targets[0], sd, 0.2, xi)
    D, Op = _np(out.depth), _np(out.opacity)
    dv, dgd, dgo = O.depth_ratio_loss(D, Op, sd)
    pv, _ = O.photometric_loss(_np(out.color), sc.targets[0], 0.2)
    assert abs(loss - (pv + xi * dv)) < REL_TOL * abs(pv + xi * dv)
    assert normwise(_np(gd), xi * dgd) < 1e-5
    assert normwise(_np(go), xi * dgo) < 1e-5


def test_batch_optimizer_matches_batch_oracle():
    """parallel.BatchMapOptimizer (the per-rank body of the multi-GPU keyframe batch, SURVEY.md
    8e) on one GPU: summed parameter-row gradients and the touched union equal the oracle's per-
    view backward summed over the batch; the one sparse Adam step equals the oracle's on the
    same gradients."""
    from paper_2507_04004_b200 import parallel as PAR
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(4096, 96, 64, lidar=8, render_views=(0, 8, 16, 24))
    rows64 = sc.rows.astype(np.float32).astype(np.float64)
    g = GaussianMap.from_rows(sc.rows)
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    eng = PAR.BatchMapOptimizer(g, kfs, R.default_lrs(3.0))
    eng.keep_reduced = True
    eng.step(range(4))
    gsum = np.zeros((len(rows64), 59))
    tun = np.zeros(len(rows64), bool)
    og = O.GaussianMap.from_rows(rows64)
    for k, c in enumerate(sc.cams):
        cam = O.Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"], c["trans_cw"])
        out = O.forward(og, cam)
        _, gc, gd, go = O.mapping_loss(out.color, out.depth, out.opacity, sc.targets[k], sc.sparse_depths[k], 0.2,
                                       0.005)
        gr, t, _ = O.backward(og, out, gc, gd, go)
        gsum += O.grads_to_rows(gr)
        tun |= t
    ids, red = eng.reduced
    tgpu = np.zeros(len(rows64), bool)
    tgpu[_np(ids).astype(np.int64)] = True
    assert np.array_equal(tgpu, tun)
    ggpu = np.zeros((len(rows64), 59))
    ggpu[_np(ids).astype(np.int64)] = _np(red)[:, :59]
    assert not eng.grads.any() and not eng.touched.any()  # consumed by the packed Adam
    for k, (a, b) in GROUPS.items():  # near-camera Gaussians included
        assert normwise(ggpu[:, a:b], gsum[:, a:b]) < REL_TOL, k
    # the Adam step on the GPU's own gradients
    exp = rows64.copy()
    st = O.AdamState()
    O.adam_rows(exp, ggpu.astype(np.float64), tgpu, st, O.default_lrs(3.0))
    assert np.max(np.abs(_np(g.rows())[:, :59] - exp)) < 1e-5
    assert np.array_equal(_np(eng.adam.t).astype(np.int64), st.t)


def test_keyframe_preparation_on_device():
    """SURVEY.md 8f row 1 on the device (gs_project_points / gs_zbuffer / gs_init_rows) against
    the reference's outputs: pixel indices and masks exact, values to fp32 rounding."""
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    z = np.load(os.path.join(GOLD, "keyframe.npz"))
    cam = R.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    pts = z["points"]
    u, v, ui, vi, zz, inside = M.project_points(pts, cam)
    ins = _np(inside).astype(bool)
    assert np.array_equal(ins, z["inside"])
    assert np.array_equal(_np(ui)[ins], z["ui"][ins]) and np.array_equal(_np(vi)[ins], z["vi"][ins])
    assert np.max(np.abs(_np(u) - z["u"]) / np.maximum(1.0, np.abs(z["u"]))) < 1e-6
    assert np.max(np.abs(_np(zz) - z["z"]) / np.maximum(1.0, np.abs(z["z"]))) < 1e-6
    *_, colors, _ = M._project(pts, cam, image=z["image"])
    assert np.max(np.abs(_np(colors) - z["colors"])) < 1e-6
    d = _np(M.zbuffer_project(pts, cam))
    assert np.array_equal(d > 0, z["depth"] > 0)
    assert np.max(np.abs(d - z["depth"]) / np.maximum(1.0, z["depth"])) < 1e-6
    init = GaussianMap(device="cuda")
    kf = M.Keyframe(cam=cam, image=z["image"], sparse_depth=z["depth"], points=pts[ins],
                    colors=z["colors"][ins].astype(np.float32))
    assert M.init_map(init, kf) == int(ins.sum())
    assert np.max(np.abs(_np(init.rows())[:, :59] - z["init_rows"])) < 1e-5
    assert not _np(init.rows())[:, 59:].any()
    g = GaussianMap.from_rows(np.load(os.path.join(GOLD, "small0.npz"))["rows"])
    kf_all = M.Keyframe(cam=cam, image=z["image"], sparse_depth=z["depth"], points=pts,
                        colors=z["colors"].astype(np.float32))
    added = M.expand_map(g, kf_all, 0.5)
    assert added == int(z["added"])
    assert np.max(np.abs(_np(g.rows())[:, :59] - z["expanded_rows"])) < 1e-5
    cfg = M.MappingConfig(n_p=3)
    kf2 = M.group_mapping_data(0, [pts[:1500], pts[1500:]], z["image"], cam, cfg, np.random.default_rng(3))
    sp = _np(kf2.sparse_depth)
    assert np.array_equal(sp > 0, z["g_sparse"] > 0)
    assert np.max(np.abs(_np(kf2.points) - z["g_points"])) < 1e-6
    assert np.max(np.abs(_np(kf2.colors) - z["g_colors"])) < 1e-6
    assert M.group_mapping_data(1, [pts], z["image"], cam, cfg, np.random.default_rng(3)) is None
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", ["small17", "s1_1500"])
def test_photometric_refine_matches_reference(name):
    """R/odometry.py:305-336 on the device (graph-captured: forward, tracking loss, masked
    gradient, gs_chain_pose, gs_pose_adam): the pose after 1, 5 and 15 iterations and the final
    loss follow the reference's trajectory from the same perturbed start."""
    from paper_2507_04004_b200 import odometry as OD
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200.gaussians import GaussianMap
    t = np.load(os.path.join(GOLD, "track.npz"))
    z = np.load(os.path.join(GOLD, name + ".npz"))
    cam = R.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    g = GaussianMap.from_rows(z["rows"])
    start = cam.with_pose(t[f"{name}_rot0"], t[f"{name}_t0"])
    for n in (1, 5, 15):
        rot, trans, loss = OD.photometric_refine(g, t[f"{name}_image"], start, n_iters=n)
        rref, tref = t[f"{name}_{n}_rot"], t[f"{name}_{n}_trans"]
        assert np.max(np.abs(rot - rref)) < 1e-6 * n, (n, rot, rref)
        assert np.max(np.abs(trans - tref)) < 1e-6 * n, (n, trans, tref)
        lref = float(t[f"{name}_{n}_loss"])
        assert abs(loss - lref) < REL_TOL * lref, (n, loss, lref)
    # the refinement converges toward the true pose (the image is the rendering at it)
    assert np.linalg.norm(trans - z["trans_cw"]) < np.linalg.norm(t[f"{name}_t0"] - z["trans_cw"])


def test_engine_edge_cases():
    """The graph-captured engine on degenerate inputs: no Gaussian in view (every one behind the
    camera), no LiDAR return (K = 0), and an empty map (R/mapper.py:240-241 DataError)."""
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.errors import DataError
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(4096, 128, 72, lidar=16, render_views=(0,))
    cam = R.camera_from(sc.cams[0])
    # 1) looking away: rotate the camera by pi about its y axis (every Gaussian behind it)
    flip = np.diag([-1.0, 1.0, -1.0])
    away = cam.with_pose(flip @ np.asarray(cam.rot_cw), flip @ np.asarray(cam.trans_cw) - np.array([0, 0, 50.0]))
    g = GaussianMap.from_rows(sc.rows)
    eng = M.MapOptimizer(g, [M.Keyframe(away, sc.targets[0], sc.sparse_depths[0])], R.default_lrs(3.0))
    eng.capture()
    before = g.rows().clone()
    eng.step(0)
    eng.step(0)
    torch.cuda.synchronize()
    assert eng.counters()["touched"] == 0 and eng.counters()["entries"] == 0
    assert torch.equal(before, g.rows())  # untouched rows are bit-identical (R/rasterizer.py:716)
    assert not eng.adam.t.any()
    assert np.isfinite(eng.loss_sum())
    # 2) no LiDAR return: the depth term is 0 and the engine still steps
    g2 = GaussianMap.from_rows(sc.rows)
    eng2 = M.MapOptimizer(g2, [M.Keyframe(cam, sc.targets[0], np.zeros_like(sc.sparse_depths[0]))],
                          R.default_lrs(3.0))
    eng2.step(0)
    torch.cuda.synchronize()
    assert float(eng2.ws.loss[2].item()) == 0.0 and not eng2.ws.g_depth.any()
    assert int(eng2.adam.t.sum().item()) == eng2.counters()["touched"] > 0
    # 3) empty map
    with pytest.raises(DataError):
        M.MapOptimizer(GaussianMap.from_rows(np.zeros((0, 59))), [M.Keyframe(cam, sc.targets[0], None)],
                       R.default_lrs(3.0))


def _mapper_keyframes():
    """Same construction as tests/golden/make_golden.py mapper_keyframes (three room keyframes,
    seed points back-projected from the LiDAR pixels)."""
    from paper_2507_04004_b200 import scenes
    sc = scenes.scene_room(2048, 128, 72, lidar=16, render_views=(0, 10, 20))
    out = []
    for c, tgt, sd in zip(sc.cams, sc.targets, sc.sparse_depths):
        sd = sd.astype(np.float32).astype(np.float64)
        tgt = tgt.astype(np.float32).astype(np.float64)
        rot = np.asarray(c["rot_cw"]).astype(np.float32).astype(np.float64)
        trans = np.asarray(c["trans_cw"]).astype(np.float32).astype(np.float64)
        ys, xs = np.nonzero(sd > 0)
        dirs = np.stack([(xs - c["cx"]) / c["fx"], (ys - c["cy"]) / c["fy"], np.ones(len(xs))], axis=1)
        pts = ((dirs * sd[ys, xs][:, None] - trans) @ rot).astype(np.float32).astype(np.float64)
        out.append(dict(width=c["width"], height=c["height"], fx=float(np.float32(c["fx"])),
                        fy=float(np.float32(c["fy"])), cx=float(np.float32(c["cx"])), cy=float(np.float32(c["cy"])),
                        rot_cw=rot, trans_cw=trans, image=tgt, sparse=sd, points=pts, colors=tgt[ys, xs]))
    return out


def test_mapper_schedule_matches_reference():
    """mapper.Mapper (R/mapper.py:267-316): init_map, expand_map
    (opacity gate on the device), optimize_map rounds with the reference's per-keyframe RNG
    streams, then one refine round -- same Gaussians added, same losses, same map."""
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    z = np.load(os.path.join(GOLD, "mapper.npz"))
    m = M.Mapper(M.MappingConfig(), seed=0)
    added = []
    for d in _mapper_keyframes():
        cam = R.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["rot_cw"], d["trans_cw"])
        kf = M.Keyframe(cam=cam, image=d["image"], sparse_depth=d["sparse"], points=d["points"], colors=d["colors"])
        n0 = len(m.gmap)
        added.append(m.submit(kf))
        assert len(m.gmap) == n0 + added[-1]
    m.refine(1)
    assert added == [int(a) for a in z["added"]]
    ref = z["losses"]
    assert np.max(np.abs(np.array(m.losses) - ref) / ref) < REL_TOL
    t = _np(m.adam.t)[:len(m.gmap)].astype(np.int64)
    assert np.array_equal(t, z["adam_t"])
    # The map after up to 7 Adam steps per Gaussian.  Adam moves every touched parameter by up to
    # lr per step whatever |g| (its first step is lr * sign(g)), so a parameter whose reference
    # gradient is at fp32 resolution can step the other way: the elementwise deviation is bounded
    # by 2 lr t; measured, its median is ~1e-5..1e-3 of lr t per group and the 99th percentile
    # <= 0.2 lr t (tools/parity_probe.py mapper_detail).
    rows = _np(m.gmap.rows())[:, :59]
    lr = O.lr_columns(m.lrs)[:59]
    dev = np.abs(rows - z["rows"])
    assert np.all(dev <= 2.0 * lr[None, :] * t[:, None] + 1e-6)
    ratio = dev / np.maximum(lr[None, :] * np.maximum(t[:, None], 1), 1e-30)
    for k, (a, b) in GROUPS.items():
        assert np.median(ratio[:, a:b]) < 1e-2, k
        assert np.quantile(ratio[:, a:b], 0.99) < 0.5, k
    snap = m.snapshot()
    assert snap is not m.gmap and len(snap) == len(m.gmap)


def test_mapping_loop_drains_queue_and_refines():
    import queue
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    q = queue.Queue()
    for d in _mapper_keyframes()[:2]:
        cam = R.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["rot_cw"], d["trans_cw"])
        q.put(M.Keyframe(cam=cam, image=d["image"], sparse_depth=d["sparse"], points=d["points"], colors=d["colors"]))
    q.put(None)
    m = M.Mapper(M.MappingConfig(), seed=0)
    M.mapping_loop(q, m)
    assert len(m.keyframes) == 2 and len(m.losses) == 3  # two submits + max(refine_rounds, 1) round
    q.join()


def test_backward_bit_deterministic_at_benchmark_scale():
    """T/test_rasterizer.py:153-162 (forward, backward and pose gradient bit-identical across
    runs) on the headline scene, S2r 1M Gaussians at 1280x720, where every (tile, entry) of the
    backward belongs to a near-plane Gaussian covering the whole image."""
    import torch
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(1 << 20, 1280, 720, lidar=32)
    cam = R.camera_from(sc.cams[0])
    g = GaussianMap.from_rows(sc.rows)
    rng = np.random.default_rng(3)
    gc = torch.as_tensor(rng.standard_normal((720, 1280, 3)) * 1e-6, dtype=torch.float32, device="cuda")
    runs = []
    for _ in range(2):
        out = R.forward(g, cam)
        grads, touched, pose = R.backward(g, out, gc, with_pose=True)
        runs.append((out.color.clone(), grads["_rows"].clone(), touched.clone(), pose.clone()))
    for a, b in zip(*runs):
        assert torch.equal(a, b)


def test_engine_bit_deterministic():
    """T/test_mapper.py:399-410: the same keyframes in the same order give bit-identical maps
    and Adam state (graph-captured engine, fused chain + Adam)."""
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(1 << 18, 640, 360, lidar=16, render_views=(0, 8, 16))
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    states = []
    for _ in range(2):
        eng = M.MapOptimizer(GaussianMap.from_rows(sc.rows), kfs, R.default_lrs(3.0))
        eng.capture()
        for k in (0, 1, 2, 2, 0, 1, 0):
            eng.step(k)
        torch.cuda.synchronize()
        states.append(eng.save_state() + (torch.tensor(eng.loss_sum()),))
    for a, b in zip(*states):
        assert torch.equal(a, b)
    # and through the Mapper (R/mapper.py:267-316): submit the same keyframe twice, seed 7
    maps = []
    for _ in range(2):
        m = M.Mapper(M.MappingConfig(), seed=7)
        for d in _mapper_keyframes()[:1] * 2:
            cam = R.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["rot_cw"], d["trans_cw"])
            m.submit(M.Keyframe(cam=cam, image=d["image"], sparse_depth=d["sparse"], points=d["points"],
                                colors=d["colors"]))
        maps.append(m.gmap.rows().clone())
    assert torch.equal(maps[0], maps[1])


@pytest.mark.parametrize("host", [False, True])
def test_engine_recovers_from_entry_overflow(host):
    """An iteration whose binning overflows the entry capacity is a no-op on the device (tile
    ranges emptied, no gradient, no Adam step, loss not accumulated); the engine notices it from
    the lagged counters, re-lays out the workspace and re-runs it.  Overflowing every iteration
    of a run therefore ends bit-identical to a run that never overflowed (same order)."""
    import torch
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(1 << 16, 320, 180, lidar=16, render_views=(0, 8))
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    order = [0, 1, 0, 1, 1]
    runs = []
    for tiny in (False, True):
        eng = M.MapOptimizer(GaussianMap.from_rows(sc.rows), kfs, R.default_lrs(3.0))
        if tiny:
            eng.ws = eng._workspace(512)  # far below E: every iteration overflows until re-laid out
        eng.capture()
        if host:
            eng.attach_host_keyframes(kfs)
            eng.run_host(order)
        else:
            for k in order:
                eng.step(k)
        eng.finish()
        torch.cuda.synchronize()
        losses = eng._h_loss[:len(order)].clone() if host else torch.zeros(1)
        runs.append(eng.save_state() + (torch.tensor(eng.loss_sum()), losses))
        assert (eng.replayed > 0) == tiny
    for a, b in zip(*runs):
        assert torch.equal(a, b)
