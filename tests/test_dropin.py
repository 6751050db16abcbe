"""The drop-in switch (paper_2507_04004_b200.dropin).

CPU (this container, where the reference is importable): `dropin.install` applied to the REAL
`splatslam` package rebinds every listed name, each replacement keeps the reference's parameter
names, and `uninstall` restores the package.

GPU: the reference package cannot travel to the GPU box, so the switch is applied to a stand-in
`splatslam` package built here in a temp dir -- modules of the same names holding the reference's
data types (a numpy `GaussianMap` restating R/gaussians.py:118-153) -- and the hot-path checks of
the reference's own tests (T/test_rasterizer.py, T/test_losses.py, T/test_mapper.py) run through
`splatslam.rasterizer.*` etc. with the reference's numpy maps, numpy image arithmetic on the
outputs, in-place Adam, and fp32-relaxed tolerances.
"""
import importlib
import inspect
import os
import sys
import types

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


def _params(obj):
    fn = obj.__init__ if inspect.isclass(obj) else obj
    try:
        sig = inspect.signature(fn)
    except (TypeError, ValueError):
        return None
    return [p.name for p in sig.parameters.values() if p.name != "self" and p.kind not in (p.VAR_POSITIONAL,
                                                                                          p.VAR_KEYWORD)]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "splatslam")), reason="reference not present (GPU box)")
def test_switch_rebinds_the_reference_package():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    try:
        import splatslam
        from paper_2507_04004_b200 import dropin
        originals = {}
        for sub, names in dropin.BINDINGS.items():
            mod = importlib.import_module(f"splatslam.{sub}")
            for name in names:
                assert hasattr(mod, name), f"splatslam.{sub}.{name} missing in the reference"
                originals[(sub, name)] = getattr(mod, name)
        saved = dropin.install(splatslam)
        try:
            for (sub, name), ref_obj in originals.items():
                mod = importlib.import_module(f"splatslam.{sub}")
                ours = getattr(mod, name)
                assert ours is not ref_obj and ours.__module__.startswith("paper_2507_04004_b200"), (sub, name)
                # the reference's parameters, in order (ours may add keyword-only extras)
                rp, op = _params(ref_obj), _params(ours)
                if rp is not None and op is not None:
                    assert op[:len(rp)] == rp, (sub, name, rp, op)
        finally:
            dropin.uninstall(splatslam, saved)
        for (sub, name), ref_obj in originals.items():
            assert getattr(importlib.import_module(f"splatslam.{sub}"), name) is ref_obj
    finally:
        sys.path.remove(REF)


# ---------------------------------------------------------------------------------------------
# GPU: the switch on a stand-in package, the reference's hot-path checks through it


class RefGaussianMap:
    """The reference's map container (R/gaussians.py:118-153): six numpy arrays, parameters() in
    PLY order, append by concatenation, snapshot by copy."""

    def __init__(self, pos, log_scale, quat, opacity_logit, sh_low, sh_high):
        self.pos, self.log_scale, self.quat = np.asarray(pos, float), np.asarray(log_scale, float), np.asarray(quat, float)
        self.opacity_logit, self.sh_low = np.asarray(opacity_logit, float), np.asarray(sh_low, float)
        self.sh_high = np.asarray(sh_high, float).reshape(len(self.pos), 15, 3)

    def __len__(self):
        return len(self.pos)

    def parameters(self):
        return {"pos": self.pos, "log_scale": self.log_scale, "quat": self.quat, "opacity_logit": self.opacity_logit,
                "sh_low": self.sh_low, "sh_high": self.sh_high}

    def append(self, other):
        for k, v in other.parameters().items():
            setattr(self, k, np.concatenate([getattr(self, k), v]))

    def snapshot(self):
        return RefGaussianMap(**{k: v.copy() for k, v in self.parameters().items()})


@pytest.fixture
def splatslam(tmp_path):
    """A stand-in `splatslam` package (modules of the reference's names), switched to this build."""
    pkg = types.ModuleType("splatslam_standin")
    pkg.__path__ = []
    for sub in ("rasterizer", "losses", "gaussians", "mapper", "odometry"):
        m = types.ModuleType(f"splatslam_standin.{sub}")
        sys.modules[m.__name__] = m
        setattr(pkg, sub, m)
    sys.modules[pkg.__name__] = pkg
    pkg.gaussians.GaussianMap = RefGaussianMap
    from paper_2507_04004_b200 import dropin
    saved = dropin.install(pkg)
    yield pkg
    dropin.uninstall(pkg, saved)
    for name in [k for k in sys.modules if k.startswith("splatslam_standin")]:
        del sys.modules[name]


SH_C0 = 0.28209479177387814


def make_scene(seed, n=50, width=48, height=32, max_op=0.92, rast=None):
    """T/test_rasterizer.py:24-57's scene recipe (random splats inside the frustum)."""
    from paper_2507_04004_b200.scenes import exp_so3
    rng = np.random.default_rng(seed)
    fx = fy = 60.0
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    rot_cw = exp_so3(0.1 * rng.standard_normal(3))
    trans_cw = 0.5 * rng.standard_normal(3)
    z = np.linspace(2.0, 8.0, n) + rng.uniform(-0.02, 0.02, n)
    rng.shuffle(z)
    u, v = rng.uniform(3, width - 4, n), rng.uniform(3, height - 4, n)
    p_cam = np.stack([(u - cx) / fx * z, (v - cy) / fy * z, z], axis=1)
    scale = rng.uniform(1.0, 3.0, (n, 3)) * (z / fx)[:, None]
    quat = rng.standard_normal((n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    op = rng.uniform(0.05, max_op, n)
    gmap = RefGaussianMap((p_cam - trans_cw) @ rot_cw, np.log(scale), quat, np.log(op / (1 - op)),
                          (rng.uniform(0.3, 0.9, (n, 3)) - 0.5) / SH_C0, 0.02 * rng.standard_normal((n, 15, 3)))
    return gmap, rast.Camera(width, height, fx, fy, cx, cy, rot_cw, trans_cw)


def _oracle(gmap, cam, cull=True, early_stop=True):
    import oracle as O
    rows = np.hstack([gmap.pos, gmap.log_scale, gmap.quat, gmap.opacity_logit[:, None], gmap.sh_low,
                      gmap.sh_high.reshape(len(gmap), 45)]).astype(np.float32).astype(np.float64)
    ocam = O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy,
                    np.asarray(cam.rot_cw, np.float32).astype(float), np.asarray(cam.trans_cw, np.float32).astype(float))
    return O.forward(O.GaussianMap.from_rows(rows), ocam, cull=cull, early_stop=early_stop)


@pytest.mark.gpu
def test_forward_through_switch_is_numpy(splatslam):
    rast = splatslam.rasterizer
    gmap, cam = make_scene(0, rast=rast)
    out = rast.forward(gmap, cam, cull=False, early_stop=True)
    assert isinstance(out.color, np.ndarray) and out.color.dtype == np.float64
    ref = _oracle(gmap, cam, cull=False)
    assert np.max(np.abs(out.color - ref.color)) < 1e-5
    assert np.max(np.abs(out.depth - ref.depth)) < 1e-4
    assert np.array_equal(out.n_contrib, ref.n_contrib)
    # the reference callers' numpy arithmetic (R/cli.py:153-159, R/mapper.py:222-225)
    img = np.clip(out.color, 0.0, 1.0)
    ys, xs = np.array([1, 5, 9]), np.array([2, 4, 8])
    assert img.shape == (cam.height, cam.width, 3) and (out.opacity[ys, xs] >= 0).all()
    for k in ("colors", "preclamp", "dirs", "u_norm", "opac"):
        assert isinstance(out.ctx[k], np.ndarray), k
    assert np.allclose(out.ctx["colors"], np.maximum(out.ctx["preclamp"], 0.0), atol=1e-6)
    assert np.allclose(np.linalg.norm(out.ctx["dirs"], axis=1), 1.0, atol=1e-6)
    assert out.ctx["entry_splat"].dtype == np.int64 and isinstance(out.ctx["proj"]["mean2d"], np.ndarray)


@pytest.mark.gpu
def test_culling_checks_through_switch(splatslam):
    """T/test_rasterizer.py:182-198: sub-1/255 splats culled everywhere; culled vs unculled PSNR."""
    rast = splatslam.rasterizer
    gmap, cam = make_scene(19, n=10, rast=rast)
    gmap.opacity_logit[:] = np.log((1 / 300) / (1 - 1 / 300))  # in place on the numpy map
    out = rast.forward(gmap, cam, cull=True)
    assert out.ctx["entry_splat"].size == 0 and not out.color.any()
    for seed in range(3):
        gmap, cam = make_scene(seed + 100, n=200, width=80, height=64, max_op=0.97, rast=rast)
        mse = np.mean((rast.forward(gmap, cam, cull=True).color - rast.forward(gmap, cam, cull=False).color) ** 2)
        assert 10.0 * np.log10(1.0 / max(mse, 1e-300)) >= 45.0


@pytest.mark.gpu
def test_backward_through_switch(splatslam):
    """T/test_rasterizer.py:221-233 (a splat behind the camera: untouched, zero gradient) and the
    gradients against the oracle; numpy grads in the reference's shapes."""
    import oracle as O
    rast = splatslam.rasterizer
    gmap, cam = make_scene(29, n=5, rast=rast)
    gmap.pos[2] = cam.center() - 10.0 * np.asarray(cam.rot_cw).T @ np.array([0, 0, 1.0])
    out = rast.forward(gmap, cam, cull=True)
    grads, touched, pose = rast.backward(gmap, out, np.ones_like(out.color), with_pose=True)
    assert isinstance(touched, np.ndarray) and not touched[2]
    for k, arr in grads.items():
        assert isinstance(arr, np.ndarray) and arr.shape == gmap.parameters()[k].shape, k
        assert not np.asarray(arr[2]).any()
    assert isinstance(pose, np.ndarray) and pose.shape == (6,)
    gmap, cam = make_scene(23, n=30, width=40, height=32, max_op=0.97, rast=rast)
    out = rast.forward(gmap, cam)
    rng = np.random.default_rng(0)
    gc = rng.standard_normal(out.color.shape)
    grads, touched, _ = rast.backward(gmap, out, gc)
    ref = _oracle(gmap, cam)
    rg, rt, _ = O.backward(O.GaussianMap.from_rows(ref.ctx["rows"]), ref, gc)
    assert np.array_equal(touched, rt)
    for k in grads:
        a, b = np.asarray(grads[k]), np.asarray(rg[k])
        assert np.max(np.abs(a - b)) <= 1e-3 * max(np.max(np.abs(b)), 1e-12), k


@pytest.mark.gpu
def test_sparse_adam_in_place_through_switch(splatslam):
    """T/test_rasterizer.py:316-359 on the reference's numpy map: updated in place, untouched rows
    bit-identical, per-splat step counts (numpy), first step = lr, 5 steps = dense Adam."""
    rast = splatslam.rasterizer
    gmap, _ = make_scene(37, n=6, rast=rast)
    rng = np.random.default_rng(4)
    state = rast.AdamState()
    lrs = rast.default_lrs(1.0)
    touched = np.array([True, False, True, False, True, False])
    before = {k: v.copy() for k, v in gmap.parameters().items()}
    rast.sparse_adam_step(gmap, {k: rng.standard_normal(v.shape) for k, v in gmap.parameters().items()}, touched,
                          state, lrs)
    for k, arr in gmap.parameters().items():
        assert np.array_equal(arr[~touched], before[k][~touched])
        assert not np.array_equal(arr[touched], before[k][touched])
    assert np.array_equal(state.t, np.array([1, 0, 1, 0, 1, 0]))
    gmap, _ = make_scene(41, n=1, rast=rast)
    state = rast.AdamState()
    before = {k: v.copy() for k, v in gmap.parameters().items()}
    rast.sparse_adam_step(gmap, {k: np.ones_like(v) for k, v in gmap.parameters().items()}, np.array([True]), state,
                          lrs)
    for k, arr in gmap.parameters().items():
        assert np.allclose(before[k] - arr, lrs[k], rtol=1e-6), k
    gmap, _ = make_scene(31, n=12, rast=rast)
    lrs = rast.default_lrs(2.0)
    state = rast.AdamState()
    reference = {k: v.copy() for k, v in gmap.parameters().items()}
    m = {k: np.zeros_like(v) for k, v in reference.items()}
    v2 = {k: np.zeros_like(v) for k, v in reference.items()}
    for t in range(1, 6):
        grads = {k: rng.standard_normal(v.shape) for k, v in gmap.parameters().items()}
        rast.sparse_adam_step(gmap, grads, np.ones(12, bool), state, lrs)
        for k in reference:
            g = grads[k]
            m[k] = 0.9 * m[k] + 0.1 * g
            v2[k] = 0.999 * v2[k] + 0.001 * g * g
            reference[k] -= lrs[k] * (m[k] / (1 - 0.9 ** t)) / (np.sqrt(v2[k] / (1 - 0.999 ** t)) + 1e-15)
    for k, arr in gmap.parameters().items():  # fp32 moments and step, float64 parameters
        assert np.max(np.abs(arr - reference[k])) <= 1e-5 * lrs[k] * 5, k


@pytest.mark.gpu
def test_losses_through_switch(splatslam):
    """T/test_losses.py known answers (fp32-relaxed), numpy in -> numpy out."""
    L = splatslam.losses
    rng = np.random.default_rng(6)
    a = rng.uniform(0, 1, (24, 32, 3))
    b = np.clip(a + 0.15 * rng.standard_normal(a.shape), 0, 1)
    val, grad = L.photometric_loss(a, a, lam=0.2)
    assert abs(val) < 1e-6 and isinstance(grad, np.ndarray)
    val, grad = L.photometric_loss(a, b, lam=0.0)
    assert np.isclose(val, np.mean(np.abs(a - b)), atol=1e-6)
    assert np.allclose(grad, np.sign(a.astype(np.float32) - b.astype(np.float32)) / a.size, atol=1e-10)
    val, _ = L.dssim_and_grad(a, a)
    assert abs(val) < 1e-6
    v1, _ = L.dssim_and_grad(a, b)
    v2, _ = L.dssim_and_grad(b, a)
    assert 0.0 <= v1 <= 1.0 and abs(v1 - v2) < 1e-6
    depth, opac, sparse = np.zeros((4, 4)), np.zeros((4, 4)), np.zeros((4, 4))
    depth[1, 2], opac[1, 2], sparse[1, 2] = 1.5, 0.5, 2.0
    val, gd, go = L.depth_ratio_loss(depth, opac, sparse)
    assert np.isclose(val, 1.0, atol=1e-6)
    mask = np.zeros((4, 4), bool)
    mask[1, 2] = True
    assert not gd[~mask].any() and not go[~mask].any()
    a4 = rng.uniform(0, 1, (4, 4, 3))
    s4 = np.zeros((4, 4))
    s4[1, 2] = 2.0
    val, *_ = L.mapping_loss(a4, np.full((4, 4), 1.5), np.full((4, 4), 0.5), a4, s4, lam=0.2, xi=1.0)
    assert np.isclose(val, 1.0, atol=1e-6)
    val, gd, go = L.depth_ratio_loss(np.ones((3, 3)), np.zeros((3, 3)), np.ones((3, 3)))
    assert np.isfinite(val) and not go.any() and np.all(np.isfinite(gd))


@pytest.mark.gpu
def test_mapper_through_switch_updates_numpy_maps(splatslam):
    """T/test_mapper.py:399-418: optimize_map on the reference's numpy map moves it in place and
    is deterministic across runs; an empty map raises DataError; init/expand grow a numpy map."""
    from paper_2507_04004_b200.errors import DataError
    mp, rast = splatslam.mapper, splatslam.rasterizer
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import scenes
    sc = scenes.scene_room(2048, 96, 64, lidar=8, render_views=(0, 8))
    kfs = [M.Keyframe(rast.Camera(c["width"], c["height"], c["fx"], c["fy"], c["cx"], c["cy"], c["rot_cw"],
                                  c["trans_cw"]), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    maps = []
    for _ in range(2):
        r = sc.rows
        g = RefGaussianMap(r[:, 0:3], r[:, 3:6], r[:, 6:10], r[:, 10], r[:, 11:14], r[:, 14:59])
        before = g.pos.copy()
        loss = mp.optimize_map(g, kfs, M.MappingConfig(), np.random.default_rng(7), rast.AdamState(),
                               rast.default_lrs(3.0))
        assert np.isfinite(loss) and not np.array_equal(g.pos, before)
        maps.append(g)
    for k in maps[0].parameters():
        assert np.array_equal(maps[0].parameters()[k], maps[1].parameters()[k]), k
    empty = RefGaussianMap(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 3)),
                           np.zeros((0, 15, 3)))
    with pytest.raises(DataError):
        mp.optimize_map(empty, kfs, M.MappingConfig(), np.random.default_rng(0), rast.AdamState(),
                        rast.default_lrs(1.0))
    pts = sc.rows[:300, 0:3]
    kf = M.Keyframe(kfs[0].cam, sc.targets[0], sc.sparse_depths[0], points=pts, colors=np.full((300, 3), 0.5))
    added = mp.init_map(empty, kf)
    assert isinstance(empty.pos, np.ndarray) and len(empty) == added > 0
