"""Pin the CPU oracle (oracle/gs_oracle.c) to golden vectors produced by the reference.

The golden .npz files come from tests/golden/make_golden.py, which runs the unmodified
reference (R/rasterizer.py, R/losses.py) in the build container.  Float64 vs float64:
tolerances are 1e-9 relative (the reference's own test bar), entry lists are exact.
"""
import glob
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SCENES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLD, "*.npz"))
                if "entry_splat" in np.load(p).files)  # the forward/backward scenes


def rel(a, b, floor=1e-9):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor))) if a.size else 0.0


def load(name):
    z = np.load(os.path.join(GOLD, name + ".npz"))
    cam = O.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    return z, cam, O.GaussianMap.from_rows(z["rows"])


@pytest.mark.parametrize("name", SCENES)
def test_forward_matches_reference(name):
    z, cam, g = load(name)
    out = O.forward(g, cam)
    assert np.array_equal(out.ctx["entry_splat"], z["entry_splat"])
    assert np.array_equal(out.ctx["tile_offsets"], z["tile_offsets"])
    assert np.array_equal(out.n_contrib, z["n_contrib"])
    for k in ("color", "depth", "opacity", "transmittance"):
        assert np.max(np.abs(getattr(out, k) - z[k])) < 1e-10, k
    assert np.max(np.abs(out.ctx["proj"]["mean2d"] - z["mean2d"])) < 1e-9
    assert rel(out.ctx["proj"]["conic"], z["conic"]) < 1e-9
    assert np.array_equal(out.ctx["proj"]["valid"], z["valid"])
    assert np.max(np.abs(out.ctx["colors"] - z["colors"])) < 1e-12
    full = O.forward(g, cam, cull=False)
    assert full.ctx["entry_splat"].size == int(z["full_entries"])
    assert np.array_equal(full.n_contrib, z["full_n_contrib"])
    assert np.max(np.abs(full.color - z["full_color"])) < 1e-10


@pytest.mark.parametrize("name", SCENES)
def test_loss_backward_adam_match_reference(name):
    z, cam, g = load(name)
    out = O.forward(g, cam)
    loss, gc, gd, go = O.mapping_loss(out.color, out.depth, out.opacity, z["target"], z["sparse_depth"],
                                      float(z["lam"]), float(z["xi"]))
    assert abs(loss - float(z["loss"])) < 1e-12 * max(1.0, abs(float(z["loss"])))
    assert np.max(np.abs(gc - z["g_color"])) < 1e-15 + 1e-9 * np.abs(z["g_color"]).max()
    assert np.max(np.abs(gd - z["g_depth"])) < 1e-12
    assert np.max(np.abs(go - z["g_opac"])) < 1e-12
    g2d = O.backward_2d(out, z["g_color"], z["g_depth"], z["g_opac"])
    for k, a in zip(("mean2d", "conic", "op", "color", "depth"), g2d[:5]):
        assert rel(a, z["g2d_" + k], floor=1e-9) < 1e-8, k
    rng = np.random.default_rng(99)
    rgc = rng.standard_normal(out.color.shape)
    rgd = rng.standard_normal(out.depth.shape)
    rgo = rng.standard_normal(out.opacity.shape)
    r2d = O.backward_2d(out, rgc, rgd, rgo)
    for k, a in zip(("mean2d", "conic", "op", "color", "depth"), r2d[:5]):
        assert rel(a, z["r2d_" + k], floor=1e-9) < 1e-8, k
    grads, touched, _ = O.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"])
    assert np.array_equal(touched, z["touched"])
    gr = O.grads_to_rows(grads)
    scale = np.abs(z["grads"]).max(axis=0) + 1e-30
    assert np.max(np.abs(gr - z["grads"]) / scale) < 1e-8
    # two optimize_map iterations (R/mapper.py:249-256)
    st = O.AdamState()
    lrs = O.default_lrs(float(z["extent"]))
    O.sparse_adam_step(g, grads, touched, st, lrs)
    l2 = O.map_iteration(g, cam, z["target"], z["sparse_depth"], st, lrs, float(z["lam"]), float(z["xi"]))
    assert abs(l2 - float(z["loss2"])) < 1e-9
    assert np.max(np.abs(g.rows() - z["rows_after2"])) < 1e-9
    assert np.array_equal(st.t, z["adam_t"])


def test_losses_match_reference():
    z = np.load(os.path.join(GOLD, "losses.npz"))
    v, g = O.photometric_loss(z["a"], z["b"], 0.2)
    assert abs(v - float(z["val"])) < 1e-12 and np.max(np.abs(g - z["grad"])) < 1e-15
    dv, dg = O.dssim_and_grad(z["a"], z["b"])
    assert abs(dv - float(z["dval"])) < 1e-12 and np.max(np.abs(dg - z["dgrad"])) < 1e-15
    for pre in ("t", "o"):
        a = z["tiny_a"] if pre == "t" else z["one_a"]
        b = z["tiny_b"] if pre == "t" else z["one_b"]
        v, g = O.photometric_loss(a, b, 0.2)
        assert abs(v - float(z[pre + "val"])) < 1e-12
        assert np.max(np.abs(g - z[pre + "grad"])) < 1e-13
    v, gd, go = O.depth_ratio_loss(z["depth"], z["opac"], z["sparse"])
    assert abs(v - float(z["dv"])) < 1e-9 * abs(float(z["dv"]))
    assert np.array_equal(gd, z["dgd"]) or np.max(np.abs(gd - z["dgd"])) < 1e-15
    assert np.max(np.abs(go - z["dgo"])) <= 1e-12 * np.abs(z["dgo"]).max()


def test_known_answers():
    # R/losses.py single-pixel example (T/test_losses.py:105-117): value 1.0
    depth = np.zeros((4, 4)); opac = np.zeros((4, 4)); sparse = np.zeros((4, 4))
    depth[1, 2] = 1.5; opac[1, 2] = 0.5; sparse[1, 2] = 2.0
    v, gd, go = O.depth_ratio_loss(depth, opac, sparse)
    assert abs(v - 1.0) < 1e-14
    # guard: zero opacity -> no opacity gradient (T/test_losses.py:159-166)
    v, gd, go = O.depth_ratio_loss(np.ones((3, 3)), np.zeros((3, 3)), np.ones((3, 3)))
    assert np.isfinite(v) and not go.any()
    # Adam first step magnitude = lr (T/test_rasterizer.py:350-359)
    rows = np.random.default_rng(0).standard_normal((1, 59))
    st = O.AdamState()
    before = rows.copy()
    lrs = O.default_lrs(1.0)
    O.adam_rows(rows, np.ones((1, 59)), np.array([True]), st, lrs)
    assert np.allclose(before - rows, O.lr_columns(lrs), rtol=1e-6)


def test_det_logf():
    for x in (1.0001, 1.5, 2.0, 3.7, 100.0, 254.9):
        assert abs(O.det_logf(x) - np.log(np.float32(x))) < 2e-7 * max(1.0, np.log(x))


def _pose_scene(z, key):
    c = z[f"{key}_cam"]
    cam = O.Camera(int(c[0]), int(c[1]), float(c[2]), float(c[3]), float(c[4]), float(c[5]), z[f"{key}_rot"],
                   z[f"{key}_trans"])
    return cam, O.GaussianMap.from_rows(z[f"{key}_rows"])


@pytest.mark.parametrize("name", SCENES)
def test_pose_gradient_matches_reference(name):
    """backward(with_pose=True): R/rasterizer.py:646-657 on the golden scenes' loss gradients."""
    p = np.load(os.path.join(GOLD, "pose.npz"))
    z, cam, g = load(name)
    out = O.forward(g, cam)
    _, _, pose = O.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"], with_pose=True)
    ref = p[f"{name}_pose"]
    assert np.max(np.abs(pose - ref)) < 1e-9 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("seed", [0, 1])
def test_pose_gradient_finite_differences(seed):
    """The reference's own check (T/test_rasterizer.py:261-280): left-perturbed T_cw, central
    differences of the cull=False, early_stop=False weighted render, plus its golden value."""
    p = np.load(os.path.join(GOLD, "pose.npz"))
    key = f"fd{seed}"
    cam, g = _pose_scene(p, key)
    wc, wd, wo = p[f"{key}_wc"], p[f"{key}_wd"], p[f"{key}_wo"]
    out = O.forward(g, cam, cull=False, early_stop=False)
    grads, _, pose = O.backward(g, out, wc, wd, wo, with_pose=True)
    assert np.max(np.abs(pose - p[f"{key}_pose"])) < 1e-9 * np.abs(p[f"{key}_pose"]).max()
    assert np.max(np.abs(O.grads_to_rows(grads) - p[f"{key}_grads"])) < 1e-9 * np.abs(p[f"{key}_grads"]).max()
    from paper_2507_04004_b200.scenes import exp_so3

    def loss(c):
        o = O.forward(g, c, cull=False, early_stop=False)
        return float((o.color * wc).sum() + (o.depth * wd).sum() + (o.opacity * wo).sum())

    step = 1e-6
    for k in range(6):
        vals = []
        for sgn in (1.0, -1.0):
            eps = np.zeros(6)
            eps[k] = sgn * step
            rot = exp_so3(eps[3:]) @ cam.rot_cw
            trans = exp_so3(eps[3:]) @ cam.trans_cw + eps[:3]
            vals.append(loss(O.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, rot, trans)))
        fd = (vals[0] - vals[1]) / (2 * step)
        assert abs(pose[k] - fd) / max(abs(fd), abs(pose[k]), 1e-4) < 1e-4, (k, pose[k], fd)


def test_keyframe_preparation_matches_reference():
    """project_points / bilinear_color / zbuffer_project / init_from_points restatements against
    the reference's outputs (tests/golden/keyframe.npz)."""
    z = np.load(os.path.join(GOLD, "keyframe.npz"))
    cam = O.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    u, v, ui, vi, zz, inside = O.project_points(z["points"], cam)
    assert np.array_equal(inside, z["inside"])
    assert np.array_equal(ui[inside], z["ui"][inside]) and np.array_equal(vi[inside], z["vi"][inside])
    assert np.max(np.abs(u - z["u"])) < 1e-9 and np.max(np.abs(zz - z["z"])) < 1e-12
    assert np.max(np.abs(O.bilinear_color(z["image"], u, v) - z["colors"])) < 1e-12
    d = O.zbuffer_project(z["points"], cam)
    assert np.array_equal(d, z["depth"])
    rows = O.init_rows(z["points"][inside], z["colors"][inside].astype(np.float32).astype(np.float64),
                       zz[inside].astype(np.float32).astype(np.float64), cam.fx)
    assert np.max(np.abs(rows - z["init_rows"])) < 1e-12
