"""Diagnostic (test infrastructure): prints the measured parity errors behind the tolerances of
tests/test_gpu_parity.py, so each bar can be set from a measurement.

    python tools/parity_probe.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from test_gpu_parity import SCENES, _np, load, normwise  # noqa: E402

from paper_2507_04004_b200 import losses as L  # noqa: E402
from paper_2507_04004_b200 import rasterizer as R  # noqa: E402

GROUPS = {"pos": (0, 3), "log_scale": (3, 6), "quat": (6, 10), "opacity_logit": (10, 11), "sh_low": (11, 14),
          "sh_high": (14, 59)}


def main():
    for name in SCENES:
        z, cam, g = load(name)
        out = R.forward(g, cam)
        img = {k: float(np.max(np.abs(_np(getattr(out, k)) - z[k]))) for k in ("color", "depth", "opacity",
                                                                                  "transmittance")}
        ncm = float(np.mean(_np(out.n_contrib) != z["n_contrib"]))
        vm = z["valid"]
        mref = z["mean2d"][vm]
        m_err = float(np.max(np.abs(_np(out.ctx["proj"]["mean2d"])[vm] - mref) / np.maximum(1.0, np.abs(mref))))
        print(f"[{name}] img {img} n_contrib_mismatch {ncm:.2e} mean2d(all valid) {m_err:.2e}")
        g2d = R.backward_2d(out, z["g_color"], z["g_depth"], z["g_opac"])
        e2 = {k: normwise(_np(a), z["g2d_" + k]) for k, a in zip(("mean2d", "conic", "op", "color", "depth"), g2d[:5])}
        print(f"   g2d {({k: f'{v:.1e}' for k, v in e2.items()})}")
        grads, touched, pose = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"], with_pose=True)
        gr = _np(grads["_rows"])[:, :59]
        near = z["pdepth"] < 0.05
        errs = {k: normwise(gr[:, a:b], z["grads"][:, a:b]) for k, (a, b) in GROUPS.items()}
        print(f"   grads all {({k: f'{v:.1e}' for k, v in errs.items()})}  near={int(near.sum())}")
        p = np.load(os.path.join(ROOT, "tests", "golden", "pose.npz"))
        print(f"   pose {normwise(_np(pose), p[name + '_pose']):.2e}")
        grads2, _, pose2 = R.backward(g, out, z["g_color"], z["g_depth"], z["g_opac"], with_pose=True)
        print(f"   deterministic grads {torch.equal(grads['_rows'], grads2['_rows'])} pose {torch.equal(pose, pose2)}")
    # mapping iterations (test_mapping_iterations_match_oracle)
    from paper_2507_04004_b200 import mapper as M
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
        dg = _np(g.rows())[:, :59] - sc.rows
        dr = og.rows() - sc.rows
        print(f"   it {it} loss rel {abs(gl - ol) / abs(ol):.2e} map delta normwise {normwise(dg, dr):.2e} "
              f"per-group {({k2: f'{normwise(dg[:, a:b], dr[:, a:b]):.1e}' for k2, (a, b) in GROUPS.items()})}")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def mapper_and_tracking():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import _mapper_keyframes
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import odometry as OD
    from paper_2507_04004_b200.gaussians import GaussianMap
    z = np.load(os.path.join(ROOT, "tests", "golden", "mapper.npz"))
    m = M.Mapper(M.MappingConfig(), seed=0)
    for d in _mapper_keyframes():
        cam = R.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["rot_cw"], d["trans_cw"])
        m.submit(M.Keyframe(cam=cam, image=d["image"], sparse_depth=d["sparse"], points=d["points"], colors=d["colors"]))
    m.refine(1)
    ref = z["losses"]
    print("mapper losses rel", np.abs(np.array(m.losses) - ref) / ref)
    gr = _np(m.gmap.rows())[:, :59]
    print("mapper rows normwise", normwise(gr, z["rows"]), {k: f"{normwise(gr[:, a:b], z['rows'][:, a:b]):.1e}" for k, (a, b) in GROUPS.items()})
    t = np.load(os.path.join(ROOT, "tests", "golden", "track.npz"))
    for name in ("small17", "s1_1500"):
        zz = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
        cam = R.Camera(int(zz["width"]), int(zz["height"]), float(zz["fx"]), float(zz["fy"]), float(zz["cx"]),
                       float(zz["cy"]), zz["rot_cw"], zz["trans_cw"])
        g = GaussianMap.from_rows(zz["rows"])
        start = cam.with_pose(t[f"{name}_rot0"], t[f"{name}_t0"])
        for n in (1, 5, 15):
            rot, trans, loss = OD.photometric_refine(g, t[f"{name}_image"], start, n_iters=n)
            print(f"track {name} n={n} rot {np.max(np.abs(rot - t[f'{name}_{n}_rot'])):.2e} "
                  f"trans {np.max(np.abs(trans - t[f'{name}_{n}_trans'])):.2e} loss rel "
                  f"{abs(loss - float(t[f'{name}_{n}_loss'])) / float(t[f'{name}_{n}_loss']):.2e}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "mapper":
    mapper_and_tracking()


def mapper_detail():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_gpu_parity import _mapper_keyframes
    from paper_2507_04004_b200 import mapper as M
    z = np.load(os.path.join(ROOT, "tests", "golden", "mapper.npz"))
    m = M.Mapper(M.MappingConfig(), seed=0)
    for d in _mapper_keyframes():
        cam = R.Camera(d["width"], d["height"], d["fx"], d["fy"], d["cx"], d["cy"], d["rot_cw"], d["trans_cw"])
        m.submit(M.Keyframe(cam=cam, image=d["image"], sparse_depth=d["sparse"], points=d["points"], colors=d["colors"]))
    m.refine(1)
    t = _np(m.adam.t)[:len(m.gmap)].astype(np.int64)
    rows = _np(m.gmap.rows())[:, :59]
    lr = O.lr_columns(m.lrs)[:59]
    dev = np.abs(rows - z["rows"])
    ratio = dev / np.maximum(lr[None, :] * np.maximum(t[:, None], 1), 1e-30)
    scale = np.max(np.abs(z["rows"]), axis=0)
    close = dev <= 1e-3 * np.maximum(scale, 1e-3)[None, :]
    for k, (a, b) in GROUPS.items():
        r = ratio[:, a:b]
        print(f"{k}: close {np.mean(close[:, a:b]):.3f} dev/(lr t) p50 {np.median(r):.2e} p99 {np.quantile(r, 0.99):.2e} "
              f"max {r.max():.2e}; scale {scale[a:b].max():.2e} lr {lr[a]:.2e}")
    print("t hist", np.bincount(t)[:12], "rows", len(rows))
    # per-Gaussian: which ones deviate (fresh vs initial)
    bad = ~close.all(axis=1)
    print("bad gaussians", int(bad.sum()), "of", len(bad), "index ranges", np.flatnonzero(bad)[:10], np.flatnonzero(bad)[-10:])


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "mapper_detail":
    mapper_detail()
