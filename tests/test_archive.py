"""Keyframe archive: the reference's on-disk formats (R/io_formats.py,
R/mapper.py:341-364) against an archive written by the reference itself
(tests/golden/kf_archive, make_golden.py record_archive).  Host-side I/O: runs on CPU."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ARCH = os.path.join(GOLD, "kf_archive")


def _src():
    z = np.load(os.path.join(GOLD, "kf_archive.npz"))
    r = np.load(os.path.join(GOLD, "room4096.npz"))
    return z, r


def test_save_keyframe_writes_the_reference_bytes(tmp_path):
    from paper_2507_04004_b200 import archive as A
    from paper_2507_04004_b200.mapper import Keyframe
    from paper_2507_04004_b200.rasterizer import Camera
    z, r = _src()
    cam = Camera(int(r["width"]), int(r["height"]), float(r["fx"]), float(r["fy"]), float(r["cx"]), float(r["cy"]),
                 r["rot_cw"], r["trans_cw"])
    kf = Keyframe(cam=cam, image=z["src_image"], sparse_depth=z["src_sparse"], points=z["src_points"],
                  colors=z["src_colors"], stamp=12.5)
    out = tmp_path / "kf"
    A.save_keyframe(out, kf)
    for name in ("pose.txt", "sparse_depth.f32", "points.ply"):
        assert (out / name).read_bytes() == open(os.path.join(ARCH, name), "rb").read(), name
    assert np.array_equal(A.load_png(out / "image.png"), A.load_png(os.path.join(ARCH, "image.png")))


def test_load_keyframe_matches_reference():
    from paper_2507_04004_b200 import archive as A
    z, r = _src()
    kf = A.load_keyframe(ARCH, (float(r["fx"]), float(r["fy"]), float(r["cx"]), float(r["cy"])))
    assert np.max(np.abs(np.asarray(kf.cam.rot_cw) - z["rot_cw"])) < 1e-15
    assert np.max(np.abs(np.asarray(kf.cam.trans_cw) - z["trans_cw"])) < 1e-12
    assert (kf.cam.width, kf.cam.height) == (int(r["width"]), int(r["height"]))
    for k in ("image", "sparse", "points", "colors"):
        got = {"image": kf.image, "sparse": kf.sparse_depth, "points": kf.points, "colors": kf.colors}[k]
        assert np.array_equal(got, z[k]), k
    assert kf.stamp == float(z["stamp"])


def test_format_errors(tmp_path):
    from paper_2507_04004_b200 import archive as A
    from paper_2507_04004_b200.errors import DataError
    p = tmp_path / "g.f32"
    p.write_bytes(b"NOTAGRID" + bytes(8))
    with pytest.raises(DataError):
        A.load_f32_grid(p)
    good = open(os.path.join(ARCH, "sparse_depth.f32"), "rb").read()
    p.write_bytes(good[:-4])
    with pytest.raises(DataError):
        A.load_f32_grid(p)
    q = tmp_path / "p.ply"
    q.write_bytes(b"ply\nformat binary_little_endian 1.0\n")
    with pytest.raises(DataError):
        A.load_point_ply(q)
    with pytest.raises(DataError):
        A.parse_tum("1 2 3 4 5 6 7\n")


def test_quaternion_round_trip():
    from paper_2507_04004_b200 import archive as A
    from paper_2507_04004_b200.scenes import exp_so3
    rng = np.random.default_rng(2)
    for _ in range(50):
        R = exp_so3(rng.standard_normal(3) * 2.0)
        assert np.max(np.abs(A.quat_to_mat(A.mat_to_quat(R)) - R)) < 1e-12
