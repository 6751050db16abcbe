"""Map I/O: the reference's Gaussian PLY (R/gaussians.py:254-305), byte for
byte against a file written by the reference itself (tests/golden/small0.ply), its error
taxonomy, and the device-state checkpoint (map + Adam moments + step counts)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PLY = os.path.join(GOLD, "small0.ply")


def _bad(tmp_path, blob: bytes):
    p = tmp_path / "bad.ply"
    p.write_bytes(blob)
    return str(p)


def test_ply_errors_match_reference_taxonomy(tmp_path):
    """R/gaussians.py:275-297: missing end_header, not-a-PLY, newer version, missing vertex
    element and truncated payload all raise DataError (checked before any device work)."""
    from paper_2507_04004_b200.errors import DataError
    from paper_2507_04004_b200.mapio import load_gaussian_ply
    good = open(PLY, "rb").read()
    head, body = good.split(b"end_header\n", 1)
    cases = [b"ply\nformat binary_little_endian 1.0\n",                      # no end_header
             b"plx\n" + head[4:] + b"end_header\n" + body,                    # not a PLY
             head.replace(b"splatmap_version 1", b"splatmap_version 9") + b"end_header\n" + body,
             head.replace(b"element vertex 50", b"element face 50") + b"end_header\n" + body,
             head + b"end_header\n" + body[:-4]]                              # truncated
    for blob in cases:
        with pytest.raises(DataError):
            load_gaussian_ply(_bad(tmp_path, blob))


def test_ply_header_is_the_reference_header():
    from paper_2507_04004_b200 import mapio
    good = open(PLY, "rb").read()
    assert good.startswith(mapio._header(50))
    assert len(good) == len(mapio._header(50)) + 50 * 59 * 4


@pytest.mark.gpu
def test_ply_roundtrip_byte_exact(tmp_path):
    from paper_2507_04004_b200 import mapio
    from paper_2507_04004_b200.gaussians import GaussianMap
    z = np.load(os.path.join(GOLD, "small0.npz"))
    g = GaussianMap.from_rows(z["rows"])
    out = tmp_path / "ours.ply"
    mapio.save_gaussian_ply(g, str(out))
    assert out.read_bytes() == open(PLY, "rb").read()  # the reference's own file
    back = mapio.load_gaussian_ply(PLY)
    assert len(back) == 50
    assert np.array_equal(back.rows()[:, :59].cpu().numpy(), z["rows"].astype(np.float32))
    assert not back.rows()[:, 59:].any()


@pytest.mark.gpu
def test_checkpoint_resumes_map_optimisation(tmp_path):
    """Three iterations, checkpoint, three more == six iterations straight (same keyframe
    order); the restored map, moments and step counts are exact."""
    import torch
    from paper_2507_04004_b200 import mapio
    from paper_2507_04004_b200 import mapper as M
    from paper_2507_04004_b200 import rasterizer as R
    from paper_2507_04004_b200 import scenes
    from paper_2507_04004_b200.gaussians import GaussianMap
    sc = scenes.scene_room(4096, 128, 72, lidar=16, render_views=(0, 1))
    kfs = [M.Keyframe(R.camera_from(c), t, s) for c, t, s in zip(sc.cams, sc.targets, sc.sparse_depths)]
    lrs = R.default_lrs(3.0)
    a = M.MapOptimizer(GaussianMap.from_rows(sc.rows), kfs, lrs)
    for k in (0, 1, 0):
        a.step(k)
    a.loss_sum()  # reset the accumulated loss
    prefix = str(tmp_path / "ckpt")
    mapio.save_checkpoint(a.g, a.adam, prefix)
    g2, adam2 = mapio.load_checkpoint(prefix)
    n = len(a.g)
    assert torch.equal(g2.rows()[:, :59], a.g.rows()[:, :59])
    assert torch.equal(adam2.m_rows[:n, :59], a.adam.m_rows[:n, :59])
    assert torch.equal(adam2.v_rows[:n, :59], a.adam.v_rows[:n, :59])
    assert torch.equal(adam2.t[:n], a.adam.t[:n])
    b = M.MapOptimizer(g2, kfs, lrs, adam=adam2)
    la, lb = [], []
    for k in (1, 0, 1):
        a.step(k)
        la.append(a.loss_sum())
        b.step(k)
        lb.append(b.loss_sum())
    assert la[0] == lb[0]  # the forward of the restored state is bit-identical
    assert np.allclose(la, lb, rtol=1e-5)
