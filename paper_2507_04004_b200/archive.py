"""Keyframe archive and its file formats (R/mapper.py:341-364,
R/io_formats.py:20-121).

A keyframe directory holds `pose.txt` (one TUM row: stamp, camera centre, quaternion x y z w of
R_wc), `image.png` (8-bit RGB), `sparse_depth.f32` (headered float32 grid) and `points.ply` (xyz
float + rgb uchar).  The formats are written exactly as the reference writes them, so archives
move between the two implementations; `load_keyframe` returns a `mapper.Keyframe` whose image,
sparse depth and seed points can go straight to the device path (`MapOptimizer`,
`group_mapping_data`, `init_map`).  Host-side file I/O: no device work happens here.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import DataError
from .plyio import PlyFormat

# ---------------------------------------------------------------------------------------------
# format tables

# headered float32 grid (R/io_formats.py:20-42): magic, width, height (uint32 LE), row-major data
GRID_MAGIC = b"F32GRID\x00"
GRID_HEAD = struct.Struct("<8sII")
# coloured seed cloud (R/io_formats.py:60-95)
POINT_PLY = PlyFormat(properties=(("x", "float"), ("y", "float"), ("z", "float"),
                                  ("red", "uchar"), ("green", "uchar"), ("blue", "uchar")))
# TUM trajectory row (R/io_formats.py:98-121): stamp, translation, quaternion x y z w
TUM_FIELDS = 8
TUM_DIGITS = 9


def _host(a) -> np.ndarray:
    return a.detach().double().cpu().numpy() if hasattr(a, "detach") else np.asarray(a, dtype=np.float64)


def _to_u8(x) -> np.ndarray:
    """[0, 1] -> 0..255, round half to even (np.round), as the reference's writers."""
    return np.round(np.clip(_host(x), 0.0, 1.0) * 255.0).astype(np.uint8)


# ---------------------------------------------------------------------------------------------
# grids, images, point clouds


def save_f32_grid(path, grid) -> None:
    g = np.ascontiguousarray(_host(grid), dtype="<f4")
    if g.ndim != 2:
        raise ValueError("grid must be 2-D")
    Path(path).write_bytes(GRID_HEAD.pack(GRID_MAGIC, g.shape[1], g.shape[0]) + g.tobytes())


def load_f32_grid(path) -> np.ndarray:
    blob = Path(path).read_bytes()
    if len(blob) < GRID_HEAD.size:
        raise DataError(f"{path}: not a float32 grid file")
    magic, w, h = GRID_HEAD.unpack_from(blob)
    if magic != GRID_MAGIC:
        raise DataError(f"{path}: not a float32 grid file")
    if len(blob) != GRID_HEAD.size + 4 * w * h:
        raise DataError(f"{path}: truncated grid ({len(blob)} != {GRID_HEAD.size + 4 * w * h} bytes)")
    return np.frombuffer(blob, dtype="<f4", offset=GRID_HEAD.size).reshape(h, w).astype(np.float64)


def save_png(path, image) -> None:
    from PIL import Image
    Image.fromarray(_to_u8(image)).save(path)


def load_png(path) -> np.ndarray:
    from PIL import Image
    px = np.asarray(Image.open(path))
    return (px[..., :3] if px.ndim == 3 else px).astype(np.float64) / 255.0


def save_point_ply(path, points, colors) -> None:
    xyz = _host(points).astype(np.float32).reshape(-1, 3)
    rgb = _to_u8(_host(colors).reshape(-1, 3))
    rec = np.empty(len(xyz), dtype=POINT_PLY.dtype)
    for i, name in enumerate(("x", "y", "z")):
        rec[name] = xyz[:, i]
    for i, name in enumerate(("red", "green", "blue")):
        rec[name] = rgb[:, i]
    Path(path).write_bytes(POINT_PLY.encode(rec))


def load_point_ply(path):
    rec = POINT_PLY.decode(Path(path).read_bytes(), str(path))
    xyz = np.stack([rec[c] for c in ("x", "y", "z")], axis=1).astype(np.float64)
    rgb = np.stack([rec[c] for c in ("red", "green", "blue")], axis=1).astype(np.float64) / 255.0
    return xyz, rgb


# ---------------------------------------------------------------------------------------------
# poses


def mat_to_quat(rot) -> np.ndarray:
    """Unit quaternion (w, x, y, z), w >= 0, of a rotation matrix: the component of largest
    magnitude is taken from the matching diagonal combination (no cancellation) and the other
    three from the off-diagonal sums / differences (the method of R/geometry.py:134-170)."""
    m = np.asarray(rot, dtype=np.float64).reshape(3, 3)
    diag = np.array([m[0, 0] + m[1, 1] + m[2, 2], m[0, 0], m[1, 1], m[2, 2]])
    k = int(np.argmax(diag))
    # 4 |q_k|^2 = 1 + sign pattern . diag(m); rows: which diagonal signs each pivot uses
    signs = {0: (1, 1, 1), 1: (1, -1, -1), 2: (-1, 1, -1), 3: (-1, -1, 1)}[k]
    r = np.sqrt(1.0 + signs[0] * m[0, 0] + signs[1] * m[1, 1] + signs[2] * m[2, 2])
    inv = 0.5 / r
    skew = np.array([m[2, 1] - m[1, 2], m[0, 2] - m[2, 0], m[1, 0] - m[0, 1]])  # 4 w (x, y, z)
    sym = {(1, 2): m[0, 1] + m[1, 0], (1, 3): m[0, 2] + m[2, 0], (2, 3): m[1, 2] + m[2, 1]}  # 4 q_i q_j
    q = np.empty(4)
    q[k] = 0.5 * r
    for j in range(4):
        if j == k:
            continue
        if 0 in (j, k):  # w pairs with the skew part
            q[j] = skew[max(j, k) - 1] * inv
        else:
            q[j] = sym[(min(j, k), max(j, k))] * inv
    if q[0] < 0.0:
        q = -q
    return q / np.linalg.norm(q)


def quat_to_mat(q) -> np.ndarray:
    """Rotation of the normalised quaternion (w, x, y, z) (R/geometry.py:118-131)."""
    w, x, y, z = np.asarray(q, dtype=np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def tum_row(t: float, rot, trans) -> str:
    q = mat_to_quat(rot)
    vals = [t, *np.asarray(trans, dtype=np.float64), q[1], q[2], q[3], q[0]]
    return " ".join(f"{v:.{TUM_DIGITS}f}" for v in vals)


def parse_tum(text: str):
    """(stamps, rotations (k, 3, 3), translations (k, 3)) of a TUM trajectory; DataError on a row
    without exactly TUM_FIELDS numbers."""
    rows = [ln.split() for ln in text.splitlines() if ln.strip() and not ln.lstrip().startswith("#")]
    bad = [r for r in rows if len(r) != TUM_FIELDS]
    if bad:
        raise DataError(f"trajectory row needs {TUM_FIELDS} fields, got {len(bad[0])}")
    v = np.array(rows, dtype=np.float64).reshape(-1, TUM_FIELDS)
    rots = np.array([quat_to_mat([r[7], r[4], r[5], r[6]]) for r in v]).reshape(-1, 3, 3)
    return v[:, 0], rots, v[:, 1:4].copy()


def save_keyframe(dirpath, kf) -> None:
    """R/mapper.py:341-349."""
    d = Path(dirpath)
    d.mkdir(parents=True, exist_ok=True)
    rot_wc = np.asarray(kf.cam.rot_cw, dtype=np.float64).T
    center = -rot_wc @ np.asarray(kf.cam.trans_cw, dtype=np.float64)
    (d / "pose.txt").write_text(tum_row(kf.stamp, rot_wc, center) + "\n")
    save_png(d / "image.png", kf.image)
    save_f32_grid(d / "sparse_depth.f32", kf.sparse_depth)
    save_point_ply(d / "points.ply", kf.points, kf.colors)


def load_keyframe(dirpath, intrinsics):
    """R/mapper.py:352-364: intrinsics (fx, fy, cx, cy); the image size comes from the files."""
    from .mapper import Keyframe
    from .rasterizer import Camera
    d = Path(dirpath)
    stamps, rots, transs = parse_tum((d / "pose.txt").read_text())
    image = load_png(d / "image.png")
    sparse = load_f32_grid(d / "sparse_depth.f32")
    points, colors = load_point_ply(d / "points.ply")
    rot_wc, center = rots[0], transs[0]
    fx, fy, cx, cy = intrinsics
    cam = Camera(image.shape[1], image.shape[0], fx, fy, cx, cy, rot_wc.T, -rot_wc.T @ center)
    return Keyframe(cam=cam, image=image, sparse_depth=sparse, points=points, colors=colors,
                    stamp=float(stamps[0]))
