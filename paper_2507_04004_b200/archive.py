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

GRID_MAGIC = b"F32GRID\x00"


def _host(a) -> np.ndarray:
    if hasattr(a, "detach"):
        return a.detach().double().cpu().numpy()
    return np.asarray(a, dtype=np.float64)


def save_f32_grid(path, grid) -> None:
    """R/io_formats.py:23-31: 8-byte magic, uint32 width, uint32 height, row-major float32."""
    grid = _host(grid).astype(np.float32)
    if grid.ndim != 2:
        raise ValueError("grid must be 2-D")
    h, w = grid.shape
    with open(path, "wb") as f:
        f.write(GRID_MAGIC)
        f.write(struct.pack("<II", w, h))
        f.write(grid.tobytes(order="C"))


def load_f32_grid(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if len(raw) < 16 or raw[:8] != GRID_MAGIC:
        raise DataError(f"{path}: not a float32 grid file")
    w, h = struct.unpack("<II", raw[8:16])
    expect = 16 + 4 * w * h
    if len(raw) != expect:
        raise DataError(f"{path}: truncated grid ({len(raw)} != {expect} bytes)")
    return np.frombuffer(raw[16:], dtype="<f4").reshape(h, w).astype(np.float64)


def save_png(path, image) -> None:
    """R/io_formats.py:45-49: [0, 1] image to 8-bit PNG (round half to even, as np.round)."""
    from PIL import Image
    data = np.round(np.clip(_host(image), 0.0, 1.0) * 255.0).astype(np.uint8)
    Image.fromarray(data).save(path)


def load_png(path) -> np.ndarray:
    from PIL import Image
    arr = np.asarray(Image.open(path), dtype=np.float64) / 255.0
    if arr.ndim == 3 and arr.shape[2] == 4:
        arr = arr[:, :, :3]
    return arr


_POINT_DTYPE = [("xyz", "<f4", 3), ("rgb", "u1", 3)]


def save_point_ply(path, points, colors) -> None:
    """R/io_formats.py:60-78: coloured point cloud, binary little-endian PLY."""
    points = _host(points).astype(np.float32).reshape(-1, 3)
    rgb = np.round(np.clip(_host(colors).reshape(-1, 3), 0.0, 1.0) * 255.0).astype(np.uint8)
    n = len(points)
    header = ("ply\nformat binary_little_endian 1.0\n" f"element vertex {n}\n"
              "property float x\nproperty float y\nproperty float z\n"
              "property uchar red\nproperty uchar green\nproperty uchar blue\n" "end_header\n")
    rec = np.zeros(n, dtype=_POINT_DTYPE)
    rec["xyz"] = points
    rec["rgb"] = rgb
    with open(path, "wb") as f:
        f.write(header.encode("ascii"))
        f.write(rec.tobytes())


def load_point_ply(path):
    raw = Path(path).read_bytes()
    end = raw.find(b"end_header\n")
    if end < 0:
        raise DataError(f"{path}: missing PLY header terminator")
    n = None
    for line in raw[:end].decode("ascii").splitlines():
        if line.startswith("element vertex"):
            n = int(line.split()[-1])
    if n is None:
        raise DataError(f"{path}: no vertex element")
    rec = np.frombuffer(raw[end + len(b"end_header\n"):], dtype=_POINT_DTYPE, count=n)
    return rec["xyz"].astype(np.float64), rec["rgb"].astype(np.float64) / 255.0


def mat_to_quat(rot) -> np.ndarray:
    """R/geometry.py:134-170: (w, x, y, z) by Shepperd's method (largest pivot)."""
    a = np.asarray(rot, dtype=np.float64).reshape(3, 3)
    t = a[0, 0] + a[1, 1] + a[2, 2]
    c = int(np.argmax([t, a[0, 0], a[1, 1], a[2, 2]]))
    if c == 0:
        r = np.sqrt(1.0 + t)
        s = 0.5 / r
        q = [0.5 * r, (a[2, 1] - a[1, 2]) * s, (a[0, 2] - a[2, 0]) * s, (a[1, 0] - a[0, 1]) * s]
    elif c == 1:
        r = np.sqrt(1.0 + a[0, 0] - a[1, 1] - a[2, 2])
        s = 0.5 / r
        q = [(a[2, 1] - a[1, 2]) * s, 0.5 * r, (a[0, 1] + a[1, 0]) * s, (a[0, 2] + a[2, 0]) * s]
    elif c == 2:
        r = np.sqrt(1.0 - a[0, 0] + a[1, 1] - a[2, 2])
        s = 0.5 / r
        q = [(a[0, 2] - a[2, 0]) * s, (a[0, 1] + a[1, 0]) * s, 0.5 * r, (a[1, 2] + a[2, 1]) * s]
    else:
        r = np.sqrt(1.0 - a[0, 0] - a[1, 1] + a[2, 2])
        s = 0.5 / r
        q = [(a[1, 0] - a[0, 1]) * s, (a[0, 2] + a[2, 0]) * s, (a[1, 2] + a[2, 1]) * s, 0.5 * r]
    q = np.asarray(q)[None]
    q = np.where(q[:, :1] < 0.0, -q, q)
    return (q / np.linalg.norm(q, axis=-1, keepdims=True))[0]


def quat_to_mat(q) -> np.ndarray:
    """R/geometry.py:118-131 (normalised (w, x, y, z))."""
    q = np.asarray(q, dtype=np.float64)[None]
    w, x, y, z = (q / np.linalg.norm(q, axis=-1, keepdims=True))[0]
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def tum_row(t: float, rot, trans) -> str:
    """R/io_formats.py:98-103: timestamp, translation, quaternion (x y z w)."""
    q = mat_to_quat(rot)
    tx, ty, tz = np.asarray(trans, dtype=np.float64)
    return f"{t:.9f} {tx:.9f} {ty:.9f} {tz:.9f} {q[1]:.9f} {q[2]:.9f} {q[3]:.9f} {q[0]:.9f}"


def parse_tum(text: str):
    """R/io_formats.py:106-121: rows of (t, rot 3x3, trans 3)."""
    stamps, rots, transs = [], [], []
    for line in text.strip().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        vals = [float(v) for v in line.split()]
        if len(vals) != 8:
            raise DataError(f"trajectory row needs 8 fields, got {len(vals)}")
        t, tx, ty, tz, qx, qy, qz, qw = vals
        stamps.append(t)
        rots.append(quat_to_mat([qw, qx, qy, qz]))
        transs.append(np.array([tx, ty, tz]))
    return np.array(stamps), np.array(rots).reshape(-1, 3, 3), np.array(transs).reshape(-1, 3)


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
