"""Synthetic mapping workloads (fixed seeds) for tests and the benchmark.

* ``scene_s1``  -- "frustum-uniform" scene of SURVEY.md Appendix A (S1), the same RNG draw
  order, so the reference's measured statistics apply.  Every splat is in view: the
  blend-heavy stress case.
* ``scene_room`` -- SLAM-like surface scene ("S2r"): splats seeded on the surfaces of a
  procedurally generated room seen from 32 viewpoints, the target image and the LiDAR
  depth ray-cast from view 0.  It follows the recipe of SURVEY.md Appendix A (S2), with
  this repo's own room generator, because the reference simulator does not exist on the
  GPU box.
* ``make_scene``  -- the small randomized scene of the reference tests
  (T/test_rasterizer.py:24-57 recipe).

Everything here is host-side numpy; it produces float64 arrays that callers convert.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SH_C0 = 0.28209479177387814


def exp_so3(phi) -> np.ndarray:
    """Rodrigues formula (rotation vector -> matrix)."""
    phi = np.asarray(phi, dtype=np.float64)
    th = float(np.linalg.norm(phi))
    k = np.array([[0.0, -phi[2], phi[1]], [phi[2], 0.0, -phi[0]], [-phi[1], phi[0], 0.0]])
    if th < 1e-8:
        a, b = 1.0 - th * th / 6.0, 0.5 - th * th / 24.0
    else:
        a, b = np.sin(th) / th, (1.0 - np.cos(th)) / (th * th)
    return np.eye(3) + a * k + b * (k @ k)


def logit(p):
    return np.log(p / (1.0 - p))


@dataclass
class SceneData:
    """Packed splat rows (n, 59) float64 in GaussianMap.parameters() order, cameras,
    target image(s), sparse LiDAR depth image(s)."""
    rows: np.ndarray
    cams: list          # list of dicts: width height fx fy cx cy rot_cw (3,3) trans_cw (3,)
    targets: list       # (H, W, 3) float64 per camera
    sparse_depths: list  # (H, W) float64 per camera, 0 = no LiDAR return
    name: str = ""


def cam_dict(width, height, fx, fy, cx, cy, rot_cw, trans_cw) -> dict:
    return {"width": int(width), "height": int(height), "fx": float(fx), "fy": float(fy),
            "cx": float(cx), "cy": float(cy), "rot_cw": np.asarray(rot_cw, dtype=np.float64),
            "trans_cw": np.asarray(trans_cw, dtype=np.float64)}


def pack_rows(pos, log_scale, quat, opacity_logit, sh_low, sh_high) -> np.ndarray:
    n = len(pos)
    return np.ascontiguousarray(np.hstack([
        pos, log_scale, quat, np.asarray(opacity_logit).reshape(n, 1), sh_low,
        np.asarray(sh_high).reshape(n, 45)]), dtype=np.float64)


# ---------------------------------------------------------------------------
# S1


def scene_s1(n: int, width: int, height: int, seed: int = 0, k_lidar: int = 30000) -> SceneData:
    rng = np.random.default_rng(seed)
    f = 0.8 * width
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    rot_cw = exp_so3(0.1 * rng.standard_normal(3))
    trans_cw = 0.5 * rng.standard_normal(3)
    z = rng.uniform(2, 8, n)
    u = rng.uniform(0, width - 1, n)
    v = rng.uniform(0, height - 1, n)
    p_cam = np.stack([(u - cx) / f * z, (v - cy) / f * z, z], axis=1)
    pos = (p_cam - trans_cw) @ rot_cw
    scale = rng.uniform(0.5, 3.0, (n, 3)) * (z / f)[:, None]
    quat = rng.standard_normal((n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    opl = logit(rng.uniform(0.05, 0.95, n))
    sh_low = (rng.uniform(0.2, 0.8, (n, 3)) - 0.5) / SH_C0
    sh_high = 0.02 * rng.standard_normal((n, 15, 3))
    cam = cam_dict(width, height, f, f, cx, cy, rot_cw, trans_cw)
    target = rng.uniform(0, 1, (height, width, 3))
    sparse = np.zeros((height, width))
    k = min(int(k_lidar), width * height)
    idx = rng.choice(width * height, k, replace=False)
    sparse.flat[idx] = rng.uniform(2, 8, k)
    return SceneData(pack_rows(pos, np.log(scale), quat, opl, sh_low, sh_high), [cam], [target], [sparse],
                     name=f"S1-{n}-{width}x{height}")


# ---------------------------------------------------------------------------
# small test scene (T/test_rasterizer.py:24-57 recipe)


def make_scene(seed, n=50, width=48, height=32, max_op=0.92, deg0=False, scale_px=3.0) -> SceneData:
    rng = np.random.default_rng(seed)
    fx = fy = 60.0
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    rot_cw = exp_so3(0.1 * rng.standard_normal(3))
    trans_cw = 0.5 * rng.standard_normal(3)
    z = np.linspace(2.0, 8.0, n) + rng.uniform(-0.02, 0.02, n)
    rng.shuffle(z)
    u = rng.uniform(3, width - 4, n)
    v = rng.uniform(3, height - 4, n)
    p_cam = np.stack([(u - cx) / fx * z, (v - cy) / fy * z, z], axis=1)
    pos = (p_cam - trans_cw) @ rot_cw
    scale = rng.uniform(1.0, scale_px, (n, 3)) * (z / fx)[:, None]
    quat = rng.standard_normal((n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    opl = logit(rng.uniform(0.05, max_op, n))
    sh_low = (rng.uniform(0.3, 0.9, (n, 3)) - 0.5) / SH_C0
    sh_high = np.zeros((n, 15, 3)) if deg0 else 0.02 * rng.standard_normal((n, 15, 3))
    cam = cam_dict(width, height, fx, fy, cx, cy, rot_cw, trans_cw)
    target = rng.uniform(0, 1, (height, width, 3))
    sparse = np.zeros((height, width))
    idx = rng.choice(width * height, max(1, width * height // 20), replace=False)
    sparse.flat[idx] = rng.uniform(2, 8, len(idx))
    return SceneData(pack_rows(pos, np.log(scale), quat, opl, sh_low, sh_high), [cam], [target], [sparse],
                     name=f"small-{seed}-{n}")


# ---------------------------------------------------------------------------
# S2r: SLAM-like room scene


@dataclass
class Room:
    lo: np.ndarray      # (B, 3) box minima; box 0 is the room shell (seen from inside)
    hi: np.ndarray      # (B, 3)
    base: np.ndarray    # (B, 6, 3) albedo per box face (-x, +x, -y, +y, -z, +z)
    cell: np.ndarray    # (B,) checker cell size (m)
    strength: np.ndarray  # (B,) checker contrast


def make_room(seed: int = 7) -> Room:
    rng = np.random.default_rng([seed, 11])
    hx, hy, hz = rng.uniform(4.6, 5.8), rng.uniform(4.0, 5.2), rng.uniform(3.0, 3.8)
    lo = [np.array([-hx, -hy, 0.0])]
    hi = [np.array([hx, hy, hz])]
    # pillar off the centre, plus 2-4 corner boxes
    px, py = rng.uniform(0.6, 1.1) * rng.choice([-1, 1]), rng.uniform(0.6, 1.1) * rng.choice([-1, 1])
    ph = rng.uniform(1.0, 1.5)
    lo.append(np.array([px - 0.3, py - 0.3, 0.0]))
    hi.append(np.array([px + 0.3, py + 0.3, ph]))
    corners = [(1, 1), (1, -1), (-1, 1), (-1, -1)]
    rng.shuffle(corners)
    for sx, sy in corners[: int(rng.integers(2, 5))]:
        cx = sx * (hx - rng.uniform(0.75, 1.1))
        cy = sy * (hy - rng.uniform(0.75, 1.1))
        half = np.array([rng.uniform(0.25, 0.5), rng.uniform(0.25, 0.5), rng.uniform(0.3, 0.9)])
        c = np.array([cx, cy, half[2]])
        lo.append(c - half)
        hi.append(c + half)
    b = len(lo)
    return Room(np.array(lo), np.array(hi), rng.uniform(0.15, 0.85, (b, 6, 3)),
                rng.uniform(0.35, 0.85, b), rng.uniform(0.25, 0.45, b))


def cast_room(room: Room, origin: np.ndarray, dirs: np.ndarray):
    """Nearest hit of rays (origin (3,), dirs (n,3)) against the room; returns (t, box, face)."""
    n = len(dirs)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / dirs
    best = np.full(n, np.inf)
    box = np.full(n, -1, np.int64)
    face = np.full(n, -1, np.int64)
    for k in range(len(room.lo)):
        t0 = (room.lo[k] - origin) * inv
        t1 = (room.hi[k] - origin) * inv
        tmin = np.minimum(t0, t1)
        tmax = np.maximum(t0, t1)
        if k == 0:  # inside the shell: exit point
            t = np.min(tmax, axis=1)
            ax = np.argmin(tmax, axis=1)
            hit = t > 1e-9
        else:
            tn = np.max(tmin, axis=1)
            tf = np.min(tmax, axis=1)
            t = tn
            ax = np.argmax(tmin, axis=1)
            hit = (tn <= tf) & (tn > 1e-9)
        better = hit & (t < best)
        best[better] = t[better]
        box[better] = k
        d_ax = dirs[np.arange(n), ax]
        # face index: 2*axis + (positive side)
        if k == 0:
            fidx = 2 * ax + (d_ax > 0)
        else:
            fidx = 2 * ax + (d_ax < 0)
        face[better] = fidx[better]
    return best, box, face


def room_albedo(room: Room, box, face, pts) -> np.ndarray:
    base = room.base[box, face]
    cell = room.cell[box]
    q = np.floor(pts / cell[:, None]).astype(np.int64)
    checker = (q.sum(axis=1) & 1).astype(np.float64) * 2.0 - 1.0
    h = (q[:, 0] * 73856093) ^ (q[:, 1] * 19349663) ^ (q[:, 2] * 83492791)
    noise = ((h & 1023) / 1023.0 - 0.5) * 0.06
    col = base * (1.0 + room.strength[box][:, None] * 0.5 * checker[:, None]) + noise[:, None]
    return np.clip(col, 0.0, 1.0)


def room_poses(room: Room, seed: int, count: int):
    """Camera poses on a loop inside the room, gazing outward-tangentially (world->camera)."""
    rng = np.random.default_rng([seed, 404])
    hx, hy = room.hi[0][0], room.hi[0][1]
    r = min(hx, hy) - 1.8 + 0.35
    zc = 1.65
    th = np.linspace(0.0, 2.0 * np.pi, count, endpoint=False) + rng.uniform(0.05, 0.25, count)
    beta = 0.35
    out = []
    for t in th:
        tang = np.array([-np.sin(t), np.cos(t), 0.0])
        inward = np.array([-np.cos(t), -np.sin(t), 0.0])
        fwd = np.cos(beta) * tang + np.sin(beta) * inward
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, [0.0, 0.0, 1.0])
        right /= np.linalg.norm(right)
        down = np.cross(fwd, right)
        rot_wc = np.column_stack([right, down, fwd])  # camera axes in world
        c = np.array([r * np.cos(t), r * np.sin(t), zc])
        out.append((rot_wc.T, -rot_wc.T @ c))
    return out


def lidar_lines(depth_img: np.ndarray, lines: int) -> np.ndarray:
    h, w = depth_img.shape
    rows = np.unique(np.round(np.linspace(0.1 * h, 0.9 * h, lines)).astype(np.int64).clip(0, h - 1))
    sparse = np.zeros_like(depth_img)
    sparse[rows, :] = depth_img[rows, :]
    return sparse


def lidar_rosette(depth_img: np.ndarray, k: int, petals: int = 7, seed: int = 3) -> np.ndarray:
    """Livox-style non-repetitive rosette r = r0 cos(k theta), sampled to ~k unique pixels."""
    h, w = depth_img.shape
    rng = np.random.default_rng(seed)
    th = np.sort(rng.uniform(0, 2 * np.pi * 16, 4 * k))
    rr = np.cos(petals * th)
    x = np.round((w - 1) / 2 + 0.5 * (w - 1) * rr * np.cos(th)).astype(np.int64)
    y = np.round((h - 1) / 2 + 0.5 * (h - 1) * rr * np.sin(th)).astype(np.int64)
    idx = np.unique(y.clip(0, h - 1) * w + x.clip(0, w - 1))[:k]
    sparse = np.zeros_like(depth_img)
    sparse.flat[idx] = depth_img.flat[idx]
    return sparse


def scene_room(n: int, width: int, height: int, focal: float | None = None, seed: int = 7,
               views: int = 32, lidar: int | str = 32, render_views=(0,)) -> SceneData:
    """S2r(n, W, H): splats on room surfaces from `views` viewpoints; targets from render_views."""
    room = make_room(seed)
    f = float(focal) if focal is not None else 700.0 * width / 1280.0
    cx, cy = (width - 1) / 2.0, (height - 1) / 2.0
    poses = room_poses(room, seed, views)
    rng = np.random.default_rng(seed)
    per = n // views
    pts, zs, cols = [], [], []
    for rot_cw, trans_cw in poses:
        rot_wc = rot_cw.T
        c = -rot_wc @ trans_cw
        u = rng.uniform(0, width - 1, per)
        v = rng.uniform(0, height - 1, per)
        d = np.stack([(u - cx) / f, (v - cy) / f, np.ones(per)], axis=1) @ rot_wc.T
        t, box, face = cast_room(room, c, d)
        p = c + t[:, None] * d
        pts.append(p)
        zs.append(t)
        cols.append(room_albedo(room, box, face, p))
    pos = np.concatenate(pts)
    z_src = np.concatenate(zs)
    color = np.concatenate(cols)
    m = len(pos)
    scale = (z_src / f)[:, None] * rng.uniform(1, 3, (m, 3))
    quat = rng.standard_normal((m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    opl = logit(rng.uniform(0.1, 0.9, m))
    sh_low = (color - 0.5) / SH_C0
    sh_high = 0.02 * rng.standard_normal((m, 15, 3))
    cams, targets, sparses = [], [], []
    for vi in render_views:
        rot_cw, trans_cw = poses[vi]
        rot_wc = rot_cw.T
        c = -rot_wc @ trans_cw
        xs, ys = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
        d = np.stack([(xs.ravel() - cx) / f, (ys.ravel() - cy) / f, np.ones(width * height)], axis=1) @ rot_wc.T
        t, box, face = cast_room(room, c, d)
        p = c + t[:, None] * d
        target = room_albedo(room, box, face, p).reshape(height, width, 3)
        depth = t.reshape(height, width)
        if isinstance(lidar, str) and lidar.startswith("rosette"):
            k = int(lidar.split(":")[1]) if ":" in lidar else 20000
            sparse = lidar_rosette(depth, k)
        else:
            sparse = lidar_lines(depth, int(lidar))
        cams.append(cam_dict(width, height, f, f, cx, cy, rot_cw, trans_cw))
        targets.append(target)
        sparses.append(sparse)
    return SceneData(pack_rows(pos, np.log(scale), quat, opl, sh_low, sh_high), cams, targets, sparses,
                     name=f"S2r-{n}-{width}x{height}")
