"""Map I/O: the reference's Gaussian PLY format and a device-state checkpoint.

`save_gaussian_ply` / `load_gaussian_ply` follow R/gaussians.py:254-305 byte for byte: binary
little-endian PLY, `comment splatmap_version 1`, one vertex of 59 float32 properties per splat in
the order x y z sx sy sz qw qx qy qz op sl0-2 sh0-44 -- which is exactly the column order of the
device parameter rows (include/gslic.h), so a save is one device->host copy of the 59 used columns
and a load one host->device copy, with no per-field shuffling.  Errors follow R/errors.py
(DataError for missing / truncated / newer-version files).

The reference never saves its optimiser state; `save_checkpoint` / `load_checkpoint` add the
Adam moments and per-Gaussian step counters (R/rasterizer.py:684-704) next to the PLY so that
map optimisation resumes exactly where it stopped.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .errors import DataError
from .gaussians import GaussianMap, as_device_map, default_device
from .plyio import PlyFormat, parse

PLY_VERSION = 1
# parameter-row columns as PLY vertex properties: position, log-scale, quaternion (w first),
# opacity logit, DC colour, 45 higher-order SH coefficients (R/gaussians.py:255-256)
FIELDS = ["x", "y", "z", "sx", "sy", "sz", "qw", "qx", "qy", "qz", "op"] + \
    [f"sl{i}" for i in range(3)] + [f"sh{i}" for i in range(45)]
NF = len(FIELDS)  # 59 = the used columns of a parameter row
GAUSSIAN_PLY = PlyFormat(properties=tuple((name, "float") for name in FIELDS),
                         comments=(f"splatmap_version {PLY_VERSION}",))


def _header(n: int) -> bytes:
    return GAUSSIAN_PLY.header(n)


def save_gaussian_ply(gmap, path) -> None:
    """R/gaussians.py:257-272: the map's 59 used row columns as one float32 record per splat."""
    g = as_device_map(gmap)
    cols = g.rows()[:, :NF].detach().to("cpu", torch.float32).contiguous().numpy()
    with open(path, "wb") as fh:
        fh.write(GAUSSIAN_PLY.encode(cols.view(GAUSSIAN_PLY.dtype).reshape(-1)))


def load_gaussian_ply(path, device=None) -> GaussianMap:
    """R/gaussians.py:275-305 onto the device; DataError for a foreign, newer or short file."""
    with open(path, "rb") as fh:
        blob = fh.read()
    head = parse(blob, str(path))
    for c in head.comments:
        key, _, val = c.partition(" ")
        if key == "splatmap_version" and int(val) > PLY_VERSION:
            raise DataError(f"{path}: unsupported splatmap version {int(val)}")
    rec = GAUSSIAN_PLY.decode(blob, str(path), head)
    rows = rec.view("<f4").reshape(len(rec), NF)
    dev = torch.device(device) if device is not None else default_device()
    return GaussianMap.from_rows(torch.from_numpy(rows.copy()).to(dev), device=dev)


def save_checkpoint(gmap, adam, path_prefix) -> tuple[str, str]:
    """<prefix>.ply (the map, reference format) + <prefix>.adam.npz (m, v rows and step counts)."""
    g = as_device_map(gmap)
    ply, st = f"{path_prefix}.ply", f"{path_prefix}.adam.npz"
    save_gaussian_ply(g, ply)
    adam.ensure(g)
    n = len(g)
    np.savez(st, version=PLY_VERSION, n=n, m=adam.m_rows[:n, :NF].cpu().numpy(),
             v=adam.v_rows[:n, :NF].cpu().numpy(), t=adam.t_dev[:n].cpu().numpy())
    return ply, st


def load_checkpoint(path_prefix, device=None):
    """Inverse of save_checkpoint: (GaussianMap, AdamState) on the device."""
    from .rasterizer import AdamState
    g = load_gaussian_ply(f"{path_prefix}.ply", device=device)
    st_path = f"{path_prefix}.adam.npz"
    if not os.path.exists(st_path):
        raise DataError(f"{st_path}: missing optimiser state")
    z = np.load(st_path)
    n = int(z["n"])
    if n != len(g):
        raise DataError(f"{st_path}: {n} Adam rows for a map of {len(g)} splats")
    adam = AdamState(device=g.device)
    adam.ensure(g)
    adam.m_rows[:n, :NF] = torch.as_tensor(z["m"], device=g.device)
    adam.v_rows[:n, :NF] = torch.as_tensor(z["v"], device=g.device)
    adam.t_dev[:n] = torch.as_tensor(z["t"], device=g.device).to(adam.t_dev.dtype)
    return g, adam
