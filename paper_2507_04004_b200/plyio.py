"""Table-driven binary PLY codec shared by the map and keyframe formats (host-side I/O).

A `PlyFormat` is the format table of one file kind: the vertex properties (name, PLY scalar
type) and the header comments.  `PlyFormat.encode` writes `ply` / `format binary_little_endian
1.0` / comments / `element vertex n` / one `property` line per column / `end_header`, then the
records; `parse` reads any binary little-endian PLY header into a `PlyHeader` (comments, vertex
count, declared properties, payload offset) and `PlyFormat.decode` checks it against the table
and views the payload as a numpy record array.  The two files of the reference the hot path
reads and writes are instances of this table:

* the Gaussian map (R/gaussians.py:254-305): 59 float32 properties in parameter-row order plus
  a `splatmap_version` comment (mapio.py);
* the keyframe seed cloud (R/io_formats.py:60-95): float32 x y z, uchar red green blue
  (archive.py).

Malformed input raises `DataError` (R/errors.py), as the reference's loaders do.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DataError

# PLY scalar type -> little-endian numpy type
SCALARS = {"char": "i1", "uchar": "u1", "short": "<i2", "ushort": "<u2", "int": "<i4", "uint": "<u4",
           "float": "<f4", "double": "<f8"}
END = b"end_header\n"


@dataclass
class PlyHeader:
    comments: list = field(default_factory=list)
    vertices: int | None = None
    properties: list = field(default_factory=list)  # (name, scalar type) of the vertex element
    payload: int = 0  # byte offset of the first record


def parse(blob: bytes, where: str = "PLY") -> PlyHeader:
    """Header of a binary little-endian PLY (vertex element only)."""
    stop = blob.find(END)
    if stop < 0:
        raise DataError(f"{where}: not a PLY file (missing end_header)")
    lines = blob[:stop].decode("ascii", "replace").split("\n")
    if not lines or lines[0] != "ply":
        raise DataError(f"{where}: not a PLY file")
    head = PlyHeader(payload=stop + len(END))
    element = None
    for ln in lines[1:]:
        words = ln.split()
        if not words:
            continue
        kind = words[0]
        if kind == "comment":
            head.comments.append(ln[len("comment "):])
        elif kind == "element":
            element = words[1] if len(words) > 1 else None
            if element == "vertex" and len(words) == 3:
                head.vertices = int(words[2])
        elif kind == "property" and element == "vertex" and len(words) == 3:
            if words[1] not in SCALARS:
                raise DataError(f"{where}: unsupported property type {words[1]!r}")
            head.properties.append((words[2], words[1]))
    if head.vertices is None:
        raise DataError(f"{where}: missing vertex element")
    return head


@dataclass(frozen=True)
class PlyFormat:
    properties: tuple  # ((name, scalar type), ...)
    comments: tuple = ()

    @property
    def dtype(self) -> np.dtype:
        return np.dtype([(name, SCALARS[t]) for name, t in self.properties])

    def header(self, n: int) -> bytes:
        rows = ["ply", "format binary_little_endian 1.0"]
        rows += [f"comment {c}" for c in self.comments]
        rows.append(f"element vertex {n}")
        rows += [f"property {t} {name}" for name, t in self.properties]
        return ("\n".join(rows) + "\n").encode("ascii") + END

    def encode(self, records: np.ndarray) -> bytes:
        rec = np.ascontiguousarray(records, dtype=self.dtype)
        return self.header(len(rec)) + rec.tobytes()

    def decode(self, blob: bytes, where: str = "PLY", head: PlyHeader | None = None) -> np.ndarray:
        head = head if head is not None else parse(blob, where)
        names = [p[0] for p in head.properties]
        if head.properties and names != [p[0] for p in self.properties]:
            raise DataError(f"{where}: unexpected vertex properties {names[:4]}...")
        n = head.vertices
        need = n * self.dtype.itemsize
        body = memoryview(blob)[head.payload:]
        if len(body) < need:
            raise DataError(f"{where}: truncated payload ({len(body)} < {need} bytes)")
        return np.frombuffer(body, dtype=self.dtype, count=n)
