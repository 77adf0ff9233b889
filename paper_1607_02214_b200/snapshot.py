"""PPLR v1 snapshot files (the reference's src/snapshot.cpp / snapshot.hpp).

Layout (little-endian): magic "PPLR", u32 version (1), u32 dims[3], u32
ghost, f64 time, u64 step, per-axis edge arrays (dims[a] + 1 f64 each), the
8-byte field-order tag "rvvvbbbp", then one f64 array of the interior cells
(x fastest) per field in the order rho, vx, vy, vz, B'x, B'y, B'z, p.

The GPU writer is ``Harness.write_snapshot`` (device capture + host drain,
``ppmlr_gpu_harness_snapshot``); this module is the host-side reader and a
plain writer for data already on the host, with the reference's checks and
messages (snapshot.cpp:58-123).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from ._native import InvalidSpec

MAGIC = b"PPLR"
FIELD_TAG = b"rvvvbbbp"
_HEAD = struct.Struct("<4sI3IIdQ")


@dataclass
class Snapshot:
    """snapshot.hpp:17-25; ``fields`` is (8, nz, ny, nx), field-major."""
    version: int = 1
    dims: tuple = (0, 0, 0)
    ghost: int = 0
    time: float = 0.0
    step: int = 0
    edges: list = field(default_factory=list)
    fields: np.ndarray | None = None

    def states(self):
        """gather_interior order: (nz, ny, nx, 8) PrimitiveState records."""
        return np.moveaxis(self.fields, 0, -1)


def read_snapshot(path) -> Snapshot:
    """read_snapshot (snapshot.cpp:88-123)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise InvalidSpec(f"snapshot: cannot open: {path}") from None
    if len(data) < 4 or data[:4] != MAGIC:
        raise InvalidSpec(f"snapshot: bad magic in {path}")
    if len(data) < _HEAD.size:
        raise InvalidSpec("snapshot: truncated while reading version")
    _, version, nx, ny, nz, ghost, time, step = _HEAD.unpack_from(data, 0)
    if version != 1:
        raise InvalidSpec(f"snapshot: unsupported version {version}")
    off = _HEAD.size
    edges = []
    for n in (nx, ny, nz):
        nb = 8 * (n + 1)
        if off + nb > len(data):
            raise InvalidSpec(f"snapshot: truncated edge array in {path}")
        edges.append(np.frombuffer(data, "<f8", n + 1, off).copy())
        off += nb
    if data[off:off + 8] != FIELD_TAG:
        raise InvalidSpec(f"snapshot: unknown field order tag in {path}")
    off += 8
    cells = nx * ny * nz
    if off + 64 * cells > len(data):
        raise InvalidSpec(f"snapshot: truncated field payload in {path}")
    fields = np.frombuffer(data, "<f8", 8 * cells, off).reshape(8, nz, ny, nx).copy()
    return Snapshot(version, (nx, ny, nz), ghost, time, step, edges, fields)


def write_snapshot(path, snap: Snapshot):
    """write_snapshot (snapshot.cpp:58-85) for host-resident data."""
    nx, ny, nz = snap.dims
    f = np.ascontiguousarray(snap.fields, dtype="<f8")
    if f.shape != (8, nz, ny, nx):
        raise InvalidSpec("snapshot: field count does not match dims")
    for a, n in enumerate(snap.dims):
        if len(snap.edges[a]) != n + 1:
            raise InvalidSpec("snapshot: edge array does not match dims")
    try:
        out = open(path, "wb")
    except OSError:
        raise InvalidSpec(f"snapshot: cannot open for writing: {path}") from None
    with out:
        out.write(_HEAD.pack(MAGIC, snap.version, nx, ny, nz, snap.ghost, snap.time, snap.step))
        for e in snap.edges:
            out.write(np.asarray(e, "<f8").tobytes())
        out.write(FIELD_TAG)
        out.write(f.tobytes())
