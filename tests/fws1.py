"""FWS1 snapshot reader / writer (format of harness.hpp:121-124, README.md:124-128):
magic "FWS1", u8 dim, per axis (u32 J, f64 a, f64 b), f64 time, N f64 row-major, little-endian.
Golden fixtures under tests/golden/ are written by the reference's own write_snapshot."""
from __future__ import annotations

import struct

import numpy as np


def read(path):
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"FWS1":
        raise ValueError(f"{path}: not an FWS1 snapshot")
    d = data[4]
    off = 5
    J, lo, hi = [], [], []
    for _ in range(d):
        j, a, b = struct.unpack_from("<Idd", data, off)
        off += 20
        J.append(j)
        lo.append(a)
        hi.append(b)
    (t,) = struct.unpack_from("<d", data, off)
    off += 8
    n = int(np.prod(J))
    vals = np.frombuffer(data, dtype="<f8", count=n, offset=off).copy().reshape(J)
    return vals, tuple(lo), tuple(hi), t


def write(path, values, lo, hi, time=0.0):
    values = np.ascontiguousarray(values, dtype="<f8")
    with open(path, "wb") as f:
        f.write(b"FWS1")
        f.write(bytes([values.ndim]))
        for J, a, b in zip(values.shape, lo, hi):
            f.write(struct.pack("<Idd", J, a, b))
        f.write(struct.pack("<d", time))
        f.write(values.tobytes())
