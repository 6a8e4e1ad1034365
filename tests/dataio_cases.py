"""Builds the vector files of tests/golden/make_golden.py DATAIO_CASES (valid and malformed)."""
import os
import struct

import numpy as np


def build_case(directory, name, spec):
    fmt, n, d, mutations = spec
    x = np.random.default_rng(abs(hash(name)) % (1 << 32) if False else sum(map(ord, name))).standard_normal(
        (n, d)).astype(np.float32)
    dims = np.full(n, d, dtype=np.int32)
    trail = b""
    truncate = 0
    header = None
    for kind, a, b, v in mutations:
        if kind == "val":
            x[a, b] = np.float32(float(v))
        elif kind == "dim":
            dims[a] = v
        elif kind == "trail":
            trail = struct.pack("<i", v)[: a] if a <= 4 else struct.pack("<i", v) + b"\0" * (a - 4)
        elif kind == "truncate":
            truncate = a
        elif kind == "header":
            header = (a, b)
    path = os.path.join(directory, name + "." + fmt)
    with open(path, "wb") as f:
        if fmt == "fvecs":
            if header is not None:
                f.write(struct.pack("<i", header[0]))
                f.write(b"\0" * 16)
                return path
            rec = np.empty(n, dtype=np.dtype([("dim", "<i4"), ("vec", "<f4", (d,))]))
            rec["dim"] = dims
            rec["vec"] = x
            f.write(rec.tobytes())
            f.write(trail)
        else:
            hn, hd = header if header is not None else (n, d)
            f.write(struct.pack("<ii", hn, hd))
            data = x.tobytes()
            f.write(data[: len(data) - truncate] if truncate else data)
    return path
