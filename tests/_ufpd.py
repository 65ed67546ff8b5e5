"""Pure-Python restatement of the reference's UFPD dataset writer / reader
(/root/reference/proj/core/src/dataset.cpp:38-175) — test infrastructure for
the device-side loader (tests/test_dataset_io.py)."""
import struct

import numpy as np

MAGIC, VERSION, HEADER = 0x44504655, 1, 36


def write(path, channels, labels=None, seed=0):
    """channels / labels: complex128 [N, K, M] (row k = user)."""
    N, K, M = channels.shape
    with open(path, "wb") as f:
        f.write(struct.pack("<IIIIQQI", MAGIC, VERSION, K, M, N, seed, 1 if labels is not None else 0))
        for arr in [channels] + ([labels] if labels is not None else []):
            # row-major K x M, interleaved (re, im) f64
            f.write(np.ascontiguousarray(arr, dtype=np.complex128).tobytes())


def read(path):
    with open(path, "rb") as f:
        data = f.read()
    magic, ver, K, M, N, seed, flags = struct.unpack("<IIIIQQI", data[:HEADER])
    assert magic == MAGIC and ver == VERSION
    per = 16 * K * M
    ch = np.frombuffer(data[HEADER:HEADER + N * per], dtype=np.complex128).reshape(N, K, M)
    lab = None
    if flags & 1:
        lab = np.frombuffer(data[HEADER + N * per:HEADER + 2 * N * per], dtype=np.complex128).reshape(N, K, M)
    return dict(K=K, M=M, N=N, seed=seed, channels=ch, labels=lab)
