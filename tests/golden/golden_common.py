"""Shared helpers for golden fixtures, parity tests and bench workloads.

No dependency on the reference or on the product: seeded input bytes,
digests, and the BASELINE.json configuration specs written as
flatten_oracle-style tuple specs (``/root/reference/pkg/tests/
flatten_oracle.py:8-16`` plus ``("indexed", bls, displs, child)``).
"""

import hashlib

import numpy as np


def seeded_bytes(seed, n):
    """n uniform random bytes from numpy PCG64(seed); identical everywhere."""
    return np.random.default_rng(seed).integers(0, 256, size=n, dtype=np.uint8)


def sha(b):
    if isinstance(b, np.ndarray):
        b = b.tobytes()
    return hashlib.sha256(bytes(b)).hexdigest()


def iov_digest(pairs):
    """sha256 over the little-endian int64 (offset, length) pairs."""
    a = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    return hashlib.sha256(a.tobytes()).hexdigest()


# --- BASELINE.json configs[0]: vector(4096, 4, 8) of MPI_DOUBLE -------------
CFG1_SPEC = ("vector", 4096, 4, 8, ("basic", 8))

# --- configs[1]: halo faces of a 514^3 float32 array (512^3 interior) -------
N3 = 514
F32 = ("basic", 4)


def cfg2_faces():
    """[(name, spec)] for the six 1-wide and six 8-wide interior-boundary
    faces.  Row-major [z, y, x]; x is the fastest (last) dimension, so the
    x-faces are the 512*512 single-element-segment worst case."""
    out = []
    for w in (1, 8):
        hi = 1 + 512 - w
        for axis, name in ((2, "x"), (1, "y"), (0, "z")):
            for side, off in (("lo", 1), ("hi", hi)):
                sub = [512, 512, 512]
                offs = [1, 1, 1]
                sub[axis] = w
                offs[axis] = off
                out.append(("%s%s-w%d" % (name, side, w),
                            ("subarray", [N3, N3, N3], sub, offs, F32)))
    return out


# --- configs[2]: hvector(256) of indexed(2048) of resized-40 struct ---------
STRUCT29 = ("struct", [1, 3, 1], [0, 8, 32], [("basic", 4), ("basic", 8), ("basic", 1)])
ELEM40 = ("resized", 0, 40, STRUCT29)


def cfg3_blocks(seed, nblocks=2048):
    rng = np.random.default_rng(seed)
    bls = rng.integers(1, 65, nblocks)
    gaps = rng.integers(0, 9, nblocks)
    displs = np.empty(nblocks, dtype=np.int64)
    cur = 0
    for i in range(nblocks):
        cur += int(gaps[i])
        displs[i] = cur
        cur += int(bls[i])
    return [int(b) for b in bls], [int(d) for d in displs]


def cfg3_spec(seed, hcount=256, nblocks=2048):
    bls, displs = cfg3_blocks(seed, nblocks)
    lb = min(d * 40 for d in displs)
    ub = max((d + b - 1) * 40 + 40 for b, d in zip(bls, displs))
    ext = ub - lb
    return ("hvector", hcount, 1, ext + 4096, ("indexed", bls, displs, ELEM40))
