"""Counter-based splitmix64 stream shared by every input generator.

This module holds NO arithmetic of the Krylov method: it only turns
(seed, tag, index) triples into reproducible integers / uniforms / normals so
that the oracle (``oracle/``) and the CUDA path see the same synthetic inputs.
The recipe is fixed in DESIGN.md ("Input recipe") after SURVEY.md §8(d):

* ``key(seed, tag)``      = splitmix64 finaliser of ``seed * 2^32 + tag``
* ``bits(seed, tag, i)``  = splitmix64 finaliser of ``key + (i + 1) * GOLDEN``
* uniform double in [0,1) = ``(bits >> 11) * 2^-53``  (exact)
* normal                  = Box-Muller on two uniforms (values are shared, not
                            re-derived on the device, so libm differences do not
                            matter)

All integer arithmetic is done on numpy uint64 arrays, which wrap modulo 2^64.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
MASK64 = (1 << 64) - 1


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def key(seed: int, tag: int) -> np.uint64:
    v = ((int(seed) << 32) + int(tag)) & MASK64
    return mix64(np.array([v], dtype=np.uint64))[0]


def bits(seed: int, tag: int, idx) -> np.ndarray:
    """64 random bits for every counter in ``idx`` (any integer array)."""
    idx = np.asarray(idx, dtype=np.uint64)
    k = key(seed, tag)
    with np.errstate(over="ignore"):
        x = k + (idx + np.uint64(1)) * GOLDEN
    return mix64(x)


def uniform(seed: int, tag: int, idx) -> np.ndarray:
    """Exact uniform doubles in [0, 1): (bits >> 11) * 2^-53."""
    b = bits(seed, tag, idx) >> np.uint64(11)
    return b.astype(np.float64) * (2.0 ** -53)


def normal(seed: int, tag: int, idx) -> np.ndarray:
    """Standard normals by Box-Muller from counters 2i and 2i+1 of the stream."""
    idx = np.asarray(idx, dtype=np.uint64)
    u1 = uniform(seed, tag, idx * np.uint64(2))
    u2 = uniform(seed, tag, idx * np.uint64(2) + np.uint64(1))
    r = np.sqrt(-2.0 * np.log1p(-u1))  # 1-u1 in (0, 1]
    return r * np.cos(2.0 * np.pi * u2)


def complex_normal(seed: int, tag: int, idx) -> np.ndarray:
    """N(0,1) + i N(0,1) with the real/imag parts from tags ``tag`` / ``tag+1``."""
    return normal(seed, tag, idx) + 1j * normal(seed, tag + 1, idx)
