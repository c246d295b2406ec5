"""Counter-based random numbers for the random signal block R.

PAPER.md §3.1 (lines 182-185) and §4.1 step 4 (line 316): R in R^{N x eta} has
independent Gaussian entries of mean 0 and variance 1/eta.

The generator is counter based so that the host (this module) and the device
(``sc_random_signals`` in the CUDA library) produce the same block without
sharing state:

    key   = splitmix64(seed ^ STREAM_SALT[stream])
    h1    = splitmix64(key + 2*ctr),  h2 = splitmix64(key + 2*ctr + 1)
    u1    = ((h1 >> 11) + 1) * 2^-53          in (0, 1]
    u2    =  (h2 >> 11)      * 2^-53          in [0, 1)
    z     = sqrt(-2 ln u1) * cos(2 pi u2)      (Box-Muller, fp64)
    R[i,q] = float32(z * sqrt(1/eta))  with ctr = i*eta + q

All arithmetic here is fp64 / uint64 and then rounded once to the storage type,
so the two sides agree to the last bit except when libm's log/cos differ by one
fp64 ulp right at an fp32 rounding boundary (probability ~2^-29 per entry).
"""

from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = 2.0 ** -53

# stream salts: 0 = signal block R, 1 = k-means++ uniforms, 2 = eigencount probes
STREAM_SALT = (0x0, 0xA5A5A5A5A5A5A5A5, 0x5BD1E9955BD1E995)


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def _key(seed: int, stream: int) -> np.uint64:
    return splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ np.uint64(STREAM_SALT[stream]))


def gaussian_block(seed: int, n: int, eta: int, row0: int = 0, dtype=np.float32,
                   variance: float | None = None, stream: int = 0, cols=None) -> np.ndarray:
    """Rows [row0, row0+n) of the N x eta Gaussian block for ``seed``.

    ``variance`` defaults to 1/eta.  ``row0`` lets a rank
    of a row-partitioned run generate exactly its own rows of the global block.
    ``cols`` (optional): only these columns of the eta-wide block (same values).
    """
    if variance is None:
        variance = 1.0 / eta
    key = _key(seed, stream)
    qs = np.arange(eta, dtype=np.uint64) if cols is None else np.asarray(cols, dtype=np.uint64)
    out = np.empty((n, len(qs)), dtype=dtype)
    scale = np.sqrt(np.float64(variance))
    chunk = max(1, (1 << 22) // max(len(qs), 1))
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        ctr = (np.arange(row0 + r0, row0 + r1, dtype=np.uint64)[:, None] * np.uint64(eta)
               + qs[None, :])
        with np.errstate(over="ignore"):
            h1 = splitmix64(key + np.uint64(2) * ctr)
            h2 = splitmix64(key + np.uint64(2) * ctr + np.uint64(1))
        u1 = ((h1 >> np.uint64(11)).astype(np.float64) + 1.0) * _TWO_M53
        u2 = (h2 >> np.uint64(11)).astype(np.float64) * _TWO_M53
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        out[r0:r1] = (z * scale).astype(dtype)
    return out


def uniforms(seed: int, count: int, offset: int = 0, stream: int = 1) -> np.ndarray:
    """``count`` fp64 uniforms in [0,1) at counters offset..offset+count-1."""
    key = _key(seed, stream)
    ctr = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(key + ctr)
    return (h >> np.uint64(11)).astype(np.float64) * _TWO_M53
