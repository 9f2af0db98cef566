"""Philox4x32-10 counter-based generator and the injected-draw contract.

Third-party algorithm: Random123 Philox4x32-10 (Salmon et al., SC'11; the
Random123 1.x headers, ``philox.h``).  Not vendored in ``/root/reference``; the
reference samples with NumPy's PCG64 ``Generator.choice`` (``samplers.py:172,
174,177``), whose draw count per call is data dependent and therefore cannot be
replayed in parallel.  Parity is defined under *injected draws*
(SURVEY.md §8c):

    x_j = Philox4x32-10(key=(seed mod 2^32, epoch),
                        ctr=(j >> 2, row, hop, batch_id))[j & 3]

and ``choice(pool, k, replace=False)`` is a partial Fisher-Yates over pool
positions with ``r = j + ((x_j * (n - j)) >> 32)``.

Pinned by the Random123 known-answer vectors (``tests/golden/philox_kat.json``).
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10.

    ctr: uint32-compatible array shaped (..., 4); key: (..., 2).
    Returns uint32 array (..., 4).
    """
    c = np.asarray(ctr, dtype=np.uint64) & MASK32
    k = np.asarray(key, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = (c[..., i].copy() for i in range(4))
    k0, k1 = k[..., 0].copy(), k[..., 1].copy()
    k0 = np.broadcast_to(k0, c0.shape).copy()
    k1 = np.broadcast_to(k1, c0.shape).copy()
    for rnd in range(10):
        if rnd:
            k0 = (k0 + np.uint64(W0)) & MASK32
            k1 = (k1 + np.uint64(W1)) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def _philox_scalar(c0, c1, c2, c3, k0, k1):
    """Python-int Philox4x32-10 (same rounds; cheaper than NumPy for one block)."""
    m = 0xFFFFFFFF
    for rnd in range(10):
        if rnd:
            k0 = (k0 + W0) & m
            k1 = (k1 + W1) & m
        p0 = 0xD2511F53 * c0
        p1 = 0xCD9E8D57 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0, p1 & m, (p0 >> 32) ^ c3 ^ k1, p0 & m)
    return c0, c1, c2, c3


def draws(seed: int, epoch: int, batch_id: int, hop: int, row: int,
          count: int) -> np.ndarray:
    """The first ``count`` uint32 draws x_0..x_{count-1} of one row stream."""
    if count <= 0:
        return np.empty(0, dtype=np.uint32)
    if count <= 64:
        out = []
        k0, k1 = seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF
        for b in range((count + 3) // 4):
            out.extend(_philox_scalar(b, row & 0xFFFFFFFF, hop & 0xFFFFFFFF,
                                      batch_id & 0xFFFFFFFF, k0, k1))
        return np.array(out[:count], dtype=np.uint32)
    blocks = (count + 3) // 4
    ctr = np.zeros((blocks, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(blocks, dtype=np.uint64)
    ctr[:, 1] = row & 0xFFFFFFFF
    ctr[:, 2] = hop & 0xFFFFFFFF
    ctr[:, 3] = batch_id & 0xFFFFFFFF
    key = np.array([seed & 0xFFFFFFFF, epoch & 0xFFFFFFFF], dtype=np.uint64)
    return philox4x32_10(ctr, key).reshape(-1)[:count]


def fisher_yates_positions(x: np.ndarray, n: int, k: int) -> list:
    """Pool positions chosen by a partial Fisher-Yates shuffle.

    For pick j: r = j + ((x_j * (n - j)) >> 32); swap positions j and r and
    emit the element now at j.  A sparse map replaces the O(n) array.
    """
    if k > n:
        raise ValueError(f"cannot take {k} of {n} without replacement")
    swapped: dict = {}
    out = []
    for j in range(k):
        r = j + ((int(x[j]) * (n - j)) >> 32)
        a = swapped.get(j, j)
        b = swapped.get(r, r)
        out.append(b)
        swapped[r] = a
    return out


class RowStream:
    """Duck-typed ``rng`` whose ``choice`` draws from one Philox row stream."""

    def __init__(self, seed, epoch, batch_id, hop, row):
        self.key = (seed, epoch, batch_id, hop, row)

    def choice(self, a, size, replace=False):
        if replace:
            raise ValueError("the injected-draw contract is WOR only")
        a = np.asarray(a)
        x = draws(*self.key, count=size)
        return a[fisher_yates_positions(x, a.size, size)]


# ---------------------------------------------------------------------------
# Injected draws of the per-epoch cache refresh (refresh_cache, cache.py:79-108;
# weighted_sample_without_replacement, samplers.py:113-135).  Two reserved row
# streams of the (seed, epoch) key, disjoint from every sampling stream
# (batch ids < 2^32 - 1):
#   random(n)[i] = ((x_{4i} >> 5) * 2^26 + (x_{4i+1} >> 6)) * 2^-53
#                  of stream (batch 0xFFFFFFFF, hop 0xFFFFFFFE, row 0)
#                  (NumPy's 53-bit double from two 32-bit words);
#   choice(a, k)  = partial Fisher-Yates of stream (batch 0xFFFFFFFF,
#                  hop 0xFFFFFFFF, row 0), the sampling contract's selection.
REFRESH_BATCH = 0xFFFFFFFF
REFRESH_HOP_RANDOM = 0xFFFFFFFE
REFRESH_HOP_CHOICE = 0xFFFFFFFF


def refresh_uniforms(seed: int, epoch: int, n: int) -> np.ndarray:
    """random(n) of the refresh contract: f64 uniforms in [0, 1)."""
    if n <= 0:
        return np.empty(0, dtype=np.float64)
    x = draws(seed, epoch, REFRESH_BATCH, REFRESH_HOP_RANDOM, 0, 4 * n).reshape(n, 4)
    a = (x[:, 0] >> np.uint32(5)).astype(np.float64)
    b = (x[:, 1] >> np.uint32(6)).astype(np.float64)
    return (a * 67108864.0 + b) / 9007199254740992.0


class RefreshRng:
    """Duck-typed ``rng`` for refresh_cache: ``random`` and WOR ``choice``."""

    def __init__(self, seed: int, epoch: int):
        self.seed, self.epoch = int(seed), int(epoch)

    def random(self, n):
        return refresh_uniforms(self.seed, self.epoch, int(n))

    def choice(self, a, size, replace=False):
        if replace:
            raise ValueError("the injected-draw contract is WOR only")
        a = np.asarray(a)
        x = draws(self.seed, self.epoch, REFRESH_BATCH, REFRESH_HOP_CHOICE, 0, int(size))
        return a[fisher_yates_positions(x, a.size, int(size))]
