"""Counter-hash random streams (oracle restatement -- test infrastructure only).

Restates /root/reference/pkg/src/vecpomdp/rng.py.  A stream is a 64-bit key;
a draw for logical row r is a pure function of (key, r, draw index):

    base(r)      = F(key + PHI * (r + 2))                 rng.py:69
    single draw  = F(base + MIX_A)                        rng.py:70-71
    draw j (1..k)= F(base + j * MIX_B)                    rng.py:72-73
    uniform      = (h >> 11) * 2**-53                     rng.py:78-79

with F the SplitMix64 finaliser (rng.py:26-31) and all arithmetic wrapping
mod 2**64.  Child streams fold one word at a time: key' = F(key + PHI*(w+1))
(rng.py:34-36); seeds enter as F(seed + PHI) (rng.py:52-54).
"""

from __future__ import annotations

import numpy as np

U64 = np.uint64
PHI = U64(0x9E3779B97F4A7C15)
MIX_A = U64(0xBF58476D1CE4E5B9)
MIX_B = U64(0x94D049BB133111EB)
_SCALE = 2.0 ** -53
_MASK = (1 << 64) - 1


def mix64(x):
    """SplitMix64 finaliser (rng.py:26-31); accepts uint64 scalars/arrays."""
    with np.errstate(over="ignore"):
        y = x ^ (x >> U64(30))
        y = y * MIX_A
        y = y ^ (y >> U64(27))
        y = y * MIX_B
        return y ^ (y >> U64(31))


def fold_word(key, word: int):
    """One derivation step, rng.py:34-36."""
    if word < 0:
        raise ValueError("derivation words must be non-negative")
    with np.errstate(over="ignore"):
        return mix64(U64(key) + PHI * (U64(word) + U64(1)))


def row_hashes(key, rows: np.ndarray, k: int | None):
    """Per-row 64-bit draws, rng.py:67-73."""
    r = np.asarray(rows, dtype=np.int64).astype(U64)
    with np.errstate(over="ignore"):
        base = mix64(U64(key) + PHI * (r + U64(2)))
        if k is None:
            return mix64(base + MIX_A)
        steps = np.arange(1, k + 1, dtype=U64) * MIX_B
        return mix64(base[:, None] + steps[None, :])


def to_unit(h):
    """53-bit mantissa uniform in [0, 1), rng.py:78-79."""
    return (h >> U64(11)).astype(np.float64) * _SCALE


class RowRng:
    """Immutable key node of the stream tree (rng.py:39-93)."""

    __slots__ = ("key",)

    def __init__(self, key):
        self.key = U64(key)

    @classmethod
    def from_seed(cls, seed: int) -> "RowRng":
        with np.errstate(over="ignore"):
            return cls(mix64(U64(seed & _MASK) + PHI))

    def derive(self, *words: int) -> "RowRng":
        k = self.key
        for w in words:
            k = fold_word(k, w)
        return RowRng(k)

    def bind(self, rows) -> "BoundRng":
        return BoundRng(self, rows)

    def uniform(self, rows, k: int | None = None) -> np.ndarray:
        return to_unit(row_hashes(self.key, rows, k))

    def normal(self, rows, k: int | None = None) -> np.ndarray:
        """Box-Muller from the derive(101)/derive(211) sub-streams, rng.py:81-89."""
        h1 = row_hashes(self.derive(101).key, rows, k)
        h2 = row_hashes(self.derive(211).key, rows, k)
        u1 = ((h1 >> U64(11)).astype(np.float64) + 1.0) * _SCALE
        u2 = (h2 >> U64(11)).astype(np.float64) * _SCALE
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)

    def uniform1(self) -> float:
        return float(self.uniform(np.zeros(1, dtype=np.int64))[0])


class BoundRng:
    """A RowRng with its logical row ids fixed (rng.py:96-120)."""

    __slots__ = ("rng", "rows")

    def __init__(self, rng: RowRng, rows):
        self.rng = rng
        self.rows = np.asarray(rows, dtype=np.int64)

    def __len__(self) -> int:
        return len(self.rows)

    def derive(self, *words: int) -> "BoundRng":
        return BoundRng(self.rng.derive(*words), self.rows)

    def uniform(self, k: int | None = None) -> np.ndarray:
        return self.rng.uniform(self.rows, k)

    def normal(self, k: int | None = None) -> np.ndarray:
        return self.rng.normal(self.rows, k)


# ---------------------------------------------------------------- Philox fast mode
#
# Not in the reference: the north_star's "counter-based Philox RNG", the
# device's optional fast stream kind (vp_model.rng_kind = VP_RNG_PHILOX,
# csrc/vp_common.cuh).  Philox4x32-10 as Salmon, Moraes, Dror & Shaw,
# "Parallel random numbers: as easy as 1, 2, 3" (SC'11) define it, pinned to the
# Random123 known-answer vectors in tests/test_rng_contract_cpu.py.  Stream keys
# derive exactly as above (SplitMix64 folds); only the per-row draw changes:
#     block(key, row, j, tag) = Philox4x32-10(ctr = (lo row, hi row, lo j, tag), key = (lo key, hi key))
#     uniform  (tag 0; j = 0 single draw, j = 1..k)  = top 53 bits of (x << 32 | y) * 2**-53
#     normal   (tag 1)  = Box-Muller pairs: block b = (j + 1) // 2, u1 = (bits(x, y) + 1) 2**-53,
#                         u2 = bits(z, w) 2**-53, R = sqrt(-2 log u1); normal j = R cos(2 pi u2) for
#                         odd j (and j = 0), R sin(2 pi u2) for even j

PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
_M32 = U64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Philox4x32-10 over arrays: ctr (..., 4) and key (..., 2) of uint32-valued ints -> (..., 4) uint32."""
    c = [np.asarray(ctr, dtype=U64)[..., i] & _M32 for i in range(4)]
    k0 = np.asarray(key, dtype=U64)[..., 0] & _M32
    k1 = np.asarray(key, dtype=U64)[..., 1] & _M32
    m0, m1 = U64(PHILOX_M0), U64(PHILOX_M1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = c[0] * m0
            p1 = c[2] * m1
            c = [(p1 >> U64(32)) ^ c[1] ^ k0, p1 & _M32, (p0 >> U64(32)) ^ c[3] ^ k1, p0 & _M32]
            k0 = (k0 + U64(PHILOX_W0)) & _M32
            k1 = (k1 + U64(PHILOX_W1)) & _M32
    return np.stack(c, axis=-1).astype(np.uint32)


def philox_row_blocks(key, rows, js, tag: int):
    """Blocks for every (row, j): rows (n,), js (k,) -> (n, k, 4)."""
    r = np.asarray(rows, dtype=np.int64).astype(U64)
    j = np.asarray(js, dtype=np.int64).astype(U64)
    n, k = len(r), len(j)
    ctr = np.empty((n, k, 4), dtype=U64)
    ctr[..., 0] = (r & _M32)[:, None]
    ctr[..., 1] = (r >> U64(32))[:, None]
    ctr[..., 2] = (j & _M32)[None, :]
    ctr[..., 3] = U64(tag)
    kk = U64(key)
    keyv = np.array([int(kk) & 0xFFFFFFFF, int(kk) >> 32], dtype=U64)
    return philox4x32_10(ctr, np.broadcast_to(keyv, (n, k, 2)))


def _bits53(hi, lo):
    return ((hi.astype(U64) << U64(32)) | lo.astype(U64)) >> U64(11)


class PhiloxRowRng(RowRng):
    """RowRng whose per-row draws are Philox4x32-10 blocks (the device fast mode)."""

    __slots__ = ()
    rng_kind = 1  # vp_rng_kind VP_RNG_PHILOX

    def derive(self, *words: int) -> "PhiloxRowRng":
        k = self.key
        for w in words:
            k = fold_word(k, w)
        return PhiloxRowRng(k)

    def uniform(self, rows, k: int | None = None) -> np.ndarray:
        js = [0] if k is None else range(1, k + 1)
        b = philox_row_blocks(self.key, rows, js, 0)
        u = _bits53(b[..., 0], b[..., 1]).astype(np.float64) * _SCALE
        return u[:, 0] if k is None else u

    def normal(self, rows, k: int | None = None) -> np.ndarray:
        js = np.array([0] if k is None else range(1, k + 1), dtype=np.int64)
        b = philox_row_blocks(self.key, rows, (js + 1) // 2, 1)
        u1 = (_bits53(b[..., 0], b[..., 1]).astype(np.float64) + 1.0) * _SCALE
        u2 = _bits53(b[..., 2], b[..., 3]).astype(np.float64) * _SCALE
        r = np.sqrt(-2.0 * np.log(u1))
        z = np.where(((js == 0) | (js % 2 == 1))[None, :], r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2))
        return z[:, 0] if k is None else z
