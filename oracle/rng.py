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
