"""Seeded synthetic input generators shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the motif-search method: no encoding
into codes, no Hamming distance, no search.  It only produces ASCII DNA
byte arrays ``uint8[n, t]`` over ``b"ACGT"`` (plus the planted ground truth
as strings), so the CUDA path and the oracle consume identical inputs.

FM model (section I.B, section IV.B; SPEC.md:154-166;
readings 2-3 of DESIGN.md section 3):
  * background bases iid uniform over A,C,G,T (25% each);
  * consensus: l iid uniform bases;
  * per sequence: an offset uniform on [0, t-l]; d DISTINCT positions of the
    consensus chosen uniformly (partial Fisher-Yates); each chosen base is
    replaced by (b + 1 + U{0,1,2}) mod 4 -- a uniformly chosen DIFFERENT base,
    so every instance is at Hamming distance exactly d (the FM model);
  * the instance overwrites the background at the offset.

RNG: SplitMix64 (Steele, Lea & Flood 2014), written out below so the byte
stream is identical on every platform and numpy version.  Bases take the top
two bits of one output; bounded integers use Lemire's multiply-shift with
rejection (exactly uniform).  The draw order is: consensus bases, then for
each sequence i = 0..n-1: t background bases, the offset, d position draws,
d replacement draws.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ALPHABET = b"ACGT"
_MASK64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & _MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)

    def bounded(self, n: int) -> int:
        """Uniform integer in [0, n) (Lemire 2019, 64-bit, with rejection)."""
        if n <= 0:
            raise ValueError("bounded(n) needs n >= 1")
        x = self.next_u64()
        m = x * n
        low = m & _MASK64
        if low < n:
            thresh = ((1 << 64) - n) % n
            while low < thresh:
                x = self.next_u64()
                m = x * n
                low = m & _MASK64
        return m >> 64

    def base(self) -> int:
        return self.next_u64() >> 62


@dataclass
class Plant:
    seq: int
    offset: int
    instance: str
    mutated_positions: list[int]


@dataclass
class PlantRecord:
    n: int
    t: int
    l: int
    d: int
    seed: int
    consensus: str
    plants: list[Plant] = field(default_factory=list)


def _bases(rng: SplitMix64, count: int) -> bytearray:
    return bytearray(ALPHABET[rng.base()] for _ in range(count))


def generate_fm(n: int, t: int, l: int, d: int, seed: int) -> tuple[np.ndarray, PlantRecord]:
    """FM-model dataset: returns (uint8[n, t] ASCII, PlantRecord)."""
    if not (n >= 1 and 1 <= l <= t and 0 <= d <= l):
        raise ValueError(f"InvalidSpec n={n} t={t} l={l} d={d}")
    rng = SplitMix64(seed)
    consensus = _bases(rng, l)
    rows = np.empty((n, t), dtype=np.uint8)
    rec = PlantRecord(n, t, l, d, seed, consensus.decode())
    for i in range(n):
        row = _bases(rng, t)
        off = rng.bounded(t - l + 1)
        idx = list(range(l))
        for k in range(d):  # partial Fisher-Yates: d distinct positions
            j = k + rng.bounded(l - k)
            idx[k], idx[j] = idx[j], idx[k]
        pos = sorted(idx[:d])
        inst = bytearray(consensus)
        for p in idx[:d]:
            b = ALPHABET.index(inst[p])
            inst[p] = ALPHABET[(b + 1 + rng.bounded(3)) % 4]
        row[off:off + l] = inst
        rows[i] = np.frombuffer(bytes(row), dtype=np.uint8)
        rec.plants.append(Plant(i, off, inst.decode(), pos))
    return rows, rec


def random_sequences(n: int, t: int, seed: int) -> np.ndarray:
    """n iid-uniform sequences of length t (no plant)."""
    rng = SplitMix64(seed ^ 0x5EED5EED)
    out = np.empty((n, t), dtype=np.uint8)
    for i in range(n):
        out[i] = np.frombuffer(bytes(_bases(rng, t)), dtype=np.uint8)
    return out


def from_strings(strings: list[str]) -> np.ndarray:
    """Equal-length strings -> uint8[n, t] (bytes as given, any case)."""
    if not strings or len({len(s) for s in strings}) != 1:
        raise ValueError("need >= 1 strings of equal length")
    return np.frombuffer("".join(strings).encode("latin-1"),
                         dtype=np.uint8).reshape(len(strings), -1).copy()


# BASELINE.json configs[0..4] (n, t, l, d); index 3 is the headline (15,4).
BASELINE_CONFIGS = [
    dict(name="(9,2) n=20 t=600", n=20, t=600, l=9, d=2),
    dict(name="(11,3) n=20 t=600", n=20, t=600, l=11, d=3),
    dict(name="(13,3) n=20 t=600", n=20, t=600, l=13, d=3),
    dict(name="(15,4) n=20 t=600", n=20, t=600, l=15, d=4),
    dict(name="(16,5) n=20 t=1000", n=20, t=1000, l=16, d=5),
]
SEEDS = (1, 2, 3)
