"""Vacancy configurations: seeded sampling, quarter restriction, enumeration (disorder.py:29-113).

The draws are the reference's exactly: SeedSequence(master_seed, spawn_key=(level, replicate))
-> PCG64 -> Generator.random(nunits) < p, reproduced bit-for-bit by the C port in libhx
(`hx_sample_masks`, csrc/hx_rng.cuh), vectorised over replicates and host threads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import PartitionMap, Supercell

__all__ = ["DefectConfiguration", "SeedSpec", "sample_defects", "sample_masks", "restrict", "enumerate_configs",
           "keys_from_words", "words_from_keys"]

ENUMERATION_CAP = 24


def keys_from_words(words: np.ndarray) -> list:
    """uint64 [n, w] little-endian words -> canonical Python-int bitmask keys (disorder.py:40-46)."""
    words = np.ascontiguousarray(words, dtype=np.uint64)
    nb = words.shape[1] * 8
    raw = words.tobytes()
    return [int.from_bytes(raw[i * nb:(i + 1) * nb], "little") for i in range(words.shape[0])]


def words_from_keys(keys, nunits: int) -> np.ndarray:
    w = max(1, (nunits + 63) // 64)
    buf = b"".join(int(k).to_bytes(8 * w, "little") for k in keys)
    return np.frombuffer(buf, dtype=np.uint64).reshape(len(keys), w).copy() if keys else np.zeros((0, w), np.uint64)


@dataclass(frozen=True, eq=False)
class DefectConfiguration:
    supercell: Supercell
    vacant: frozenset

    def __post_init__(self):
        if self.vacant and (min(self.vacant) < 0 or max(self.vacant) >= self.supercell.nunits):
            raise ValueError("vacant unit index out of range")

    @property
    def key(self) -> int:
        mask = 0
        for u in self.vacant:
            mask |= 1 << u
        return mask

    @classmethod
    def from_key(cls, supercell: Supercell, key: int) -> "DefectConfiguration":
        return cls(supercell, frozenset(u for u in range(supercell.nunits) if key >> u & 1))

    def __len__(self) -> int:
        return len(self.vacant)


@dataclass(frozen=True)
class SeedSpec:
    """Stream id (master_seed, level, replicate) (disorder.py:57-68)."""

    master_seed: int
    level: int = 0
    replicate: int = 0

    def generator(self) -> np.random.Generator:
        return np.random.default_rng(np.random.SeedSequence(self.master_seed, spawn_key=(self.level, self.replicate)))


def _c_port_ok(seed, level, rep_hi) -> bool:
    return 0 <= seed < 2**64 and 0 <= level < 2**64 and 0 <= rep_hi < 2**64


def sample_masks(nunits: int, p_vac: float, master_seed: int, level: int, rep0: int, count: int) -> np.ndarray:
    """uint64 words [count, ceil(nunits/64)] for replicates rep0 .. rep0+count-1."""
    if not 0.0 <= p_vac <= 1.0:
        raise ValueError(f"p_vac must be in [0, 1], got {p_vac}")
    if _c_port_ok(master_seed, level, rep0 + count):
        return _lib.host_sample_masks(master_seed, level, rep0, count, p_vac, nunits)
    # seeds wider than 64 bits: numpy's own SeedSequence (identical algorithm, arbitrary width)
    out = np.zeros((count, max(1, (nunits + 63) // 64)), dtype=np.uint64)
    for i in range(count):
        d = SeedSpec(master_seed, level, rep0 + i).generator().random(nunits) < p_vac
        for u in np.flatnonzero(d):
            out[i, u >> 6] |= np.uint64(1) << np.uint64(u & 63)
    return out


def sample_defects(supercell: Supercell, p_vac: float, seed: SeedSpec) -> DefectConfiguration:
    """Each removable unit vacant independently with probability p_vac (disorder.py:71-81)."""
    w = sample_masks(supercell.nunits, p_vac, seed.master_seed, seed.level, seed.replicate, 1)
    return DefectConfiguration.from_key(supercell, keys_from_words(w)[0])


def restrict(config: DefectConfiguration, partition: PartitionMap, r: int) -> DefectConfiguration:
    """Parent outcome restricted to quarter r, re-indexed onto the subcell (disorder.py:84-94)."""
    if config.supercell is not partition.parent:
        raise ValueError("configuration does not live on the partition's parent")
    if not 1 <= r <= partition.R:
        raise ValueError(f"subdomain label out of range: {r}")
    vac = frozenset(int(partition.unit_map[u]) for u in config.vacant if partition.unit_assignment[u] == r)
    return DefectConfiguration(partition.subcell(r), vac)


def restrict_words(parent_words: np.ndarray, partition: PartitionMap) -> np.ndarray:
    """Vectorised restriction of parent masks -> [n, 4, sub_words] (r = 1..4 in axis 1)."""
    return _lib.restrict_masks(parent_words, partition.parent.nunits, partition.unit_assignment,
                               partition.unit_map, partition.subcells[0].nunits)


def enumerate_configs(supercell: Supercell, p_vac: float, cap: int = ENUMERATION_CAP):
    """All 2^N outcomes with binomial weights (disorder.py:97-113)."""
    if not 0.0 <= p_vac <= 1.0:
        raise ValueError(f"p_vac must be in [0, 1], got {p_vac}")
    n = supercell.nunits
    if n > cap:
        raise ValueError(f"{n} removable units exceed the enumeration cap of {cap}; use Monte Carlo sampling instead")
    wts = [p_vac**j * (1.0 - p_vac) ** (n - j) for j in range(n + 1)]
    for mask in range(1 << n):
        yield DefectConfiguration.from_key(supercell, mask), wts[bin(mask).count("1")]
