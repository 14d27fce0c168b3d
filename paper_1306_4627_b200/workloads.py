"""Synthetic inputs for the BASELINE.json configurations (no datasets exist).

Every generator is seeded and deterministic on any platform:
  * C1 / C4: generate_random (std::mt19937_64, alphabet[r % |A|];
    proj/src/io.cpp:103-115) with the reference's child-seed offset
    (proj/include/wavelcs/bench.hpp:74).
  * C2: wlcs_generate_pairs (include/wavelcs_capi.h): per pair lengths
    200 + r % 801, 20-letter protein alphabet, per-string seeds from a master
    std::mt19937_64.
  * C3: DNA of 100k + per-position mutation: one uniform
    draw u per source symbol (numpy MT19937, seed given): u < 0.10 substitute
    by one of the 3 other bases, u < 0.12 delete, u < 0.14 insert a uniform
    base then copy, else copy.
  * C5: 2M x 500k bytes, Zipf(s=1.1) over 256 ranks by inverse CDF,
    rank k -> byte k-1 (numpy MT19937).
"""
from __future__ import annotations

import numpy as np

DNA = b"ACGT"
PROTEIN = b"ACDEFGHIKLMNPQRSTVWY"
CHILD_SEED_OFFSET = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def generate_random(length: int, alphabet: bytes, seed: int) -> bytes:
    from . import generate_random as _gen
    return _gen(length, alphabet, seed & MASK64)


def mutate(x: bytes, seed: int) -> bytes:
    rng = np.random.Generator(np.random.MT19937(seed))
    n = len(x)
    u = rng.random(n)
    sub = rng.integers(1, 4, n)
    ins = rng.integers(0, 4, n)
    src = np.frombuffer(x, np.uint8)
    lut = np.zeros(256, np.int64)
    for i, c in enumerate(DNA):
        lut[c] = i
    dna = np.frombuffer(DNA, np.uint8)
    code = lut[src]
    substituted = dna[(code + sub) % 4]
    out_sym = np.where(u < 0.10, substituted, src)
    keep = ~((u >= 0.10) & (u < 0.12))
    insert = (u >= 0.12) & (u < 0.14)
    # each kept source position emits [inserted base?] + symbol
    counts = keep.astype(np.int64) + (insert & keep).astype(np.int64)
    out = np.empty(int(counts.sum()), np.uint8)
    pos = np.cumsum(counts) - counts
    ins_pos = pos[insert & keep]
    out[ins_pos] = dna[ins[insert & keep]]
    sym_pos = (pos + (insert & keep).astype(np.int64))[keep]
    out[sym_pos] = out_sym[keep]
    return out.tobytes()


def zipf_bytes(n: int, seed: int, s: float = 1.1) -> bytes:
    rng = np.random.Generator(np.random.MT19937(seed))
    w = 1.0 / np.arange(1, 257, dtype=np.float64) ** s
    cdf = np.cumsum(w / w.sum())
    idx = np.searchsorted(cdf, rng.random(n), side="right")
    return np.minimum(idx, 255).astype(np.uint8).tobytes()


def config_pair(name: str, seed: int = 20130619) -> tuple[bytes, bytes]:
    """(x, y) of a single-pair configuration c1 | c3 | c4 | c5."""
    if name == "c1":
        return (generate_random(10000, DNA, 1),
                generate_random(10000, DNA, 1 + CHILD_SEED_OFFSET))
    if name == "c3":
        x = generate_random(100000, DNA, seed)
        return x, mutate(x, seed + 1)
    if name == "c4":
        return (generate_random(1000000, DNA, seed),
                generate_random(1000000, DNA, seed + CHILD_SEED_OFFSET))
    if name == "c5":
        return zipf_bytes(2000000, seed), zipf_bytes(500000, seed + 1)
    raise ValueError(name)
