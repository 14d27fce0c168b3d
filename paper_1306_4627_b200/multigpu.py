"""Host-side multi-GPU planning (one process per GPU, torch.distributed).

Two decompositions:

* Batch sharding (config C2): pairs are independent units; rank r takes a
  contiguous pair range balanced by cells (sum m_k * n_k).  No data-path
  collective; only the lengths come back (per-rank D2H or an all_gather).
* Column strips (config C4): the column string is cut into word-aligned
  strips, one per rank; every row's carry leaving strip g enters strip g+1.
  Rows are processed in bands of `band_rows`; after each band, rank g sends
  the band's carry bits (band_rows bits) to rank g+1 (NCCL send/recv over
  NVLink in the GPU path, gloo in the CPU tests), so rank g works on band b
  while rank g+1 works on band b-1 (pipelined block wavefront, efficiency
  B / (B + G - 1) for B bands on G ranks).  The LCS length is the sum over
  strips of the zero bits of each strip's final V (one all_reduce).
"""
from __future__ import annotations

import numpy as np


def shard_pairs(x_off: np.ndarray, y_off: np.ndarray, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pair range [lo, hi) of `rank`, balanced by cells."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    m = np.diff(np.asarray(x_off, dtype=np.int64))
    n = np.diff(np.asarray(y_off, dtype=np.int64))
    pairs = len(m)
    if pairs == 0:
        return 0, 0
    cum = np.concatenate([[0], np.cumsum(m * n + 1)])  # +1: empty pairs still count
    total = cum[-1]
    lo = int(np.searchsorted(cum, total * rank / world, side="left"))
    hi = int(np.searchsorted(cum, total * (rank + 1) / world, side="left"))
    if rank == world - 1:
        hi = pairs
    return min(lo, pairs), min(hi, pairs)


def strip_bounds(n_cols: int, world: int, align_bits: int = 64) -> list[tuple[int, int]]:
    """Column ranges [c0, c1) per rank; every boundary is a multiple of
    align_bits (so a strip's top-word carry is the strip's carry)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    words = -(-n_cols // align_bits)
    bounds = []
    for g in range(world):
        w0 = words * g // world
        w1 = words * (g + 1) // world
        bounds.append((min(n_cols, w0 * align_bits), min(n_cols, w1 * align_bits)))
    return bounds


def band_ranges(rows: int, band_rows: int) -> list[tuple[int, int]]:
    if band_rows < 1:
        raise ValueError("band_rows must be >= 1")
    return [(r, min(rows, r + band_rows)) for r in range(0, rows, band_rows)]


def pack_carries(bits: np.ndarray) -> np.ndarray:
    """Per-row carry bits (uint8 0/1) -> packed bytes for the wire."""
    return np.packbits(np.asarray(bits, np.uint8), bitorder="little")


def unpack_carries(packed: np.ndarray, rows: int) -> np.ndarray:
    return np.unpackbits(np.asarray(packed, np.uint8), count=rows, bitorder="little")
