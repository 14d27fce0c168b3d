"""Host-side multi-GPU planning (one process per GPU, torch.distributed).

Two decompositions:

* Batch sharding (config C2): pairs are independent units; rank r takes a
  contiguous pair range balanced by cells (sum m_k * n_k).  No data-path
  collective; only the lengths come back (per-rank D2H or an all_gather).
* Column split (config C4): the column string is cut into slices, one per
  rank; every row's carry leaving slice g enters slice g+1.  On the GPU the
  carries travel inside the fill (wlcs_colsplit_fill): the producer's strip
  kernel stores one self-validating word per 16 rows straight into the
  consumer's inbox over NVLink (IPC peer pointer), the consumer's kernel
  polls it -- a pipelined block wavefront with no host round trips.  With the
  bidirectional split (forward top half, reversed bottom half) the LCS length
  is max_k F[k] + R[k] over the middle row, combined with one all_gather of
  per-slice zero counts and one MAX all_reduce (colsplit_combine_dist).
  The CPU tests run the same host logic over gloo with the oracle standing in
  for the device fill (carry bits sent per band of rows).
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


def colsplit_bounds(n_cols: int, world: int) -> list[tuple[int, int]]:
    """Column slices [lo, hi) per rank for wlcs_colsplit_fill (32-aligned)."""
    return strip_bounds(n_cols, world, align_bits=32)


def zero_bits(words: np.ndarray, width: int) -> np.ndarray:
    """0/1 array (uint8, length width): 1 where the bit of V is ZERO.  words are
    little-endian bit vectors (uint32 from the device, uint64 from the oracle)."""
    w = np.ascontiguousarray(words)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:width]
    return (1 - bits).astype(np.uint8)


def colsplit_combine(bounds, v_fwd, v_rev, n_cols: int) -> int:
    """LCS length from every slice's final forward / reverse vectors (one
    process holding all slices): max_k F[k] + R[k]."""
    zf = np.concatenate([zero_bits(v, hi - lo) for (lo, hi), v in zip(bounds, v_fwd)])
    # reversed problem: column r is original column n-1-r; slice g covers
    # reversed columns [n - hi, n - lo), so the reversed order is g = G-1 .. 0
    zr = np.concatenate([zero_bits(v, hi - lo)
                         for (lo, hi), v in reversed(list(zip(bounds, v_rev)))])
    F = np.concatenate([[0], np.cumsum(zf, dtype=np.int64)])
    R = np.concatenate([[0], np.cumsum(zr, dtype=np.int64)])
    assert len(F) == n_cols + 1 and len(R) == n_cols + 1
    return int(np.max(F + R[::-1]))


def colsplit_local(lo: int, hi: int, v_fwd, v_rev):
    """This slice's zero totals and the per-k local parts of F and R
    (k = lo .. hi): F_loc[k-lo] = zeros of v_fwd below k-lo,
    R_loc[k-lo] = zeros of v_rev below hi-k."""
    zf = zero_bits(v_fwd, hi - lo)
    zr = zero_bits(v_rev, hi - lo)
    f_loc = np.concatenate([[0], np.cumsum(zf, dtype=np.int64)])
    r_cum = np.concatenate([[0], np.cumsum(zr, dtype=np.int64)])
    r_loc = r_cum[::-1]  # index k-lo -> r_cum[hi-k]
    return int(f_loc[-1]), int(r_cum[-1]), f_loc, r_loc


def colsplit_combine_dist(lo: int, hi: int, v_fwd, v_rev, dist, device=None) -> int:
    """Distributed combine: one all_gather of (forward, reverse) zero totals,
    then the slice's max of F + R and one MAX all_reduce."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    tf, tr, f_loc, r_loc = colsplit_local(lo, hi, v_fwd, v_rev)
    mine = torch.tensor([tf, tr], dtype=torch.int64, device=device)
    allt = [torch.zeros(2, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allt, mine)
    tot = torch.stack(allt).cpu().numpy()
    pref_f = int(tot[:rank, 0].sum())       # forward zeros left of the slice
    suf_r = int(tot[rank + 1:, 1].sum())    # reverse zeros of the slices to the right
    best = torch.tensor([int(np.max(f_loc + r_loc)) + pref_f + suf_r], dtype=torch.int64,
                        device=device)
    dist.all_reduce(best, op=dist.ReduceOp.MAX)
    return int(best.item())
