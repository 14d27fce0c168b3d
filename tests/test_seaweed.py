"""Semi-local LCS (seaweed combing) model behind the row-band prototype
(paper_1306_4627_b200/csrc/seaweed.cu), checked on the CPU against the
oracle's `lcs_cell` restatement (oracle/lcs_oracle.c, following
proj/src/kernels_scalar.cpp:6-16 and proj/include/wavelcs/cell.hpp:30-38):

* combing a band from the canonical start gives, for every top seaweed k,
  its exit column e_k (n = the right side);
* H(i, j) = (j - i) - #{k in [i, j): e_k < j} equals LCS(a, b[i:j]);
* bands compose exactly through C[j] = max_{i<=j} T[i] + H(i, j).

Pure-Python test model (small sizes); the device kernels are checked against
the oracle in tests/test_gpu_parity.py."""
import random

import pytest


def comb(a: bytes, b: bytes):
    m, n = len(a), len(b)
    h = [m - 1 - i for i in range(m)]   # left seaweeds, numbered bottom to top
    v = [m + j for j in range(n)]       # top seaweeds, left to right
    for i in range(m):
        for j in range(n):
            if a[i] == b[j] or h[i] > v[j]:
                h[i], v[j] = v[j], h[i]
    e = [n] * n
    for j in range(n):
        if v[j] >= m:
            e[v[j] - m] = j
    return e


def H(e, i, j):
    return (j - i) - sum(1 for k in range(i, j) if e[k] < j)


def compose(bands, b: bytes) -> int:
    n = len(b)
    T = [0] * (n + 1)
    for band in bands:
        e = comb(band, b)
        T = [max(T[i] + H(e, i, j) for i in range(j + 1)) for j in range(n + 1)]
    return T[n]


def rand_str(rng, n, alphabet):
    return bytes(rng.choice(alphabet) for _ in range(n))


@pytest.mark.parametrize("alphabet", [b"AC", b"ACGT", b"ACDEFGHIKLMNPQRSTVWY"])
def test_string_substring_lcs(restatement, alphabet):
    rng = random.Random(len(alphabet))
    for _ in range(60):
        a = rand_str(rng, rng.randint(0, 9), alphabet)
        b = rand_str(rng, rng.randint(0, 9), alphabet)
        e = comb(a, b)
        for i in range(len(b) + 1):
            for j in range(i, len(b) + 1):
                assert H(e, i, j) == restatement.length_cells(a, b[i:j]), (a, b, i, j)


@pytest.mark.parametrize("bands", [1, 2, 3, 5])
def test_band_composition(restatement, bands):
    rng = random.Random(100 + bands)
    for _ in range(40):
        alphabet = rng.choice([b"AB", b"ACGT", bytes(range(256))])
        a = rand_str(rng, rng.randint(0, 40), alphabet)
        b = rand_str(rng, rng.randint(0, 40), alphabet)
        cuts = sorted(rng.randint(0, len(a)) for _ in range(bands - 1))
        parts = [a[x:y] for x, y in zip([0] + cuts, cuts + [len(a)])]
        assert compose(parts, b) == restatement.length_cells(a, b)
