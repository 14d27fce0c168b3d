"""Pins the CPU oracle (oracle/lcs_oracle.c) to the reference.

Golden vectors of the reference's own tests (proj/tests/test_core.cpp,
test_kernels.cpp, test_parallel.cpp, acceptance.cpp) and direct comparison
with the reference library compiled from /root/reference sources
(oracle/_ref) and with the committed fixtures it generated (tests/golden).
CPU only.
"""
import gzip
import itertools
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
DNA = b"ACGT"
OFF = 0x9E3779B97F4A7C15


def _ref_or_skip():
    import oracle
    if not os.path.exists(oracle.REFERENCE_SO):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return oracle.Reference()


def test_lcs_cell_examples(restatement):
    # test_core.cpp:18-30 -- match -> Diag, tie -> Left, up > left -> Up
    dp, back = restatement.fill_tables(b"A", b"A")
    assert dp[1, 1] == 1 and back[0, 0] == 0
    dp, back = restatement.fill_tables(b"A", b"G")
    assert dp[1, 1] == 0 and back[0, 0] == 2
    dp, back = restatement.fill_tables(b"GX", b"YG")
    # cell (2,2): x=X, y=G mismatch; up = c[1][2] = 1, left = c[2][1] = 0 -> Up
    assert dp[2, 2] == 1 and back[1, 1] == 1


def test_classic_pair(restatement):
    # test_core.cpp:50-56, 74-85
    assert restatement.length_cells(b"ABCBDAB", b"BDCABA") == 4
    assert restatement.length_bitpar(b"ABCBDAB", b"BDCABA") == 4
    assert restatement.brute_force(b"ABCBDAB", b"BDCABA") == 4
    assert restatement.subsequence(b"ABCBDAB", b"BDCABA") == b"BDAB"
    assert restatement.subsequence_bitrows(b"ABCBDAB", b"BDCABA") == b"BDAB"


def test_identity_and_empty(restatement):
    # test_core.cpp:32-48, 58-72
    assert restatement.length_bitpar(b"ATGC", b"ATGC") == 4
    assert restatement.subsequence(b"ATGC", b"ATGC") == b"ATGC"
    dp, back = restatement.fill_tables(b"ATGC", b"ATGC")
    assert all(back[k, k] == 0 for k in range(4))
    assert restatement.length_bitpar(b"", b"ATGC") == 0
    assert restatement.length_cells(b"", b"") == 0
    dp, back = restatement.fill_tables(b"ATGC", b"ATGCA")
    assert restatement.traceback(back, b"ATGC", 0, 5) == b""
    with pytest.raises(IndexError):
        restatement.traceback(restatement.fill_tables(b"ATGC", b"AT")[1], b"ATGC", 5, 2)


def test_all_same_and_no_match(restatement):
    # test_kernels.cpp:94-102
    assert restatement.length_bitpar(b"A" * 300, b"A" * 200) == 200
    assert restatement.length_bitpar(b"A" * 300, b"C" * 200) == 0


def test_exhaustive_binary_up_to_7(restatement):
    # acceptance.cpp:66-96 -- every {A,C} pair of lengths <= 7 vs brute force
    universe = [bytes(s) for L in range(8) for s in itertools.product(b"AC", repeat=L)]
    bad = 0
    for x in universe:
        for y in universe:
            bf = restatement.brute_force(x, y)
            if restatement.length_cells(x, y) != bf or restatement.length_bitpar(x, y) != bf:
                bad += 1
    assert len(universe) ** 2 == 65025 and bad == 0


def test_bitpar_equals_cells_random(restatement):
    rng = np.random.default_rng(11)
    for alpha in (b"AC", DNA, b"ACDEFGHIKLMNPQRSTVWY", bytes(range(256))):
        a = np.frombuffer(alpha, np.uint8)
        for _ in range(60):
            x = a[rng.integers(0, len(a), int(rng.integers(0, 300)))].tobytes()
            y = a[rng.integers(0, len(a), int(rng.integers(0, 300)))].tobytes()
            assert restatement.length_bitpar(x, y) == restatement.length_cells(x, y)
            assert restatement.subsequence_bitrows(x, y) == restatement.subsequence(x, y)


def test_append_property(restatement):
    # acceptance.cpp:149-168
    rng = np.random.Generator(np.random.MT19937(0xA99E9D))
    for _ in range(100):
        x = restatement.generate_random(int(rng.integers(0, 401)), DNA, int(rng.integers(0, 2**63)))
        y = restatement.generate_random(int(rng.integers(0, 401)), DNA, int(rng.integers(0, 2**63)))
        c = DNA[int(rng.integers(0, 4)):][:1]
        assert restatement.length_bitpar(x + c, y + c) == restatement.length_bitpar(x, y) + 1


def test_strip_decomposition(restatement):
    # column strips chained by one carry bit per row
    x = restatement.generate_random(4000, DNA, 3)
    y = restatement.generate_random(3001, DNA, 4)
    from paper_1306_4627_b200 import multigpu
    for world in (1, 2, 3, 5):
        carries = None
        total = 0
        for c0, c1 in multigpu.strip_bounds(len(y), world):
            V = np.full(max(1, (c1 - c0 + 63) // 64), 2**64 - 1, np.uint64)
            carries = restatement.strip_rows(x, y[c0:c1], V, carries)
            total += restatement.strip_zeros(V, c1 - c0)
        assert total == restatement.length_bitpar(x, y)


def test_golden_small_pairs(restatement):
    data = json.load(open(os.path.join(GOLDEN, "small_pairs.json")))
    assert len(data["cases"]) == 300
    for case in data["cases"]:
        x, y = bytes.fromhex(case["x"]), bytes.fromhex(case["y"])
        assert restatement.length_bitpar(x, y) == case["length"]
        assert restatement.subsequence(x, y).hex() == case["subsequence"]


def test_golden_c1(restatement):
    data = json.load(open(os.path.join(GOLDEN, "c1.json")))
    x = restatement.generate_random(10000, DNA, 1)
    y = restatement.generate_random(10000, DNA, 1 + OFF)
    assert data["length"] == 6538  # SURVEY.md 8(c) checkpoint
    assert restatement.length_bitpar(x, y) == 6538
    assert restatement.subsequence_bitrows(x, y).decode() == data["subsequence"]


def test_checkpoint_20k(restatement):
    x = restatement.generate_random(20000, DNA, 1)
    y = restatement.generate_random(20000, DNA, 1 + OFF)
    assert restatement.length_bitpar(x, y) == 13061


@pytest.mark.slow
def test_checkpoint_100k(restatement):
    x = restatement.generate_random(100000, DNA, 1)
    y = restatement.generate_random(100000, DNA, 1 + OFF)
    assert restatement.length_bitpar(x, y) == 65344  # SURVEY.md 8(c), reference-measured


def test_golden_c3_fixture_consistent(restatement):
    path = os.path.join(GOLDEN, "c3.json.gz")
    if not os.path.exists(path):
        pytest.skip("c3 fixture not generated")
    from paper_1306_4627_b200 import workloads
    data = json.load(gzip.open(path, "rt"))
    x, y = workloads.config_pair("c3")
    assert (len(x), len(y)) == (data["m"], data["n"])
    assert restatement.length_bitpar(x, y) == data["length"]


def test_restatement_matches_reference_tables():
    ref = _ref_or_skip()
    import oracle
    res = oracle.Restatement()
    rng = np.random.Generator(np.random.MT19937(0xACCE5507))
    for _ in range(40):
        x = res.generate_random(int(rng.integers(0, 300)), DNA, int(rng.integers(0, 2**63)))
        y = res.generate_random(int(rng.integers(0, 300)), DNA, int(rng.integers(0, 2**63)))
        dp_r, back_r = ref.fill_tables(x, y, workers=3, block=7)
        dp_o, back_o = res.fill_tables(x, y)
        assert np.array_equal(dp_r, dp_o) and np.array_equal(back_r, back_o)
        sub = ref.traceback(back_r, x, len(x), len(y))
        assert sub == res.subsequence(x, y) == res.subsequence_bitrows(x, y)
        assert ref.lcs_length(x, y) == res.length_bitpar(x, y)


def test_generate_random_matches_reference():
    ref = _ref_or_skip()
    import oracle
    res = oracle.Restatement()
    for seed in (0, 1, 320, 1 + OFF, 2**64 - 1):
        assert res.generate_random(777, DNA, seed) == ref.generate_random(777, DNA, seed)


def test_capacity_formula_matches_reference():
    ref = _ref_or_skip()
    import oracle
    res = oracle.Restatement()
    for m, n, budget in [(4, 4, 16), (4, 4, 1024), (0, 0, 1), (0, 0, 4), (20724, 20724, 2**31),
                         (20725, 20725, 2**31), (10**6, 10**6, 2**64 - 1)]:
        try:
            ref.check_capacity(m, n, budget)
            raised = False
        except oracle.ReferenceError_ as e:
            raised = e.kind == "CapacityError"
        assert raised == res.capacity_exceeded(m, n, budget), (m, n, budget)


def test_oracle_generate_pairs_matches_library(restatement):
    """The reference arm of bench.py builds its C2 inputs with the oracle's
    restatement of the generator (it must not load the product library);
    both must produce the same bytes."""
    import ctypes

    import paper_1306_4627_b200 as wl
    P = 2000
    xs, xo, ys, yo = restatement.generate_pairs(P, 200, 1000, b"ACDEFGHIKLMNPQRSTVWY", 20130619)
    a = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
    xs2, ys2 = np.empty(P * 1000, np.uint8), np.empty(P * 1000, np.uint8)
    xo2, yo2 = np.empty(P + 1, np.uint64), np.empty(P + 1, np.uint64)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    wl._check(wl.lib.wlcs_generate_pairs(ctypes.c_size_t(P), ctypes.c_size_t(200),
                                         ctypes.c_size_t(1000), a.ctypes.data, ctypes.c_size_t(20),
                                         ctypes.c_uint64(20130619), xs2.ctypes.data,
                                         xo2.ctypes.data_as(u64p), ys2.ctypes.data,
                                         yo2.ctypes.data_as(u64p)))
    assert np.array_equal(xo, xo2) and np.array_equal(yo, yo2)
    assert np.array_equal(xs[: xo[-1]], xs2[: xo2[-1]]) and np.array_equal(ys[: yo[-1]], ys2[: yo2[-1]])


def test_cells_mt_equals_two_row_loop(restatement):
    """The multi-threaded two-row lcs_cell loop used for the full-size C4/C5
    goldens (SURVEY.md 8(c) check (i)) against the one-thread loop."""
    rng = np.random.default_rng(17)
    for t in range(60):
        m, n = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        k = int(rng.integers(1, 6))
        x = bytes(rng.integers(65, 65 + k, m).astype(np.uint8))
        y = bytes(rng.integers(65, 65 + k, n).astype(np.uint8))
        assert restatement.length_cells_mt(x, y, int(rng.integers(1, 9))) == restatement.length_cells(x, y)


def test_large_goldens_two_oracles_agree():
    """at the full C4 / C5 sizes (which the reference cannot
    run: 5 TB of tables) the two-row lcs_cell loop (i) and the 64-bit Hyyro
    length (ii) agree (tests/golden/make_large_golden*.py)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "large_configs.json")) as f:
        g = json.load(f)
    for name in ("c4", "c5"):
        assert g[name]["lcs_length_cells"] == g[name]["lcs_length"], name
