"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Bit-exact for every length and every recovered subsequence (integer/byte
work: no tolerance).  Mirrors the reference's own tests:
proj/tests/test_core.cpp, test_kernels.cpp, test_parallel.cpp, acceptance.cpp.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DNA = b"ACGT"
PROTEIN = b"ACDEFGHIKLMNPQRSTVWY"
CHILD_SEED_OFFSET = 0x9E3779B97F4A7C15  # include/wavelcs/bench.hpp:74


def rand_pairs(rng, n, lo, hi, alphabet):
    a = np.frombuffer(alphabet, dtype=np.uint8)
    xs, ys = [], []
    for _ in range(n):
        m = int(rng.integers(lo, hi + 1))
        k = int(rng.integers(lo, hi + 1))
        xs.append(a[rng.integers(0, len(a), m)].tobytes())
        ys.append(a[rng.integers(0, len(a), k)].tobytes())
    return xs, ys


def check_batch(wl, restatement, xs, ys):
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    got = wl.lcs_length_batch(xb, xo, yb, yo)
    want = restatement.length_batch(xb, xo, yb, yo)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first pair {bad[0]}: got {got[bad[0]]} want {want[bad[0]]} (m={len(xs[bad[0]])}, n={len(ys[bad[0]])})"


def test_golden_lengths(wl):
    # proj/tests/test_core.cpp:58-62
    assert wl.lcs_length(b"", b"") == 0
    assert wl.lcs_length(b"ATGC", b"ATGC") == 4
    assert wl.lcs_length(b"ABCBDAB", b"BDCABA") == 4
    assert wl.lcs_length(b"", b"ATGC") == 0


def test_golden_subsequences(wl):
    # proj/tests/test_core.cpp:69-85, test_cli.cpp:82-91
    assert wl.lcs_subsequence(b"ABCBDAB", b"BDCABA") == b"BDAB"
    assert wl.lcs_subsequence(b"ATGC", b"ATGC") == b"ATGC"
    assert wl.lcs_subsequence(b"ATGC", b"") == b""


@pytest.mark.parametrize("alphabet", [DNA, PROTEIN])
def test_batch_small_random(wl, restatement, alphabet):
    rng = np.random.default_rng(1234)
    xs, ys = rand_pairs(rng, 3000, 0, 300, alphabet)
    check_batch(wl, restatement, xs, ys)


def test_batch_c2_sample(wl, restatement):
    rng = np.random.default_rng(77)
    xs, ys = rand_pairs(rng, 4096, 200, 1000, PROTEIN)
    check_batch(wl, restatement, xs, ys)


def test_batch_edges(wl, restatement):
    rng = np.random.default_rng(5)
    a = np.arange(256, dtype=np.uint8)
    xs = [b"", b"A", b"", b"AAAA", b"A" * 1000, b"ACGT" * 3000, bytes(a), bytes(a[::-1]) * 3]
    ys = [b"", b"", b"A", b"AAAA", b"C" * 1000, b"TGCA" * 2500, bytes(a) * 2, bytes(a)]
    # large alphabet (overflows a warp's match-mask slice) and very long pairs
    for _ in range(40):
        m, n = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        xs.append(a[rng.integers(0, 256, m)].tobytes())
        ys.append(a[rng.integers(0, 256, n)].tobytes())
    xs.append(rng.integers(0, 4, 20000).astype(np.uint8).tobytes())
    ys.append(rng.integers(0, 4, 9000).astype(np.uint8).tobytes())
    check_batch(wl, restatement, xs, ys)


def test_batch_sampled_map_misses(wl, restatement):
    """A warp's first task builds with a byte -> code map sampled from the
    first 32 column bytes of each lane.  Here every column string starts with
    a run of one letter and holds its other letters (which the rows share)
    only later, so the sampled map always misses bytes: the build must fall
    back to the full presence pass and still return the oracle's lengths."""
    rng = np.random.default_rng(4242)
    letters = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWYZ", np.uint8)
    xs, ys = [], []
    for i in range(3000):
        head = int(rng.integers(33, 120))
        tail = int(rng.integers(1, 400))
        col = b"A" * head + letters[rng.integers(0, len(letters), tail)].tobytes()
        row = letters[rng.integers(0, len(letters), int(rng.integers(len(col), 1100)))].tobytes()
        xs.append(row)
        ys.append(col)
    check_batch(wl, restatement, xs, ys)


def test_batch_large_alphabet_many(wl, restatement):
    """Thousands of 256-symbol pairs: their alphabets overflow the first
    pass's mask budget and take the one-word-per-lane second pass (columns
    <= 1024) or the strip kernel (wider); also through the device entry point."""
    import torch
    rng = np.random.default_rng(99)
    a = np.arange(256, dtype=np.uint8)
    xs, ys = [], []
    for _ in range(3000):
        m, n = int(rng.integers(1, 1400)), int(rng.integers(1, 1400))
        xs.append(a[rng.integers(0, 256, m)].tobytes())
        ys.append(a[np.minimum(rng.zipf(1.3, n), 256) - 1].tobytes())
    check_batch(wl, restatement, xs, ys)
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    dev = torch.device("cuda", 0)
    d_xs = torch.from_numpy(np.concatenate([xb, np.zeros(16, np.uint8)])).to(dev)
    d_ys = torch.from_numpy(np.concatenate([yb, np.zeros(16, np.uint8)])).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(len(xs), dtype=torch.int32, device=dev)
    wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                               len(xs), int(xo[-1]), int(yo[-1]), d_out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().astype(np.uint32),
                          restatement.length_batch(xb, xo, yb, yo))


def test_batch_device_tight_buffers(wl, restatement):
    """Device buffers of exactly the strings' size (no tail padding): the
    pairs at the buffer ends take the bounds-checked sweep and the byte-gather
    chunk path; everything else the fast path."""
    import torch
    rng = np.random.default_rng(4242)
    for alphabet in (DNA, PROTEIN):
        xs, ys = rand_pairs(rng, 700, 1, 900, alphabet)
        xb, xo, yb, yo = wl.pack_pairs(xs, ys)
        dev = torch.device("cuda", 0)
        d_xs = torch.from_numpy(xb.copy()).to(dev)
        d_ys = torch.from_numpy(yb.copy()).to(dev)
        d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
        d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
        d_out = torch.zeros(len(xs), dtype=torch.int32, device=dev)
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(),
                                   d_yo.data_ptr(), len(xs), int(xo[-1]), int(yo[-1]),
                                   d_out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(d_out.cpu().numpy().astype(np.uint32),
                              restatement.length_batch(xb, xo, yb, yo))


@pytest.mark.parametrize("m,n", [(1, 1), (5, 300), (300, 5), (1000, 1000), (4097, 33), (33, 4097),
                                 (5000, 200), (12345, 6789)])
def test_single_pair_lengths(wl, restatement, m, n):
    rng = np.random.default_rng(m * 7919 + n)
    x = rng.choice(np.frombuffer(DNA, np.uint8), m).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), n).tobytes()
    assert wl.lcs_length(x, y) == restatement.length_bitpar(x, y)


def test_c1_checkpoint(wl, restatement):
    # generate_random(10000, "ACGT", 1) vs seed 1 + offset -> 6538
    x = restatement.generate_random(10000, DNA, 1)
    y = restatement.generate_random(10000, DNA, 1 + CHILD_SEED_OFFSET)
    assert wl.lcs_length(x, y) == 6538
    sub = wl.lcs_subsequence(x, y)
    assert len(sub) == 6538
    assert sub == restatement.subsequence_bitrows(x, y)


@pytest.mark.parametrize("alphabet", [DNA, PROTEIN, b"AC"])
def test_subsequence_random(wl, restatement, alphabet):
    rng = np.random.default_rng(len(alphabet))
    a = np.frombuffer(alphabet, np.uint8)
    for _ in range(60):
        m, n = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        x = a[rng.integers(0, len(a), m)].tobytes()
        y = a[rng.integers(0, len(a), n)].tobytes()
        assert wl.lcs_subsequence(x, y) == restatement.subsequence(x, y), (x, y)


def test_capacity_semantics(wl):
    # proj/tests/test_core.cpp:122-126
    with pytest.raises(wl.CapacityError):
        wl.lcs_length(b"ATGC", b"ATGC", 16)
    assert wl.lcs_length(b"ATGC", b"ATGC", 1024) == 4
    with pytest.raises(wl.CapacityError):
        wl.lcs_length(b"", b"", 1)


# ---------------------------------------------------------------- fixtures
import gzip  # noqa: E402
import json  # noqa: E402
import os  # noqa: E402
import subprocess  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_golden_small_pairs_reference_tracebacks(wl):
    """300 pairs whose lengths and tracebacks came from the reference itself."""
    data = json.load(open(os.path.join(GOLDEN, "small_pairs.json")))
    xs = [bytes.fromhex(c["x"]) for c in data["cases"]]
    ys = [bytes.fromhex(c["y"]) for c in data["cases"]]
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    got = wl.lcs_length_batch(xb, xo, yb, yo)
    assert got.tolist() == [c["length"] for c in data["cases"]]
    for x, y, c in zip(xs, ys, data["cases"]):
        assert wl.lcs_length(x, y) == c["length"]
        assert wl.lcs_subsequence(x, y).hex() == c["subsequence"]


def test_golden_c1_subsequence(wl):
    data = json.load(open(os.path.join(GOLDEN, "c1.json")))
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c1")
    assert wl.lcs_subsequence(x, y).decode() == data["subsequence"]


def test_golden_c2_sample(wl):
    import ctypes
    data = json.load(open(os.path.join(GOLDEN, "c2_sample.json")))
    pairs = 512
    xs = np.empty(pairs * 1000, np.uint8)
    ys = np.empty(pairs * 1000, np.uint8)
    xo = np.empty(pairs + 1, np.uint64)
    yo = np.empty(pairs + 1, np.uint64)
    a = np.frombuffer(PROTEIN, np.uint8)
    wl._check(wl.lib.wlcs_generate_pairs(pairs, 200, 1000, a.ctypes.data, len(a), 20130619,
                                         xs.ctypes.data,
                                         xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                         ys.ctypes.data,
                                         yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    got = wl.lcs_length_batch(xs[: int(xo[-1])], xo, ys[: int(yo[-1])], yo)
    assert got.tolist() == data["lengths"]


def test_golden_c3_reference_subsequence(wl):
    """Config C3 (100k x ~100k mutated DNA): the recovered string must equal
    the reference's own traceback (fixture generated by oracle/_ref)."""
    data = json.load(gzip.open(os.path.join(GOLDEN, "c3.json.gz"), "rt"))
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c3")
    assert wl.lcs_length(x, y, wl.NO_BUDGET) == data["length"]
    sub = wl.lcs_subsequence(x, y, wl.NO_BUDGET)
    assert len(sub) == data["length"]
    assert sub.decode() == data["subsequence"]


def test_batch_device_entry_point(wl, restatement):
    import torch
    rng = np.random.default_rng(21)
    xs, ys = rand_pairs(rng, 1000, 0, 700, PROTEIN)
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    dev = torch.device("cuda", 0)
    d_xs = torch.from_numpy(np.concatenate([xb, np.zeros(16, np.uint8)])).to(dev)
    d_ys = torch.from_numpy(np.concatenate([yb, np.zeros(16, np.uint8)])).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(1000, dtype=torch.int32, device=dev)
    wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                               1000, int(xo[-1]), int(yo[-1]), d_out.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().astype(np.uint32),
                          restatement.length_batch(xb, xo, yb, yo))


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_large_configs_properties(wl, restatement, name):
    """C4 (1M x 1M DNA) and C5 (2M x 500k Zipf bytes) at full size through
    size-independent properties, plus a 200k prefix against the oracle."""
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair(name)
    L = wl.lcs_length(x, y, wl.NO_BUDGET)
    assert 0 < L <= min(len(x), len(y))
    assert wl.lcs_length(y, x, wl.NO_BUDGET) == L                  # symmetry
    c = x[-1:]
    assert wl.lcs_length(x + c, y + c, wl.NO_BUDGET) == L + 1      # append (acceptance 4)
    px, py = x[:200000], y[:150000]
    assert wl.lcs_length(px, py, wl.NO_BUDGET) == restatement.length_bitpar(px, py)


def test_cpp_facade_reference_unit_cases():
    """The reference's unit cases against the C++ facade (tests/cpp)."""
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_facade")
    assert os.path.exists(exe), "build() must produce tests/cpp/test_facade"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


# ---- cell-wavefront (DPX) variant: same integer results as the oracle ----

def check_batch_variant(wl, restatement, xs, ys, variant):
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    got = wl.lcs_length_batch(xb, xo, yb, yo, variant=variant)
    want = restatement.length_batch(xb, xo, yb, yo)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first pair {bad[0]}: got {got[bad[0]]} want {want[bad[0]]}"


@pytest.mark.parametrize("alphabet", [DNA, PROTEIN])
def test_wavefront_batch_random(wl, restatement, alphabet):
    rng = np.random.default_rng(99)
    xs, ys = rand_pairs(rng, 2000, 0, 400, alphabet)
    check_batch_variant(wl, restatement, xs, ys, wl.VARIANT_WAVEFRONT)


def test_wavefront_batch_edges(wl, restatement):
    rng = np.random.default_rng(6)
    a = np.arange(256, dtype=np.uint8)
    xs = [b"", b"A", b"", b"AAAA", b"A" * 1000, bytes(a), b"AC" * 2100, b"G" * 5000]
    ys = [b"", b"", b"A", b"AAAA", b"C" * 1000, bytes(a[::-1]), b"CA" * 2100, b"G" * 4500]
    for _ in range(30):  # 256-symbol alphabet, bands of 128 rows with ragged ends
        m, n = int(rng.integers(1, 700)), int(rng.integers(1, 700))
        xs.append(a[rng.integers(0, 256, m)].tobytes())
        ys.append(a[rng.integers(0, 256, n)].tobytes())
    check_batch_variant(wl, restatement, xs, ys, wl.VARIANT_WAVEFRONT)


def test_wavefront_batch_bands_and_rows_per_lane(wl, restatement):
    """The DPX batch kernel's band structure: every rows-per-lane value R = 4..16
    (rows 1..1024 in one band), several bands per pair (rows > 1024, the
    boundary row handed through shared memory), and the column limit (2048)
    on both sides of it (wider pairs go to the pair kernel)."""
    rng = np.random.default_rng(4242)
    xs, ys = [], []
    for rows in list(range(1, 1100, 37)) + [1024, 1025, 2048, 2049, 3000, 5000]:
        for alphabet in (DNA, PROTEIN):
            al = np.frombuffer(alphabet, np.uint8)
            n = int(rng.integers(1, min(rows, 2048) + 1))
            xs.append(rng.choice(al, rows).tobytes())
            ys.append(rng.choice(al, n).tobytes())
    for n in (2047, 2048, 2049):
        xs.append(rng.choice(np.frombuffer(DNA, np.uint8), 3000).tobytes())
        ys.append(rng.choice(np.frombuffer(DNA, np.uint8), n).tobytes())
    check_batch_variant(wl, restatement, xs, ys, wl.VARIANT_WAVEFRONT)


@pytest.mark.parametrize("m,n", [(1, 1), (127, 129), (129, 127), (1000, 1000), (4096, 33),
                                 (5000, 200), (20000, 7000), (150000, 70000)])
def test_wavefront_pair(wl, restatement, m, n):
    rng = np.random.default_rng(m * 7 + n)
    x = rng.choice(np.frombuffer(DNA, np.uint8), m).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), n).tobytes()
    want = restatement.length_bitpar(x, y)
    assert wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT) == want
    assert wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_BITPARALLEL) == want


def test_wavefront_pair_rebase(wl, restatement):
    """Identical strings: the LCS grows by one per column, so the 16-bit
    packed values must be re-based (every 8192 steps) well before 2^16."""
    rng = np.random.default_rng(77)
    x = rng.choice(np.frombuffer(DNA, np.uint8), 100_000).tobytes()
    assert wl.lcs_length(x, x, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT) == 100_000
    y = x[:60_000] + b"T" * 20_000 + x[60_000:90_000]  # 110,000 columns
    assert wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT) == \
        restatement.length_bitpar(x, y)


# ---- row-band decomposition (semi-local LCS prototype, csrc/seaweed.cu) ----

@pytest.mark.parametrize("bands", [1, 2, 3, 4])
@pytest.mark.parametrize("alphabet", [DNA, PROTEIN, bytes(range(256))])
def test_rowbands_random(wl, restatement, bands, alphabet):
    rng = np.random.default_rng(bands * 31 + len(alphabet))
    al = np.frombuffer(alphabet, np.uint8)
    for m, n in [(1, 1), (1, 40), (40, 1), (255, 257), (700, 300), (300, 700), (2500, 1900)]:
        x = rng.choice(al, m).tobytes()
        y = rng.choice(al, n).tobytes()
        assert wl.lcs_length_rowbands(x, y, bands) == restatement.length_bitpar(x, y), (m, n)


def test_rowbands_edges(wl, restatement):
    assert wl.lcs_length_rowbands(b"", b"ACGT", 3) == 0
    assert wl.lcs_length_rowbands(b"ACGT", b"", 3) == 0
    assert wl.lcs_length_rowbands(b"ACGT", b"ACGT", 9) == 4  # more bands than rows
    x = b"A" * 3000
    assert wl.lcs_length_rowbands(x, x, 4) == 3000          # identical strings
    assert wl.lcs_length_rowbands(x, b"C" * 2000, 4) == 0   # no match at all
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c1")                        # 10k x 10k
    assert wl.lcs_length_rowbands(x, y, 4) == 6538


def test_wavefront_c1_checkpoint(wl):
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c1")
    assert wl.lcs_length(x, y, variant=wl.VARIANT_WAVEFRONT) == 6538


# ---- multi-GPU column split, played in order on ONE device ----
# (a slice's fill only runs once its inbox is complete, so no kernel waits on
# another; the carries still travel through the inbox words exactly as they do
# between GPUs)

def _colsplit_in_order(wl, x, y, world):
    from paper_1306_4627_b200 import multigpu
    bounds = multigpu.colsplit_bounds(len(y), world)
    words = wl.colsplit_inbox_words(len(x))
    inbox_f = [wl.device_alloc(4 * words) for _ in range(world)]
    inbox_r = [wl.device_alloc(4 * words) for _ in range(world)]
    vf, vr = [None] * world, [None] * world
    try:
        for g in range(world):  # forward: slice g reads inbox_f[g], writes inbox_f[g+1]
            lo, hi = bounds[g]
            vf[g], _ = wl.colsplit_fill(x, y, lo, hi, wl.COLSPLIT_FORWARD,
                                        in_fwd=inbox_f[g] if g > 0 else 0,
                                        out_fwd=inbox_f[g + 1] if g + 1 < world else 0)
        for g in reversed(range(world)):  # reverse: right to left
            lo, hi = bounds[g]
            _, vr[g] = wl.colsplit_fill(x, y, lo, hi, wl.COLSPLIT_REVERSE,
                                        in_rev=inbox_r[g] if g + 1 < world else 0,
                                        out_rev=inbox_r[g - 1] if g > 0 else 0)
    finally:
        for p in inbox_f + inbox_r:
            wl.device_free(p)
    return multigpu.colsplit_combine(bounds, vf, vr, len(y))


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_colsplit_in_order(wl, restatement, world):
    rng = np.random.default_rng(world)
    x = rng.choice(np.frombuffer(DNA, np.uint8), 20011).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), 30007).tobytes()
    assert _colsplit_in_order(wl, x, y, world) == restatement.length_bitpar(x, y)


def test_colsplit_c1(wl):
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c1")
    assert _colsplit_in_order(wl, x, y, 2) == 6538


def test_single_process_multi_gpu_entry_points(wl, restatement):
    rng = np.random.default_rng(3)
    xs, ys = rand_pairs(rng, 500, 0, 300, PROTEIN)
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    want = restatement.length_batch(xb, xo, yb, yo)
    assert np.array_equal(wl.lcs_length_batch_multi(xb, xo, yb, yo, 1), want)
    x, y = xs[7] * 20, ys[9] * 30
    assert wl.lcs_length_strips(x, y, 1) == restatement.length_bitpar(x, y)
    n = wl.device_count()
    with pytest.raises(wl.ConfigError):
        wl.lcs_length_batch_multi(xb, xo, yb, yo, n + 1)
    with pytest.raises(wl.ConfigError):
        wl.lcs_length_strips(b"ACGT" * 5000, b"GATTACA" * 5000, n + 1)


# ---- the reference's full tables on the device ----

@pytest.mark.parametrize("m,n,alphabet", [(1, 1, DNA), (7, 6, DNA), (37, 129, DNA), (300, 200, PROTEIN),
                                          (1000, 999, DNA), (64, 2050, PROTEIN)])
def test_fill_tables_match_oracle(wl, restatement, m, n, alphabet):
    rng = np.random.default_rng(m + 3 * n)
    a = np.frombuffer(alphabet, np.uint8)
    x = a[rng.integers(0, len(a), m)].tobytes()
    y = a[rng.integers(0, len(a), n)].tobytes()
    dp, back = wl.fill_tables(x, y)
    want_dp, want_back = restatement.fill_tables(x, y)
    assert np.array_equal(dp, want_dp)
    assert np.array_equal(back, want_back)


def test_fill_tables_match_reference_tests(wl, restatement):
    # acceptance.cpp:101-138 style: 200 seeded small cases, tables identical
    # to the (restated) serial fill, tracebacks identical
    rng = np.random.default_rng(2024)
    for _ in range(200):
        m, n = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        x = rng.choice(np.frombuffer(b"AC", np.uint8), m).tobytes()
        y = rng.choice(np.frombuffer(b"AC", np.uint8), n).tobytes()
        dp, back = wl.fill_tables(x, y)
        want_dp, want_back = restatement.fill_tables(x, y)
        assert np.array_equal(dp, want_dp) and np.array_equal(back, want_back)
        assert restatement.traceback(back, x, m, n) == wl.lcs_subsequence(x, y)


def test_fill_tables_capacity(wl):
    with pytest.raises(wl.CapacityError):
        wl.fill_tables(b"ATGC", b"ATGC", 16)
    dp, back = wl.fill_tables(b"", b"ATGC")
    assert dp.shape == (1, 5) and not dp.any() and back.shape == (0, 4)


# ---- traceback shapes: skinny tables, far-from-diagonal paths, 256 symbols ----

@pytest.mark.parametrize("m,n", [(1, 50000), (50000, 1), (3, 20000), (20000, 3), (2000, 9000),
                                 (9000, 2000), (20000, 3000), (257, 255)])
def test_subsequence_shapes(wl, restatement, m, n):
    # skinny tables drive the walk's Left runs to column 0 and the
    # speculative walk's fallback (paths far from the diagonal)
    rng = np.random.default_rng(m + 31 * n)
    x = rng.choice(np.frombuffer(DNA, np.uint8), m).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), n).tobytes()
    assert wl.lcs_subsequence(x, y) == restatement.subsequence(x, y)


def test_subsequence_long_left_jumps(wl, restatement):
    """Rows whose next match lies hundreds of columns to the left (the warp
    walker's window is 96 columns: these take its serial row step), runs of
    identical symbols, and blocks whose candidate walks never merge."""
    rng = np.random.default_rng(97)
    cases = [
        (b"Z" * 3, b"Z" + b"A" * 3000),
        (b"AB" * 400 + b"Z", b"Z" + b"C" * 5000 + b"AB" * 100),
        (b"Q" + b"AC" * 2000, b"AC" * 100 + b"G" * 4000 + b"Q"),
        (b"A" * 1500, b"A" * 700),
        (b"A" * 700, b"A" * 1500),
    ]
    for _ in range(4):
        m, n = int(rng.integers(300, 3000)), int(rng.integers(3000, 12000))
        x = rng.choice(np.frombuffer(b"AC", np.uint8), m).tobytes()
        y = rng.choice(np.frombuffer(b"ACGT" * 3 + b"NNNNNNNNNNNNNNNNNNNNNNNNN", np.uint8), n).tobytes()
        cases.append((x, y))
    for x, y in cases:
        assert wl.lcs_subsequence(x, y) == restatement.subsequence(x, y), (len(x), len(y))


def test_subsequence_byte_alphabet(wl, restatement):
    rng = np.random.default_rng(256)
    for m, n in [(3000, 2500), (700, 4000), (4000, 700)]:
        x = rng.integers(0, 256, m).astype(np.uint8).tobytes()
        y = rng.integers(0, 256, n).astype(np.uint8).tobytes()
        assert wl.lcs_length(x, y) == restatement.length_bitpar(x, y)
        assert wl.lcs_subsequence(x, y) == restatement.subsequence(x, y)


def test_subsequence_similar_strings(wl, restatement):
    # C3-like: a mutated copy keeps the path near the diagonal; shifted copies
    # move it far off the diagonal (the walk's window must follow)
    from paper_1306_4627_b200 import workloads
    x = restatement.generate_random(12000, DNA, 77)
    for y in (workloads.mutate(x, 5), x[3000:] + x[:3000], b"ACGT" * 500 + x):
        assert wl.lcs_subsequence(x, y) == restatement.subsequence(x, y)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_large_configs_golden(wl, name):
    """Full-size C4 / C5 lengths equal the CPU oracle's (tests/golden/
    large_configs.json, made by tests/golden/make_large_golden.py); both
    fill variants and the in-order column split."""
    import json
    import os
    from paper_1306_4627_b200 import workloads
    with open(os.path.join(os.path.dirname(__file__), "golden", "large_configs.json")) as f:
        want = json.load(f)[name]["lcs_length"]
    x, y = workloads.config_pair(name)
    assert wl.lcs_length(x, y, wl.NO_BUDGET) == want
    assert wl.lcs_length(x, y, wl.NO_BUDGET, variant=wl.VARIANT_WAVEFRONT) == want
    if name == "c4":
        assert _colsplit_in_order(wl, x, y, 2) == want


def test_batch_many_tiny_pairs(wl, restatement):
    # 200k pairs of 0..40 symbols: exercises the plan/scan/scatter at scale and
    # the empty-pair early outs (proj/tests/test_parallel.cpp:236-242)
    rng = np.random.default_rng(11)
    pairs = 200_000
    lm = rng.integers(0, 41, pairs)
    ln = rng.integers(0, 41, pairs)
    a = np.frombuffer(DNA, np.uint8)
    xb = a[rng.integers(0, 4, int(lm.sum()))].tobytes()
    yb = a[rng.integers(0, 4, int(ln.sum()))].tobytes()
    xo = np.concatenate([[0], np.cumsum(lm)]).astype(np.uint64)
    yo = np.concatenate([[0], np.cumsum(ln)]).astype(np.uint64)
    got = wl.lcs_length_batch(xb, xo, yb, yo)
    want = restatement.length_batch(np.frombuffer(xb, np.uint8), xo, np.frombuffer(yb, np.uint8), yo)
    assert np.array_equal(got, want)


def test_batch_device_plan_paths(wl, restatement):
    """The plan + scatter run as one cooperative launch when all its blocks fit
    the device at once (up to ~300k pairs on a B200) and as two kernels beyond:
    one device-entry call of each size, against the oracle."""
    import torch
    rng = np.random.default_rng(12)
    dev = torch.device("cuda", 0)
    a = np.frombuffer(DNA, np.uint8)
    for pairs in (150_000, 400_000):
        lm = rng.integers(0, 33, pairs)
        ln = rng.integers(0, 33, pairs)
        xb = a[rng.integers(0, 4, int(lm.sum()))]
        yb = a[rng.integers(0, 4, int(ln.sum()))]
        xo = np.concatenate([[0], np.cumsum(lm)]).astype(np.uint64)
        yo = np.concatenate([[0], np.cumsum(ln)]).astype(np.uint64)
        d_xs = torch.from_numpy(np.concatenate([xb, np.zeros(16, np.uint8)])).to(dev)
        d_ys = torch.from_numpy(np.concatenate([yb, np.zeros(16, np.uint8)])).to(dev)
        d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
        d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
        d_out = torch.zeros(pairs, dtype=torch.int32, device=dev)
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                                   pairs, int(xo[-1]), int(yo[-1]), d_out.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(d_out.cpu().numpy().astype(np.uint32),
                              restatement.length_batch(xb, xo, yb, yo)), pairs


@pytest.mark.parametrize("alphabet", [DNA, PROTEIN, bytes(range(7, 47))])
def test_batch_every_lane_shape(wl, restatement, alphabet):
    # The batch planner picks, from the shorter string's word count W, a lane
    # shape (S lanes x K words, K <= 10), a mask layout (K <= 4, the 10-word
    # rows of K = 9-10, or 4-word slots) and, for W = 5-8, the half-length
    # S = 2 shape queued last.  Every W from 1 to 40 words at both ends of
    # its 32-column range, as the x and as the y string, with row strings
    # from 1 byte to well past the column string, plus a skewed mix.
    rng = np.random.default_rng(20261020)
    a = np.frombuffer(alphabet, dtype=np.uint8)
    xs, ys = [], []
    for w in range(1, 41):
        for cols in (32 * w - 31, 32 * w):
            for rows in (1, 15, 17, cols, cols + 1, 3 * cols + 5):
                rows = max(rows, cols)  # the column string is the shorter one
                c = a[rng.integers(0, len(a), cols)].tobytes()
                r = a[rng.integers(0, len(a), rows)].tobytes()
                if rng.integers(0, 2):
                    xs.append(c); ys.append(r)
                else:
                    xs.append(r); ys.append(c)
    xr, yr = rand_pairs(rng, 1500, 1, 1400, alphabet)
    check_batch(wl, restatement, xs + xr, ys + yr)


# ---- round 2: device second pass, caller-stream ordering, column-split liveness

def _device_batch(wl, xs, ys, stream=None, tight=False):
    import torch
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    dev = torch.device("cuda", 0)
    pad = np.zeros(0 if tight else 16, np.uint8)
    d_xs = torch.from_numpy(np.concatenate([xb, pad])).to(dev)
    d_ys = torch.from_numpy(np.concatenate([yb, pad])).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.full((len(xs),), -1, dtype=torch.int32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream()
    wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                               len(xs), int(xo[-1]), int(yo[-1]), d_out.data_ptr(), s.cuda_stream)
    return (xb, xo, yb, yo), d_out, s


def test_batch_device_wide_pairs_second_pass(wl, restatement):
    """The device entry point has no host fallback: pairs wider than the first
    pass's lane shapes (shorter string > 10,240 bytes) and byte alphabets with
    all 256 values in one 1024-column block (257 codes) are finished by the
    device second pass in column blocks (bitpar_wide.cu)."""
    import torch
    rng = np.random.default_rng(2026)
    a = np.arange(256, dtype=np.uint8)
    xs, ys = [], []
    for k in range(40):
        m = int(rng.integers(10000, 26000))
        n = int(rng.integers(10241, 21000))
        alpha = a if k % 2 else np.frombuffer(DNA, np.uint8)
        xs.append(alpha[rng.integers(0, len(alpha), m)].tobytes())
        ys.append(alpha[rng.integers(0, len(alpha), n)].tobytes())
    for _ in range(300):  # 1024-4096 columns, every byte value present
        m, n = int(rng.integers(1024, 4097)), int(rng.integers(1024, 4097))
        xs.append(a[rng.integers(0, 256, m)].tobytes())
        ys.append(np.concatenate([a, a[rng.integers(0, 256, n - 256)]])[rng.permutation(n)].tobytes())
    for _ in range(200):  # mixed with ordinary first-pass pairs
        m, n = int(rng.integers(1, 900)), int(rng.integers(1, 900))
        xs.append(rng.choice(np.frombuffer(PROTEIN, np.uint8), m).tobytes())
        ys.append(rng.choice(np.frombuffer(PROTEIN, np.uint8), n).tobytes())
    (xb, xo, yb, yo), d_out, _ = _device_batch(wl, xs, ys)
    torch.cuda.synchronize()
    want = restatement.length_batch(xb, xo, yb, yo)
    got = d_out.cpu().numpy().astype(np.uint32)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[0]}: {got[bad[0]]} vs {want[bad[0]]}"
    # the host entry point routes the wide pairs to the strip kernel instead
    assert np.array_equal(wl.lcs_length_batch(xb, xo, yb, yo), want)


def test_batch_device_is_ordered_on_caller_stream(wl, restatement):
    """Asynchronous device entry on a side stream: inputs written by a kernel
    on that stream just before the call, and the output read after it on the
    same stream, without any host synchronisation in between."""
    import torch
    rng = np.random.default_rng(77)
    xs, ys = rand_pairs(rng, 4000, 100, 1000, PROTEIN)
    xb, xo, yb, yo = wl.pack_pairs(xs, ys)
    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(side):
        d_xs = torch.zeros(len(xb) + 16, dtype=torch.uint8, device=dev)
        d_ys = torch.zeros(len(yb) + 16, dtype=torch.uint8, device=dev)
        d_xs[: len(xb)].copy_(torch.from_numpy(np.array(xb)), non_blocking=False)
        d_ys[: len(yb)].copy_(torch.from_numpy(np.array(yb)), non_blocking=False)
        d_xo = torch.from_numpy(np.array(xo.view(np.int64))).to(dev)
        d_yo = torch.from_numpy(np.array(yo.view(np.int64))).to(dev)
        d_out = torch.full((len(xs),), -1, dtype=torch.int32, device=dev)
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(),
                                   d_yo.data_ptr(), len(xs), len(xb), len(yb), d_out.data_ptr(),
                                   side.cuda_stream)
        res = d_out.to(torch.int64) + 0  # consumer kernel on the same stream
    side.synchronize()
    assert np.array_equal(res.cpu().numpy().astype(np.uint32),
                          restatement.length_batch(xb, xo, yb, yo))


def test_length_device_honours_stream(wl, restatement):
    import torch
    rng = np.random.default_rng(5)
    x = rng.choice(np.frombuffer(DNA, np.uint8), 30000).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), 20000).tobytes()
    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(side):
        d_x = torch.zeros(len(x) + 16, dtype=torch.uint8, device=dev)
        d_y = torch.zeros(len(y) + 16, dtype=torch.uint8, device=dev)
        torch.cuda._sleep(20_000_000)  # keep the side stream busy before the copies land
        d_x[: len(x)].copy_(torch.from_numpy(np.frombuffer(x, np.uint8).copy()))
        d_y[: len(y)].copy_(torch.from_numpy(np.frombuffer(y, np.uint8).copy()))
        out = ctypes.c_uint32()
        wl._check(wl.lib.wlcs_length_device(d_x.data_ptr(), len(x), d_y.data_ptr(), len(y),
                                            wl.VARIANT_BITPARALLEL, ctypes.byref(out),
                                            side.cuda_stream))
    assert out.value == restatement.length_bitpar(x, y)


@pytest.mark.parametrize("slices,max_ctas", [(2, 4), (3, 6), (4, 8), (4, 16), (2, 0), (4, 0)])
def test_colsplit_slices_run_concurrently(wl, restatement, slices, max_ctas):
    """The column split's fused hand-off with every slice's producer and
    consumer RUNNING AT THE SAME TIME (one launch, one CTA pool per slice and
    direction) and -- for max_ctas > 0 -- far fewer warps per pool than strips
    per problem: the liveness case of the shared-ticket design."""
    rng = np.random.default_rng(slices * 100 + max_ctas)
    x = rng.choice(np.frombuffer(DNA, np.uint8), 6000).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), 180_000).tobytes()
    assert wl.colsplit_emulate(x, y, slices, max_ctas) == restatement.length_bitpar(x, y)


def test_colsplit_concurrent_byte_alphabet(wl, restatement):
    rng = np.random.default_rng(9)
    a = np.arange(256, dtype=np.uint8)
    x = a[np.minimum(rng.zipf(1.1, 5000), 256) - 1].tobytes()
    y = a[np.minimum(rng.zipf(1.1, 70_000), 256) - 1].tobytes()
    assert wl.colsplit_emulate(x, y, 3, 6) == restatement.length_bitpar(x, y)


# ---- bounded-memory (banded) traceback --------------------------------------

@pytest.mark.parametrize("m,n,alphabet,row_cap", [
    (3000, 2500, DNA, 500_000), (5000, 700, PROTEIN, 300_000), (2000, 5000, DNA, 900_000),
    (2049, 1999, b"AC", 400_000), (12000, 12000, DNA, 4 << 20), (8192, 130, DNA, 120_000)])
def test_subsequence_banded_matches_reference(wl, restatement, m, n, alphabet, row_cap):
    """With the traceback's device memory capped far below M * N / 8 the
    string comes from row bands recomputed from checkpoints -- it must still
    be the reference's traceback byte for byte (LEFT rule)."""
    rng = np.random.default_rng(m * 31 + n)
    a = np.frombuffer(alphabet, np.uint8)
    x = a[rng.integers(0, len(a), m)].tobytes()
    y = a[rng.integers(0, len(a), n)].tobytes()
    assert row_cap < m * n // 8
    assert wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=row_cap) == restatement.subsequence_bitrows(x, y)


def test_golden_c3_subsequence_banded(wl):
    """C3 (100k x ~100k mutated DNA; the full stored traceback needs 1.25 GB)
    with a 24 MB cap: the reference's own traceback string (tests/golden)."""
    import gzip
    import json
    import os
    from paper_1306_4627_b200 import workloads
    with gzip.open(os.path.join(os.path.dirname(__file__), "golden", "c3.json.gz"), "rt") as f:
        data = json.load(f)
    x, y = workloads.config_pair("c3")
    sub = wl.lcs_subsequence(x, y, wl.NO_BUDGET, row_cap=24 << 20)
    assert len(sub) == data["length"]
    assert sub.decode() == data["subsequence"]


def test_subsequence_cap_too_small(wl):
    x = b"ACGT" * 5000
    with pytest.raises(MemoryError):
        wl.lcs_subsequence(x, x[::-1], wl.NO_BUDGET, row_cap=1000)


def test_batch_c2_full_against_oracle(wl, restatement):
    """The whole C2 batch (65,536 protein pairs, BASELINE configs[1]) through
    the host entry point against the oracle's lengths -- every pair, not a
    sample (the bench's equivalence gate runs on the reference's sample)."""
    xs, xo, ys, yo = restatement.generate_pairs(65536, 200, 1000, PROTEIN, 20130619)
    got = wl.lcs_length_batch(xs[: xo[-1]], xo, ys[: yo[-1]], yo)
    want = restatement.length_batch(xs, xo, ys, yo)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("chunks,taper", [(2, 1), (3, 0), (5, 1), (7, 1)])
def test_batch_pipeline_chunkings(wl, restatement, monkeypatch, chunks, taper):
    """The host batch's copy/compute pipeline cut into 2-7 chunks, equal or
    tapered (capi.cu batch_pipe_copies): every chunking gives the oracle's
    lengths, long (strip-kernel) pairs included."""
    monkeypatch.setenv("WLCS_BATCH_CHUNKS", str(chunks))
    monkeypatch.setenv("WLCS_BATCH_TAPER", str(taper))
    gx, gxo, gy, gyo = restatement.generate_pairs(60000, 150, 700, PROTEIN, 1234 + chunks)
    xl = [gx[gxo[k]:gxo[k + 1]].tobytes() for k in range(60000)]
    yl = [gy[gyo[k]:gyo[k + 1]].tobytes() for k in range(60000)]
    # a few pairs wider than the lane shapes (finished by the strip kernel)
    rng = np.random.default_rng(chunks)
    al = np.frombuffer(PROTEIN, np.uint8)
    for p in rng.choice(60000, 3, replace=False):
        xl[p] = rng.choice(al, 12000).tobytes()
        yl[p] = rng.choice(al, 15000).tobytes()
    xs, xo, ys, yo = wl.pack_pairs(xl, yl)
    got = wl.lcs_length_batch(xs, xo, ys, yo)
    want = restatement.length_batch(xs, xo, ys, yo)
    assert np.array_equal(got, want)


def test_single_pair_pageable_and_pinned_inputs(wl, restatement):
    """Single-pair H2D goes through the pinned stage ring for pageable
    buffers larger than one 4 MB stage; page-locked buffers go direct."""
    import ctypes as ct
    rng = np.random.default_rng(8)
    x = rng.choice(np.frombuffer(DNA, np.uint8), 9_000_000).tobytes()
    y = rng.choice(np.frombuffer(DNA, np.uint8), 3000).tobytes()
    want = restatement.length_bitpar(x, y)
    assert wl.lcs_length(x, y, wl.NO_BUDGET) == want
    p = wl.lib.wlcs_host_alloc(len(x))
    try:
        ct.memmove(p, x, len(x))
        out = ct.c_uint32()
        wl._check(wl.lib.wlcs_length_ex(p, len(x), y, len(y), wl.NO_BUDGET, wl.VARIANT_BITPARALLEL,
                                        ct.byref(out)))
        assert out.value == want
    finally:
        wl.lib.wlcs_host_free(ct.c_void_p(p))
