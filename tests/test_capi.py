"""C-ABI boundary checks that need no GPU.

* the library loads and exports every function include/wavelcs_capi.h
  declares;
* without a usable CUDA device every compute entry point fails loudly with
  NoDeviceError (there is no CPU fallback);
* host-only semantics that must match the reference exactly:
  check_capacity (src/tables.cpp:9-24) including its message, and
  generate_random (src/io.cpp:103-115);
* the Python mirror maps statuses onto the reference's exception types.
"""
import ctypes
import json
import hashlib
import os
import re

import numpy as np
import pytest

import paper_1306_4627_b200 as wl

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DNA = b"ACGT"


def declared_functions():
    text = open(os.path.join(ROOT, "include", "wavelcs_capi.h")).read()
    return sorted(set(re.findall(r"\b(wlcs_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(wl.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert wl.lib.wlcs_abi_version() == 1


def test_facade_symbols_exported():
    out = os.popen(f"nm -DC --defined-only {wl.LIB_PATH}").read()
    for sym in ("wavelcs::lcs_length(", "wavelcs::lcs_subsequence(", "wavelcs::check_capacity(",
                "wavelcs::lcs_length_batch(", "wavelcs::generate_random("):
        assert sym in out, sym


def test_sm100a_code_in_library():
    out = os.popen(f"cuobjdump -lelf {wl.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out[:500]


@pytest.mark.skipif(wl.device_count() > 0, reason="a GPU is visible")
def test_no_cpu_fallback():
    with pytest.raises(wl.NoDeviceError):
        wl.lcs_length(b"ACGT", b"AGT")
    with pytest.raises(wl.NoDeviceError):
        wl.lcs_subsequence(b"ACGT", b"AGT")
    xb, xo, yb, yo = wl.pack_pairs([b"AC"], [b"CA"])
    with pytest.raises(wl.NoDeviceError):
        wl.lcs_length_batch(xb, xo, yb, yo)


def test_capacity_semantics():
    # test_core.cpp:122-126; check_capacity counts the (0,0) cell
    with pytest.raises(wl.CapacityError) as e:
        wl.check_capacity(4, 4, 16)
    assert str(e.value) == "tables for M=4, N=4 need 116 bytes, over the 16-byte budget"
    wl.check_capacity(4, 4, 1024)
    with pytest.raises(wl.CapacityError):
        wl.check_capacity(0, 0, 1)
    wl.check_capacity(10**6, 10**6, wl.NO_BUDGET)
    with pytest.raises(wl.CapacityError) as e:
        wl.check_capacity(2**40, 2**40, 2**63)
    assert "more than 2^64" in str(e.value)


def test_capacity_checked_before_device():
    # the budget error must win over any device error (reference check order)
    with pytest.raises(wl.CapacityError):
        wl.lcs_length(b"ATGC", b"ATGC", 16)


def test_capacity_message_matches_reference():
    import oracle
    if not os.path.exists(oracle.REFERENCE_SO):
        pytest.skip("oracle/_ref not built")
    ref = oracle.Reference()
    for m, n, b in [(4, 4, 16), (100, 7, 999), (0, 0, 1)]:
        with pytest.raises(oracle.ReferenceError_) as r:
            ref.check_capacity(m, n, b)
        with pytest.raises(wl.CapacityError) as o:
            wl.check_capacity(m, n, b)
        assert r.value.msg == str(o.value)


def test_generate_random_matches_reference(restatement):
    for seed in (1, 320, 1 + 0x9E3779B97F4A7C15):
        assert wl.generate_random(1000, DNA, seed) == restatement.generate_random(1000, DNA, seed)
    with pytest.raises(ValueError):
        wl.generate_random(10, b"", 1)


def test_generate_pairs_fixture():
    data = json.load(open(os.path.join(HERE, "golden", "c2_sample.json")))
    pairs = 512
    xs = np.empty(pairs * 1000, np.uint8)
    ys = np.empty(pairs * 1000, np.uint8)
    xo = np.empty(pairs + 1, np.uint64)
    yo = np.empty(pairs + 1, np.uint64)
    a = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
    wl._check(wl.lib.wlcs_generate_pairs(pairs, 200, 1000, a.ctypes.data, len(a), 20130619,
                                         xs.ctypes.data,
                                         xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                         ys.ctypes.data,
                                         yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    assert hashlib.sha256(xs[: int(xo[-1])].tobytes()).hexdigest() == data["x_sha256"]
    assert hashlib.sha256(ys[: int(yo[-1])].tobytes()).hexdigest() == data["y_sha256"]
    m, n = np.diff(xo.astype(np.int64)), np.diff(yo.astype(np.int64))
    assert m.min() >= 200 and m.max() <= 1000 and n.min() >= 200 and n.max() <= 1000


def test_invalid_offsets_rejected():
    xs = np.zeros(8, np.uint8)
    off_bad = np.array([0, 5, 3], np.uint64)
    off_ok = np.array([0, 2, 4], np.uint64)
    with pytest.raises((ValueError, wl.NoDeviceError)):
        wl.lcs_length_batch(xs, off_bad, xs, off_ok)


def test_workloads_deterministic():
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair("c3")
    assert len(x) == 100000 and abs(len(y) - 100000) < 1000
    assert workloads.config_pair("c3") == (x, y)
    z = np.frombuffer(workloads.zipf_bytes(100000, 7), np.uint8)
    top = np.bincount(z, minlength=256).argmax()
    assert top == 0 and 0.15 < (z == 0).mean() < 0.26   # Zipf(1.1): p(rank 1) ~ 0.207
