"""oracle -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Two CPU checkers for the LCS table fill of the reference (/root/reference,
"wavelcs"):

* ``Restatement`` -- ctypes binding of ``oracle/lcs_oracle.c``, a plain-C
  restatement of ``lcs_cell`` (proj/include/wavelcs/cell.hpp:30-38),
  ``fill_block_scalar`` (proj/src/kernels_scalar.cpp:5-17), ``traceback``
  (proj/src/serial.cpp:36-61) and ``generate_random`` (proj/src/io.cpp:103-115),
  plus a 64-bit Hyyro bit-parallel length and a bit-row traceback.
* ``Reference`` -- ctypes binding of ``oracle/_ref/libwavelcs_ref.so``, the
  UNMODIFIED reference library compiled from its own sources by
  ``oracle/Makefile`` with the extern-"C" shim ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this package.  The product library
(``paper_1306_4627_b200``) never does.

Pinning: ``tests/test_oracle.py`` checks the restatement against every golden
vector the reference's tests hold (test_core.cpp, test_kernels.cpp,
acceptance.cpp criteria 1, 2, 4) and against the compiled reference.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liblcs_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libwavelcs_ref.so")

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_sz = ctypes.c_size_t


def build() -> None:
    """Compile the restatement and (when /root/reference exists) the reference."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _buf(data) -> tuple:
    if isinstance(data, str):
        data = data.encode("latin-1")
    arr = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    arr = np.ascontiguousarray(arr, dtype=np.uint8)
    if arr.size == 0:
        arr = np.zeros(1, dtype=np.uint8)[:0]
    return arr, arr.ctypes.data_as(_u8p), arr.size


class Restatement:
    """The plain-C restatement (oracle/lcs_oracle.c)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        lib.orc_length_cells.restype = ctypes.c_uint32
        lib.orc_length_cells.argtypes = [_u8p, _sz, _u8p, _sz]
        lib.orc_length_bitpar.restype = ctypes.c_uint32
        lib.orc_length_bitpar.argtypes = [_u8p, _sz, _u8p, _sz]
        lib.orc_length_cells_mt.restype = ctypes.c_uint32
        lib.orc_length_cells_mt.argtypes = [_u8p, _sz, _u8p, _sz, ctypes.c_int]
        lib.orc_fill_tables.restype = None
        lib.orc_fill_tables.argtypes = [_u8p, _sz, _u8p, _sz, _u32p, _u8p]
        lib.orc_traceback.restype = _sz
        lib.orc_traceback.argtypes = [_u8p, _sz, _sz, _u8p, _sz, _sz, _u8p]
        lib.orc_subsequence_bitrows.restype = ctypes.c_int64
        lib.orc_subsequence_bitrows.argtypes = [_u8p, _sz, _u8p, _sz, _u8p]
        lib.orc_brute_force.restype = ctypes.c_int64
        lib.orc_brute_force.argtypes = [_u8p, _sz, _u8p, _sz]
        lib.orc_capacity_exceeded.restype = ctypes.c_int
        lib.orc_capacity_exceeded.argtypes = [ctypes.c_uint64] * 3
        lib.orc_generate_random.restype = None
        lib.orc_generate_random.argtypes = [_sz, _u8p, _sz, ctypes.c_uint64, _u8p]
        lib.orc_strip_rows.restype = None
        lib.orc_strip_rows.argtypes = [_u8p, _sz, _u8p, _sz, _u64p, _u8p, _u8p]
        lib.orc_strip_zeros.restype = ctypes.c_uint64
        lib.orc_strip_zeros.argtypes = [_u64p, _sz]
        lib.orc_length_batch.restype = None
        lib.orc_generate_pairs.restype = None
        lib.orc_generate_pairs.argtypes = [_sz, _sz, _sz, _u8p, _sz, ctypes.c_uint64, _u8p, _u64p,
                                           _u8p, _u64p]
        lib.orc_length_batch.argtypes = [_u8p, _u64p, _u8p, _u64p, _sz, _u32p]
        self.lib = lib

    def length_cells(self, x, y) -> int:
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        return int(self.lib.orc_length_cells(xp, m, yp, n))

    def length_cells_mt(self, x, y, threads: int = 0) -> int:
        """Two-row lcs_cell loop over column strips on `threads` host threads
        (SURVEY.md 8(c) check (i) at full size)."""
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        return int(self.lib.orc_length_cells_mt(xp, m, yp, n, threads or (os.cpu_count() or 1)))

    def length_bitpar(self, x, y) -> int:
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        return int(self.lib.orc_length_bitpar(xp, m, yp, n))

    def fill_tables(self, x, y):
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        dp = np.empty((m + 1, n + 1), dtype=np.uint32)
        back = np.empty((m, n), dtype=np.uint8)
        self.lib.orc_fill_tables(xp, m, yp, n, dp.ctypes.data_as(_u32p),
                                 back.ctypes.data_as(_u8p))
        return dp, back

    def traceback(self, back: np.ndarray, x, i: int, j: int) -> bytes:
        xa, xp, m = _buf(x)
        rows, cols = back.shape
        back = np.ascontiguousarray(back, dtype=np.uint8)
        out = np.empty(max(1, min(rows, cols)), dtype=np.uint8)
        r = self.lib.orc_traceback(back.ctypes.data_as(_u8p), rows, cols, xp, i, j,
                                   out.ctypes.data_as(_u8p))
        if r == ctypes.c_size_t(-1).value:
            raise IndexError("traceback: position outside table")
        return out[:r].tobytes()

    def subsequence(self, x, y) -> bytes:
        """Reference traceback string via the full arrow table (small sizes)."""
        dp, back = self.fill_tables(x, y)
        return self.traceback(back, x, back.shape[0], back.shape[1])

    def subsequence_bitrows(self, x, y) -> bytes:
        """Reference traceback string via stored bit rows (M*N/8 bytes)."""
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        out = np.empty(max(1, min(m, n)), dtype=np.uint8)
        r = self.lib.orc_subsequence_bitrows(xp, m, yp, n, out.ctypes.data_as(_u8p))
        if r < 0:
            raise MemoryError("oracle bit-row traceback allocation failed")
        return out[:r].tobytes()

    def brute_force(self, x, y) -> int:
        xa, xp, m = _buf(x)
        ya, yp, n = _buf(y)
        r = self.lib.orc_brute_force(xp, m, yp, n)
        if r < 0:
            raise ValueError("brute_force_lcs: inputs too long for enumeration")
        return int(r)

    def capacity_exceeded(self, m: int, n: int, budget: int) -> bool:
        return bool(self.lib.orc_capacity_exceeded(m, n, budget))

    def generate_random(self, length: int, alphabet, seed: int) -> bytes:
        aa, ap, alen = _buf(alphabet)
        out = np.empty(max(1, length), dtype=np.uint8)
        self.lib.orc_generate_random(length, ap, alen, seed & (2**64 - 1), out.ctypes.data_as(_u8p))
        return out[:length].tobytes()

    def generate_pairs(self, pairs: int, lo: int, hi: int, alphabet, seed: int):
        """The C2 batch procedure (master MT19937-64 -> per-pair lengths and
        seeds -> generate_random); returns (xs, x_off, ys, y_off) numpy arrays."""
        aa, ap, alen = _buf(alphabet)
        xs = np.empty(max(1, pairs * hi), np.uint8)
        ys = np.empty(max(1, pairs * hi), np.uint8)
        xo = np.empty(pairs + 1, np.uint64)
        yo = np.empty(pairs + 1, np.uint64)
        self.lib.orc_generate_pairs(pairs, lo, hi, ap, alen, seed & (2**64 - 1),
                                    xs.ctypes.data_as(_u8p), xo.ctypes.data_as(_u64p),
                                    ys.ctypes.data_as(_u8p), yo.ctypes.data_as(_u64p))
        return xs, xo, ys, yo

    def strip_rows(self, x, ystrip, V: np.ndarray, carry_in: np.ndarray | None):
        """Rows of x over one column strip; V (uint64, ceil(ns/64)) updated in
        place; returns the per-row carry-out (uint8)."""
        xa, xp, m = _buf(x)
        ya, yp, ns = _buf(ystrip)
        cout = np.zeros(max(1, m), np.uint8)
        cin = None if carry_in is None else np.ascontiguousarray(carry_in, np.uint8)
        self.lib.orc_strip_rows(xp, m, yp, ns, V.ctypes.data_as(_u64p),
                                None if cin is None else cin.ctypes.data_as(_u8p),
                                cout.ctypes.data_as(_u8p))
        return cout[:m]

    def strip_zeros(self, V: np.ndarray, ns: int) -> int:
        return int(self.lib.orc_strip_zeros(V.ctypes.data_as(_u64p), ns))

    def length_batch(self, xs: np.ndarray, xoff: np.ndarray, ys: np.ndarray,
                     yoff: np.ndarray) -> np.ndarray:
        pairs = len(xoff) - 1
        out = np.empty(pairs, dtype=np.uint32)
        xs = np.ascontiguousarray(xs, dtype=np.uint8)
        ys = np.ascontiguousarray(ys, dtype=np.uint8)
        xoff = np.ascontiguousarray(xoff, dtype=np.uint64)
        yoff = np.ascontiguousarray(yoff, dtype=np.uint64)
        self.lib.orc_length_batch(xs.ctypes.data_as(_u8p), xoff.ctypes.data_as(_u64p),
                                  ys.ctypes.data_as(_u8p), yoff.ctypes.data_as(_u64p),
                                  pairs, out.ctypes.data_as(_u32p))
        return out


class ReferenceError_(RuntimeError):
    """An exception raised inside the reference library, re-raised by kind."""

    def __init__(self, code: int, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.code, self.kind, self.msg = code, kind, msg


_REF_KINDS = {1: "CapacityError", 2: "ConfigError", 3: "out_of_range", 4: "invalid_argument",
              5: "InputError", 9: "exception"}


class Reference:
    """The reference library itself (oracle/_ref/libwavelcs_ref.so)."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = ctypes.CDLL(path)
        c = ctypes.c_char_p
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_default_workers.restype = ctypes.c_uint
        lib.ref_check_capacity.argtypes = [_sz, _sz, _sz]
        lib.ref_lcs_length_serial.argtypes = [c, _sz, c, _sz, _sz, _u32p]
        lib.ref_lcs_length_parallel.argtypes = [c, _sz, c, _sz, ctypes.c_uint, _sz, _sz, _u32p,
                                                ctypes.POINTER(ctypes.c_double)]
        lib.ref_lcs_subsequence.argtypes = [c, _sz, c, _sz, ctypes.c_uint, _sz, ctypes.c_char_p,
                                            _sz, ctypes.POINTER(_sz),
                                            ctypes.POINTER(ctypes.c_double)]
        lib.ref_fill_tables.argtypes = [c, _sz, c, _sz, ctypes.c_uint, _sz, _u32p, _u8p]
        lib.ref_traceback.argtypes = [_u8p, _sz, _sz, c, _sz, _sz, _sz, ctypes.c_char_p,
                                      ctypes.POINTER(_sz)]
        lib.ref_brute_force.argtypes = [c, _sz, c, _sz, _u32p]
        lib.ref_generate_random.argtypes = [_sz, c, _sz, ctypes.c_uint64, ctypes.c_char_p]
        lib.ref_batch_lengths.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_void_p, _u64p, _sz,
                                          ctypes.c_uint, _u32p, ctypes.POINTER(ctypes.c_double)]
        self.lib = lib

    def _check(self, rc: int) -> None:
        if rc:
            raise ReferenceError_(rc, _REF_KINDS.get(rc, "exception"),
                                  self.lib.ref_last_error().decode("latin-1"))

    @staticmethod
    def _b(data) -> bytes:
        return data.encode("latin-1") if isinstance(data, str) else bytes(data)

    def default_workers(self) -> int:
        return int(self.lib.ref_default_workers())

    def check_capacity(self, m: int, n: int, budget: int) -> None:
        self._check(self.lib.ref_check_capacity(m, n, budget))

    def lcs_length(self, x, y, budget: int = 2 * 1024 ** 3) -> int:
        x, y = self._b(x), self._b(y)
        out = ctypes.c_uint32()
        self._check(self.lib.ref_lcs_length_serial(x, len(x), y, len(y), budget,
                                                   ctypes.byref(out)))
        return int(out.value)

    def lcs_length_parallel(self, x, y, workers: int = 0, block: int = 64,
                            budget: int = 2 ** 64 - 1) -> tuple[int, float]:
        x, y = self._b(x), self._b(y)
        out = ctypes.c_uint32()
        sec = ctypes.c_double()
        workers = workers or self.default_workers()
        self._check(self.lib.ref_lcs_length_parallel(x, len(x), y, len(y), workers, block, budget,
                                                     ctypes.byref(out), ctypes.byref(sec)))
        return int(out.value), float(sec.value)

    def lcs_subsequence(self, x, y, workers: int = 0,
                        budget: int = 2 ** 64 - 1) -> tuple[bytes, float]:
        x, y = self._b(x), self._b(y)
        cap = max(1, min(len(x), len(y)))
        out = ctypes.create_string_buffer(cap)
        n = _sz()
        sec = ctypes.c_double()
        workers = workers or self.default_workers()
        self._check(self.lib.ref_lcs_subsequence(x, len(x), y, len(y), workers, budget, out, cap,
                                                 ctypes.byref(n), ctypes.byref(sec)))
        return out.raw[: n.value], float(sec.value)

    def fill_tables(self, x, y, workers: int = 1, block: int = 64):
        x, y = self._b(x), self._b(y)
        m, n = len(x), len(y)
        dp = np.empty((m + 1, n + 1), dtype=np.uint32)
        back = np.empty((m, n), dtype=np.uint8)
        self._check(self.lib.ref_fill_tables(x, m, y, n, workers, block, dp.ctypes.data_as(_u32p),
                                             back.ctypes.data_as(_u8p)))
        return dp, back

    def traceback(self, back: np.ndarray, x, i: int, j: int) -> bytes:
        x = self._b(x)
        back = np.ascontiguousarray(back, dtype=np.uint8)
        rows, cols = back.shape
        out = ctypes.create_string_buffer(max(1, min(rows, cols)))
        n = _sz()
        self._check(self.lib.ref_traceback(back.ctypes.data_as(_u8p), rows, cols, x, len(x), i, j,
                                           out, ctypes.byref(n)))
        return out.raw[: n.value]

    def brute_force(self, x, y) -> int:
        x, y = self._b(x), self._b(y)
        out = ctypes.c_uint32()
        self._check(self.lib.ref_brute_force(x, len(x), y, len(y), ctypes.byref(out)))
        return int(out.value)

    def generate_random(self, length: int, alphabet, seed: int) -> bytes:
        a = self._b(alphabet)
        out = ctypes.create_string_buffer(max(1, length))
        self._check(self.lib.ref_generate_random(length, a, len(a), seed & (2**64 - 1), out))
        return out.raw[:length]

    def batch_lengths(self, xs: np.ndarray, xoff: np.ndarray, ys: np.ndarray, yoff: np.ndarray,
                      threads: int = 0) -> tuple[np.ndarray, float]:
        pairs = len(xoff) - 1
        out = np.empty(pairs, dtype=np.uint32)
        xs = np.ascontiguousarray(xs, dtype=np.uint8)
        ys = np.ascontiguousarray(ys, dtype=np.uint8)
        xoff = np.ascontiguousarray(xoff, dtype=np.uint64)
        yoff = np.ascontiguousarray(yoff, dtype=np.uint64)
        sec = ctypes.c_double()
        threads = threads or self.default_workers()
        self._check(self.lib.ref_batch_lengths(xs.ctypes.data, xoff.ctypes.data_as(_u64p),
                                               ys.ctypes.data, yoff.ctypes.data_as(_u64p), pairs,
                                               threads, out.ctypes.data_as(_u32p),
                                               ctypes.byref(sec)))
        return out, float(sec.value)
