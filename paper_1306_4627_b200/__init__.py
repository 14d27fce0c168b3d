"""paper_1306_4627_b200 -- B200-native LCS table fill ("wavelcs" drop-in).

Python mirror of the reference's operator interface for the hot path
(/root/reference/proj/include/wavelcs/serial.hpp:24-30,
 /root/reference/proj/include/wavelcs/parallel.hpp:92-93) on top of the
C-ABI library ``_lib/libwavelcs_b200.so`` (include/wavelcs_capi.h).

Same names, argument meaning and error behaviour as the reference:

* ``lcs_length(x, y, memory_budget=DEFAULT_MEMORY_BUDGET)``
      -> int; raises ``CapacityError`` exactly when the reference's
      ``check_capacity`` would (src/tables.cpp:9-24).
* ``lcs_subsequence(x, y, memory_budget=...)``
      -> bytes identical to ``traceback(lcs_fill_parallel(x, y).back, x, M, N)``
      (src/serial.cpp:36-61, LEFT tie-break of cell.hpp:27-38).
* ``lcs_length_batch(xs, x_off, ys, y_off)`` -> numpy uint32 lengths (new).

There is no CPU fallback: importing works without a GPU (so the CPU test
suite can check the library and its exports), but every compute call raises
``NoDeviceError`` when CUDA is unavailable, and importing raises
``ImportError`` if the compiled library is missing.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence as _Seq

import numpy as np

__all__ = [
    "CapacityError", "ConfigError", "InputError", "EquivalenceError", "CudaError",
    "NoDeviceError", "DEFAULT_MEMORY_BUDGET", "NO_BUDGET", "VARIANT_BITPARALLEL",
    "VARIANT_WAVEFRONT", "lcs_length", "lcs_subsequence", "lcs_length_batch",
    "lcs_length_batch_device", "check_capacity", "generate_random", "device_count", "lib",
    "LIB_PATH", "pack_pairs",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WLCS_LIB_PATH") or os.path.join(HERE, "_lib", "libwavelcs_b200.so")

DEFAULT_MEMORY_BUDGET = 2 * 1024 ** 3  # kDefaultMemoryBudget, include/wavelcs/tables.hpp:12
NO_BUDGET = 2 ** 64 - 1
VARIANT_BITPARALLEL = 0
VARIANT_WAVEFRONT = 1


class CapacityError(RuntimeError):
    """include/wavelcs/errors.hpp:8-11."""


class ConfigError(RuntimeError):
    """include/wavelcs/errors.hpp:14-17."""


class InputError(RuntimeError):
    """include/wavelcs/errors.hpp:20-23."""


class EquivalenceError(AssertionError):
    """include/wavelcs/errors.hpp:27-30 (serial/parallel disagreement)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the library."""


class NoDeviceError(CudaError):
    """No usable CUDA device -- the library has no CPU fallback."""


_STATUS = {
    1: CapacityError,
    2: ConfigError,
    3: IndexError,          # std::out_of_range
    4: ValueError,          # std::invalid_argument
    5: InputError,
    6: CudaError,
    7: NoDeviceError,
    8: MemoryError,
    9: RuntimeError,
}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
        "g.build()'` (or `make lib`). There is no CPU fallback.")

lib = ctypes.CDLL(LIB_PATH)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_sz = ctypes.c_size_t
_vp = ctypes.c_void_p

lib.wlcs_abi_version.restype = ctypes.c_int
lib.wlcs_last_error.restype = ctypes.c_char_p
lib.wlcs_device_count.restype = ctypes.c_int
lib.wlcs_check_capacity.argtypes = [_sz, _sz, _sz]
lib.wlcs_length_ex.argtypes = [_vp, _sz, _vp, _sz, _sz, ctypes.c_int, _u32p]
lib.wlcs_subsequence.argtypes = [_vp, _sz, _vp, _sz, _sz, _vp, _sz, ctypes.POINTER(_sz)]
lib.wlcs_subsequence_ex.argtypes = [_vp, _sz, _vp, _sz, _sz, _sz, _vp, _sz, ctypes.POINTER(_sz)]
lib.wlcs_length_batch_ex.argtypes = [_vp, _u64p, _vp, _u64p, _sz, ctypes.c_int, _u32p]
lib.wlcs_length_batch_device.argtypes = [_vp, _vp, _vp, _vp, _sz, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, _vp, _vp]
lib.wlcs_length_device.argtypes = [_vp, _sz, _vp, _sz, ctypes.c_int, _u32p, _vp]
lib.wlcs_host_alloc.restype = _vp
lib.wlcs_host_alloc.argtypes = [_sz]
lib.wlcs_host_free.argtypes = [_vp]
lib.wlcs_generate_random.argtypes = [_sz, _vp, _sz, ctypes.c_uint64, _vp]
lib.wlcs_generate_pairs.argtypes = [_sz, _sz, _sz, _vp, _sz, ctypes.c_uint64, _vp, _u64p, _vp,
                                    _u64p]
lib.wlcs_set_timing.argtypes = [ctypes.c_int]
lib.wlcs_last_kernel_ms.argtypes = [ctypes.POINTER(ctypes.c_float)]
lib.wlcs_probe_int_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
lib.wlcs_colsplit_inbox_words.argtypes = [_sz, ctypes.POINTER(ctypes.c_size_t)]
lib.wlcs_colsplit_fill.argtypes = [_vp, _sz, _vp, _sz, _sz, _sz, ctypes.c_int, _vp, _vp, _vp, _vp,
                                   _vp, _vp]
lib.wlcs_device_alloc.argtypes = [_sz, ctypes.POINTER(ctypes.c_void_p)]
lib.wlcs_device_zero.argtypes = [_vp, _sz]
lib.wlcs_device_free.argtypes = [_vp]
lib.wlcs_ipc_handle.argtypes = [_vp, ctypes.c_char_p]
lib.wlcs_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
lib.wlcs_ipc_close.argtypes = [_vp]
lib.wlcs_fill_tables.argtypes = [_vp, _sz, _vp, _sz, _sz, _vp, _vp]
lib.wlcs_colsplit_emulate.argtypes = [_vp, _sz, _vp, _sz, ctypes.c_int, ctypes.c_int, _u32p]
lib.wlcs_length_rowbands.argtypes = [_vp, _sz, _vp, _sz, ctypes.c_int, _u32p]
lib.wlcs_length_batch_multi.argtypes = [_vp, _u64p, _vp, _u64p, _sz, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_uint32)]
lib.wlcs_length_strips.argtypes = [_vp, _sz, _vp, _sz, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_uint32)]


def _check(rc: int) -> None:
    if rc:
        msg = lib.wlcs_last_error().decode("utf-8", "replace")
        raise _STATUS.get(rc, RuntimeError)(msg)


def _as_bytes(s) -> bytes:
    if isinstance(s, str):
        return s.encode("latin-1")
    if isinstance(s, np.ndarray):
        return s.astype(np.uint8, copy=False).tobytes()
    return bytes(s)


def device_count() -> int:
    return int(lib.wlcs_device_count())


def check_capacity(m: int, n: int, memory_budget: int = DEFAULT_MEMORY_BUDGET) -> None:
    """check_capacity (include/wavelcs/tables.hpp:16); raises CapacityError."""
    _check(lib.wlcs_check_capacity(m, n, memory_budget))


def lcs_length(x, y, memory_budget: int = DEFAULT_MEMORY_BUDGET,
               variant: int = VARIANT_BITPARALLEL) -> int:
    """Length lcs_length(x, y, memory_budget)  (include/wavelcs/serial.hpp:24-25)."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    out = ctypes.c_uint32()
    _check(lib.wlcs_length_ex(xb, len(xb), yb, len(yb), memory_budget, variant,
                              ctypes.byref(out)))
    return int(out.value)


def lcs_subsequence(x, y, memory_budget: int = DEFAULT_MEMORY_BUDGET, row_cap: int = 0) -> bytes:
    """traceback(lcs_fill_parallel(x, y).back, x, M, N) as one call (serial.hpp:30).
    row_cap bounds the traceback's device memory (0 = automatic); beyond it
    the traceback runs in row bands recomputed from checkpoints."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    cap = max(1, min(len(xb), len(yb)))
    out = ctypes.create_string_buffer(cap)
    n = _sz()
    _check(lib.wlcs_subsequence_ex(xb, len(xb), yb, len(yb), memory_budget, row_cap, out, cap,
                                   ctypes.byref(n)))
    return out.raw[: n.value]


def pack_pairs(xs: _Seq, ys: _Seq):
    """Pack two lists of strings into (bytes, offsets) arrays for the batch API."""
    def pack(seq):
        bs = [_as_bytes(s) for s in seq]
        off = np.zeros(len(bs) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
        buf = np.frombuffer(b"".join(bs), dtype=np.uint8) if bs else np.zeros(0, np.uint8)
        return np.ascontiguousarray(buf), off
    xbuf, xoff = pack(xs)
    ybuf, yoff = pack(ys)
    return xbuf, xoff, ybuf, yoff


def _as_u8(a) -> np.ndarray:
    if isinstance(a, (bytes, bytearray, memoryview)):
        return np.frombuffer(a, dtype=np.uint8)
    return np.ascontiguousarray(a, dtype=np.uint8)


def lcs_length_batch(xs, x_off, ys, y_off, variant: int = VARIANT_BITPARALLEL) -> np.ndarray:
    """Lengths of many independent pairs (host arrays or bytes)."""
    xs = _as_u8(xs)
    ys = _as_u8(ys)
    x_off = np.ascontiguousarray(x_off, dtype=np.uint64)
    y_off = np.ascontiguousarray(y_off, dtype=np.uint64)
    pairs = len(x_off) - 1
    if len(y_off) != pairs + 1:
        raise ValueError("x_off and y_off must have the same length")
    out = np.zeros(max(pairs, 0), dtype=np.uint32)
    if pairs <= 0:
        return out
    _check(lib.wlcs_length_batch_ex(xs.ctypes.data, x_off.ctypes.data_as(_u64p), ys.ctypes.data,
                                    y_off.ctypes.data_as(_u64p), pairs, variant,
                                    out.ctypes.data_as(_u32p)))
    return out


def lcs_length_batch_device(d_xs: int, d_xoff: int, d_ys: int, d_yoff: int, pairs: int,
                            xs_bytes: int, ys_bytes: int, d_out: int, stream: int = 0,
                            variant: int = VARIANT_BITPARALLEL) -> None:
    """Batch on device pointers (e.g. torch tensors' data_ptr())."""
    _check(lib.wlcs_length_batch_device(d_xs, d_xoff, d_ys, d_yoff, pairs, xs_bytes, ys_bytes,
                                        variant, d_out, stream or None))


def generate_random(length: int, alphabet, seed: int) -> bytes:
    """generate_random (include/wavelcs/io.hpp:34): std::mt19937_64, alphabet[r % |A|]."""
    a = _as_bytes(alphabet)
    out = ctypes.create_string_buffer(max(1, length))
    _check(lib.wlcs_generate_random(length, a, len(a), seed & (2 ** 64 - 1), out))
    return out.raw[:length]


# ---- multi-GPU column split (include/wavelcs_capi.h, wlcs_colsplit_*) ----
COLSPLIT_FORWARD = 1
COLSPLIT_REVERSE = 2


def colsplit_inbox_words(m: int) -> int:
    w = ctypes.c_size_t()
    _check(lib.wlcs_colsplit_inbox_words(m, ctypes.byref(w)))
    return int(w.value)


def device_alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    _check(lib.wlcs_device_alloc(nbytes, ctypes.byref(p)))
    return int(p.value)


def device_zero(ptr: int, nbytes: int) -> None:
    _check(lib.wlcs_device_zero(ptr, nbytes))


def device_free(ptr: int) -> None:
    _check(lib.wlcs_device_free(ptr))


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib.wlcs_ipc_handle(ptr, buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check(lib.wlcs_ipc_open(handle, ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    _check(lib.wlcs_ipc_close(ptr))


def colsplit_fill(x, y, col_lo: int, col_hi: int, problems: int = 3, in_fwd: int = 0,
                  out_fwd: int = 0, in_rev: int = 0, out_rev: int = 0):
    """This rank's slice of the bidirectional fill; returns (v_fwd, v_rev) as
    uint32 arrays (None for a problem not run)."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    words = (col_hi - col_lo + 31) // 32
    vf = np.zeros(words, np.uint32) if problems & COLSPLIT_FORWARD else None
    vr = np.zeros(words, np.uint32) if problems & COLSPLIT_REVERSE else None
    _check(lib.wlcs_colsplit_fill(xb, len(xb), yb, len(yb), col_lo, col_hi, problems,
                                  in_fwd or None, out_fwd or None, in_rev or None,
                                  out_rev or None,
                                  vf.ctypes.data if vf is not None else None,
                                  vr.ctypes.data if vr is not None else None))
    return vf, vr


def lcs_length_batch_multi(xs, x_off, ys, y_off, n_gpus: int) -> np.ndarray:
    """Batch sharded over devices 0..n_gpus-1 of this process."""
    xs = _as_u8(xs)
    ys = _as_u8(ys)
    x_off = np.ascontiguousarray(x_off, np.uint64)
    y_off = np.ascontiguousarray(y_off, np.uint64)
    pairs = len(x_off) - 1
    out = np.zeros(max(pairs, 0), np.uint32)
    _check(lib.wlcs_length_batch_multi(xs.ctypes.data, x_off.ctypes.data_as(_u64p), ys.ctypes.data,
                                       y_off.ctypes.data_as(_u64p), pairs, n_gpus,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return out


def lcs_length_strips(x, y, n_gpus: int) -> int:
    """One pair, column split over devices 0..n_gpus-1 of this process."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    out = ctypes.c_uint32()
    _check(lib.wlcs_length_strips(xb, len(xb), yb, len(yb), n_gpus, ctypes.byref(out)))
    return int(out.value)


def colsplit_emulate(x, y, slices: int, max_ctas: int = 0) -> int:
    """The multi-GPU column split of (x rows, y columns) with `slices` ranks
    played as CTA pools of ONE launch on the current device (the inboxes are
    filled and polled while both sides run).  max_ctas caps the grid."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    out = ctypes.c_uint32()
    _check(lib.wlcs_colsplit_emulate(xb, len(xb), yb, len(yb), slices, max_ctas,
                                     ctypes.byref(out)))
    return int(out.value)


def lcs_length_rowbands(x, y, bands: int) -> int:
    """LCS length with the rows of x cut into `bands` bands that are combed
    independently (semi-local LCS) and composed exactly (prototype of the
    row split; csrc/seaweed.cu)."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    out = ctypes.c_uint32()
    _check(lib.wlcs_length_rowbands(xb, len(xb), yb, len(yb), bands, ctypes.byref(out)))
    return int(out.value)


def fill_tables(x, y, memory_budget: int = DEFAULT_MEMORY_BUDGET):
    """The reference's FillResult (lcs_fill_serial, include/wavelcs/serial.hpp:
    21-22) filled on the device: (dp uint32 (m+1, n+1), back uint8 (m, n))."""
    xb, yb = _as_bytes(x), _as_bytes(y)
    m, n = len(xb), len(yb)
    dp = np.zeros((m + 1, n + 1), np.uint32)
    back = np.zeros((m, n), np.uint8)
    _check(lib.wlcs_fill_tables(xb, m, yb, n, memory_budget, dp.ctypes.data,
                                back.ctypes.data if back.size else None))
    return dp, back
