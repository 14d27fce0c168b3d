/*
 * wavelcs_capi.h -- C-ABI of the B200-native LCS table-fill library
 * (libwavelcs_b200.so).  Plain pointers and sizes only; no CUDA, C++ or
 * torch types cross this boundary.
 *
 * Drop-in boundary for the reference "wavelcs" (paths relative to
 * /root/reference/proj).  Each entry point names the reference interface it
 * replaces; INTEGRATION.md shows the binding a maintainer adds on the
 * reference side (a ctypes stub and the C++ facade in include/wavelcs_b200.hpp).
 *
 * Conventions
 *   - x is the "parent" string (DP rows, index i), y the "child" string (DP
 *     columns, index j), exactly as in lcs_fill_parallel(x, y, cfg)
 *     (include/wavelcs/parallel.hpp:92-93).  Strings are raw bytes; every
 *     byte value 0..255 is a symbol (include/wavelcs/sequence.hpp:10-12).
 *   - Host-pointer entry points are synchronous: results are valid on return.
 *   - Every call returns a wlcs_status; on failure wlcs_last_error() gives a
 *     thread-local message.  The C++ facade maps statuses back onto the
 *     reference's exception types (include/wavelcs/errors.hpp:8-30).
 *   - The library is re-entrant: each host thread gets its own CUDA stream
 *     and workspace per device; there is no global mutable state on the fast
 *     path.  The current CUDA device of the calling thread is used.
 *   - The CUDA kernels are mandatory: there is no CPU fallback.  Without a
 *     usable GPU every compute entry point returns WLCS_E_NO_DEVICE.
 */
#ifndef WAVELCS_CAPI_H
#define WAVELCS_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WLCS_ABI_VERSION 1

typedef enum wlcs_status {
    WLCS_OK = 0,
    WLCS_E_CAPACITY = 1,         /* wavelcs::CapacityError   (src/tables.cpp:16-23)  */
    WLCS_E_CONFIG = 2,           /* wavelcs::ConfigError     (src/parallel.cpp:52-54) */
    WLCS_E_OUT_OF_RANGE = 3,     /* std::out_of_range        (src/serial.cpp:37-41)   */
    WLCS_E_INVALID_ARGUMENT = 4, /* std::invalid_argument                              */
    WLCS_E_INPUT = 5,            /* wavelcs::InputError                                */
    WLCS_E_CUDA = 6,             /* CUDA runtime error                                 */
    WLCS_E_NO_DEVICE = 7,        /* no usable CUDA device: no CPU fallback exists      */
    WLCS_E_OUT_OF_MEMORY = 8,    /* device allocation failed                           */
    WLCS_E_INTERNAL = 9
} wlcs_status;

/* Budget sentinel: skip the reference's table-capacity check. */
#define WLCS_NO_BUDGET ((size_t)-1)
/* kDefaultMemoryBudget (include/wavelcs/tables.hpp:12): 2 GiB. */
#define WLCS_DEFAULT_BUDGET ((size_t)2 * 1024 * 1024 * 1024)

/* Fill-kernel variants (both give bit-identical lengths). */
#define WLCS_VARIANT_BITPARALLEL 0 /* Hyyro bit-vector, 32 cells per 3 int ops */
#define WLCS_VARIANT_WAVEFRONT 1   /* tiled anti-diagonal cell wavefront (DPX) */

int wlcs_abi_version(void);
const char* wlcs_last_error(void);
/* Number of visible CUDA devices (0 when none). */
int wlcs_device_count(void);

/* check_capacity(m, n, budget)  -- include/wavelcs/tables.hpp:16,
 * src/tables.cpp:9-24: 4(M+1)(N+1) + MN bytes, computed in 128 bits.
 * Returns WLCS_E_CAPACITY with the reference's message when exceeded. */
int wlcs_check_capacity(size_t m, size_t n, size_t memory_budget);

/* Length  -- replaces Length lcs_length(const Sequence& x, const Sequence& y,
 * std::size_t memory_budget)  (include/wavelcs/serial.hpp:24-25,
 * src/serial.cpp:32-34).  memory_budget keeps the reference's semantics
 * (CapacityError when the reference's tables would not fit); pass
 * WLCS_NO_BUDGET to lift it.  The device path itself is O(M + N) memory. */
int wlcs_length(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t memory_budget,
                uint32_t* out);

/* Same, choosing the fill kernel variant (WLCS_VARIANT_*). */
int wlcs_length_ex(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t memory_budget,
                   int variant, uint32_t* out);

/* Recovered subsequence  -- replaces the composition the reference's callers
 * use: lcs_fill_parallel(x, y, cfg) then traceback(fill.back, x, M, N)
 * (tools/wavelcs_main.cpp:78-86; include/wavelcs/serial.hpp:30,
 * include/wavelcs/parallel.hpp:92-93).  The result is byte-identical to the
 * reference's traceback, LEFT tie-break included (include/wavelcs/cell.hpp:27-38).
 * out must hold at least min(m, n) bytes (cap); *out_len receives the length.
 * Capacity check as in wlcs_length. */
int wlcs_subsequence(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                     size_t memory_budget, uint8_t* out, size_t cap, size_t* out_len);

/* Same, with a cap on the traceback's device memory (stored bit rows plus
 * checkpoints), row_cap bytes; 0 = automatic (half the free device memory, at
 * most 8 GiB).  Within the cap the fill stores every row (M * N / 8 bytes);
 * beyond it the traceback runs in row bands: a first fill keeps the bit
 * vector of every B-th row, then each band is filled again from its
 * checkpoint and walked, bottom band first -- the same rows and rule, hence
 * the same string, in O(N (M / B + B)) bits.  WLCS_E_OUT_OF_MEMORY when even
 * one 256-row band does not fit row_cap. */
int wlcs_subsequence_ex(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                        size_t memory_budget, size_t row_cap, uint8_t* out, size_t cap,
                        size_t* out_len);

/* Batch of independent pairs (new; the reference loops one pair at a time,
 * src/bench.cpp:77-129).  Pair k is x = xs[x_off[k] .. x_off[k+1]) and
 * y = ys[y_off[k] .. y_off[k+1]); offsets are absolute, non-decreasing,
 * pairs + 1 entries each.  out[k] = lcs_length(x_k, y_k).  Host pointers;
 * page-locked host buffers give full-speed DMA (see wlcs_host_alloc). */
int wlcs_length_batch(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                      const uint64_t* y_off, size_t pairs, uint32_t* out);

/* Same with the kernel variant. */
int wlcs_length_batch_ex(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                         const uint64_t* y_off, size_t pairs, int variant, uint32_t* out);

/* Batch on DEVICE pointers already resident in HBM (current device),
 * ASYNCHRONOUS: the whole batch is enqueued on `stream` (a cudaStream_t; NULL
 * = the legacy default stream, e.g. torch's default stream) and the call
 * returns without waiting -- d_out is valid once the stream's work up to this
 * point has completed.  No host round trip: pairs the first pass cannot hold
 * (alphabet over its mask budget, or wider than its lane shapes) are finished
 * by a second pass whose length is read on the device.  d_xs and d_ys must be
 * 16-byte aligned (cudaMalloc / torch allocations are); each pair's strings
 * must lie inside [d_xs, d_xs + xs_bytes) / [d_ys, d_ys + ys_bytes). */
int wlcs_length_batch_device(const uint8_t* d_xs, const uint64_t* d_x_off, const uint8_t* d_ys,
                             const uint64_t* d_y_off, size_t pairs, uint64_t xs_bytes,
                             uint64_t ys_bytes, int variant, uint32_t* d_out, void* stream);

/* Single pair on DEVICE pointers (length only; budget not applied; 16-byte
 * aligned buffers).  The fill is ordered after the work enqueued on `stream`
 * (NULL = the legacy default stream) before the call; synchronous: *out is
 * valid on return. */
int wlcs_length_device(const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n, int variant,
                       uint32_t* out, void* stream);

/* Instrumentation for bench.py: when on, the batch entry points bracket their
 * main kernel with CUDA events on the launching stream; wlcs_last_kernel_ms
 * returns that kernel's duration (ms) for the calling thread's last batch. */
int wlcs_set_timing(int on);
int wlcs_last_kernel_ms(float* ms);

/* Integer ALU-pipe peak of the current device (int32 ops/s, best of reps),
 * measured by a LOP3 stream kernel: the roofline denominator of the fill. */
int wlcs_probe_int_peak(int reps, double* ops_per_s);

/* Page-locked host memory for zero-copy-speed transfers (cudaHostAlloc). */
void* wlcs_host_alloc(size_t bytes);
void wlcs_host_free(void* p);

/* generate_random(length, alphabet, seed)  -- include/wavelcs/io.hpp:34,
 * src/io.cpp:103-115 (std::mt19937_64, alphabet[rng() % |alphabet|]).
 * Synthetic-input helper for benchmarks and tests; host-only. */
int wlcs_generate_random(size_t length, const uint8_t* alphabet, size_t alphabet_len,
                         uint64_t seed, uint8_t* out);

/* Synthetic batch for benchmarks/tests (BASELINE config C2 procedure):
 * master = std::mt19937_64(seed); per pair k: m = lo + master() % (hi-lo+1),
 * n likewise, then seed_x = master(), seed_y = master() and
 * x_k = generate_random(m, alphabet, seed_x), y_k = generate_random(n, ...).
 * xs / ys must hold pairs*hi bytes; offsets pairs+1 entries. */
int wlcs_generate_pairs(size_t pairs, size_t lo, size_t hi, const uint8_t* alphabet,
                        size_t alphabet_len, uint64_t seed, uint8_t* xs, uint64_t* x_off,
                        uint8_t* ys, uint64_t* y_off);

/* ---- multi-GPU column split of one long pair ----
 *
 * The bidirectional bit-parallel fill of (x, y) is cut into column slices,
 * one per GPU / rank; rank g owns columns [col_lo, col_hi) of y.  Two
 * problems share the slice: FORWARD = rows x[0, m/2) against y[col_lo,
 * col_hi); REVERSE = rows x[m/2, m) reversed against the slice reversed.
 * Between neighbouring slices only one carry word per 16 rows travels (the
 * strip kernel's hand-off): forward carries flow from rank g-1 to rank g,
 * reverse carries from rank g+1 to rank g.  The producer's kernel writes them
 * straight into the consumer's INBOX (device memory of the consumer GPU,
 * reached through a peer / IPC pointer) as self-validating words; the
 * consumer's kernel polls its inbox -- the exchange is fused into the fill.
 *
 * Inboxes: wlcs_colsplit_inbox_words(m) 32-bit words per problem, allocated
 * with wlcs_device_alloc (zeroed) and shared across processes with
 * wlcs_ipc_handle / wlcs_ipc_open.  An inbox must be re-zeroed
 * (wlcs_device_zero) before every fill that uses it.
 *
 * wlcs_colsplit_fill: problems = WLCS_COLSPLIT_FORWARD | WLCS_COLSPLIT_REVERSE
 * (both in one launch in production; separately when a single device plays
 * several ranks in order, see tests).  d_in_* = this rank's inboxes (NULL
 * for the first slice of that direction), d_out_* = the neighbour's inboxes
 * (NULL for the last slice).  On return v_fwd / v_rev (host arrays of
 * ceil((col_hi - col_lo) / 32) words, may be NULL for a problem not run)
 * hold the slice's final bit vectors; the LCS length is then
 *   max_k F[k] + R[k],  F[k] = zero bits of the forward vectors below column
 *   k, R[k] = zero bits of the reverse vectors below n - k
 * (paper_1306_4627_b200/multigpu.py: colsplit_combine). */
#define WLCS_COLSPLIT_FORWARD 1
#define WLCS_COLSPLIT_REVERSE 2
int wlcs_colsplit_inbox_words(size_t m, size_t* words);
int wlcs_colsplit_fill(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t col_lo,
                       size_t col_hi, int problems, const uint32_t* d_in_fwd,
                       uint32_t* d_out_fwd, const uint32_t* d_in_rev, uint32_t* d_out_rev,
                       uint32_t* v_fwd, uint32_t* v_rev);

/* The reference's full tables, filled on the device:
 * replaces lcs_fill_serial / lcs_fill_parallel's FillResult
 * (include/wavelcs/serial.hpp:21-22, parallel.hpp:92-93) for callers that
 * need the tables themselves.  dp: (m+1)*(n+1) uint32 cells, row-major,
 * layout of DpTable (tables.hpp:20-45); back: m*n arrows (Diag 0 / Up 1 /
 * Left 2), layout of BacktrackTable (tables.hpp:49-71).  Host buffers.
 * memory_budget is checked exactly as check_capacity (tables.cpp:9-24). */
int wlcs_fill_tables(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                     size_t memory_budget, uint32_t* dp, uint8_t* back);

/* The reference's block-kernel plugin contract (BlockArgs,
 * include/wavelcs/kernels.hpp:23-35 of the reference; compute_block,
 * parallel.hpp:78-79): fill cells [i_first, i_last] x [j_first, j_last]
 * (1-based, inclusive) of the caller's HOST tables -- c: DP cells
 * c[i * c_stride + j], b: arrows b[(i-1) * b_stride + (j-1)] -- from their
 * final row i_first - 1 and column j_first - 1, on the device, with
 * lcs_cell's values and arrows.  x[i-1] / y[j-1] are the i-th / j-th
 * symbols.  An empty range is a no-op. */
int wlcs_fill_block(const uint8_t* x, const uint8_t* y, uint32_t* c, size_t c_stride, uint8_t* b,
                    size_t b_stride, size_t i_first, size_t i_last, size_t j_first, size_t j_last);

/* Single-process multi-GPU conveniences, devices 0..n_gpus-1
 * of the calling process, one host thread per device:
 *  - wlcs_length_batch_multi: pairs sharded into contiguous ranges balanced by
 *    cells (no exchange during compute);
 *  - wlcs_length_strips: one pair, column split across the devices with the
 *    carries written straight into the neighbour's inbox over peer access
 *    (the same fused hand-off as wlcs_colsplit_fill), then the F+R combine.
 * n_gpus <= 1 runs the single-device path; n_gpus above the visible device
 * count is WLCS_E_CONFIG. */
int wlcs_length_batch_multi(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                            const uint64_t* y_off, size_t pairs, int n_gpus, uint32_t* out);
int wlcs_length_strips(const uint8_t* x, size_t m, const uint8_t* y, size_t n, int n_gpus,
                       uint32_t* out);

/* The column split of ONE device's pair played as `slices` ranks inside a
 * single strip-kernel launch (2 * slices problems, one CTA pool each; slice
 * g's first strips poll inboxes that slices g-1 / g+1 fill while running --
 * the same fused hand-off as wlcs_colsplit_fill between GPUs).  max_ctas > 0
 * caps the grid (tests: fewer warps per pool than strips per problem);
 * slices <= 4.  x = rows, y = the split column string.  *out = LCS length. */
int wlcs_colsplit_emulate(const uint8_t* x, size_t m, const uint8_t* y, size_t n, int slices,
                          int max_ctas, uint32_t* out);

/* Row-band decomposition of one pair (prototype): the
 * rows of x are cut into `bands` equal bands that are combed INDEPENDENTLY
 * (semi-local LCS, seaweed combing; one warp per band, all bands in one
 * launch) and composed top to bottom through their DP boundaries
 * (C[j] = max_{i<=j} T[i] + H(i, j), exact).  The route to splitting a long
 * pair's rows across GPUs; today a correctness prototype (cell-level combing,
 * O(n^2) combine), not the fast path.  Replaces no reference entry point: the
 * reference's only schedule is the row-serial wavefront
 * (proj/src/parallel.cpp:172-226).  *out = LCS length. */
int wlcs_length_rowbands(const uint8_t* x, size_t m, const uint8_t* y, size_t n, int bands,
                         uint32_t* out);

/* Device memory helpers for the inboxes (current device). */
int wlcs_device_alloc(size_t bytes, void** d_ptr); /* zero-filled */
int wlcs_device_zero(void* d_ptr, size_t bytes);
int wlcs_device_free(void* d_ptr);
/* cudaIpcMemHandle_t as 64 opaque bytes, for exchanging inboxes between
 * processes (one process per GPU); peer access is enabled on open. */
int wlcs_ipc_handle(void* d_ptr, uint8_t handle[64]);
int wlcs_ipc_open(const uint8_t handle[64], void** d_ptr);
int wlcs_ipc_close(void* d_ptr);

#ifdef __cplusplus
}
#endif

#endif /* WAVELCS_CAPI_H */
