// wlcs_device.h -- internal interface between the host C-ABI (capi.cu) and
// the kernel translation units.  Not installed; not part of the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace wlcs {

// Batch of packed pairs, all pointers DEVICE pointers.
struct BatchDev {
    const uint8_t* xs;
    const uint64_t* xoff;  // pairs + 1 offsets into xs
    uint64_t xs_bytes;     // extent of xs (chunk loads never read past it)
    const uint8_t* ys;
    const uint64_t* yoff;
    uint64_t ys_bytes;
    uint32_t* out;         // pairs lengths
    uint32_t pairs;        // entries to process (of ids when set)
    const uint32_t* ids;   // optional: entry i is pair ids[i] (nullptr: pair i)
    int pm_bytes;          // shared-memory bytes for match masks per warp
    int kmax;              // largest words-per-lane K of a lane shape (<= 12)
    int long_to_host;      // 1: pairs wider than 32 * kmax words are skipped (the host
                           // runs them through the strip kernel); 0: second pass
    // filled by batch_launch from the workspace
    uint32_t* vals;
    uint32_t* meta;
    uint32_t* overflow;
    const uint4* safe16;   // 16 zero bytes in device memory
};

size_t batch_workspace_bytes(uint32_t pairs, int pm_bytes);
int batch_smem_per_cta(int pm_bytes);
cudaError_t batch_launch(BatchDev d, void* workspace, int sms, cudaStream_t stream,
                         cudaEvent_t ev_main0 = nullptr, cudaEvent_t ev_main1 = nullptr);
cudaError_t int_peak_probe(int reps, double* ops_per_s, uint32_t* scratch);
uint32_t* batch_overflow_count_ptr(void* workspace, uint32_t pairs);
uint32_t* batch_overflow_list_ptr(void* workspace, uint32_t pairs);

// Second pass (bitpar_wide.cu): the first pass's overflow list, finished on
// the device at one word per lane with the 257-code mask table; pairs wider
// than 32 words sweep 1024-column blocks with carries through `carry`.
struct WideDev {
    const uint8_t* xs;
    const uint64_t* xoff;
    uint64_t xs_bytes;
    const uint8_t* ys;
    const uint64_t* yoff;
    uint64_t ys_bytes;
    uint32_t* out;
    const uint32_t* list;   // pair ids (the first pass's overflow list)
    const uint32_t* count;  // device count of list entries (<= cap)
    uint32_t cap;
    uint32_t pairs_total;   // pairs of the whole batch (carry-slot layout)
    uint16_t* carry[2];     // wide_scratch_words() words each (ping-pong)
    // filled by wide_launch from the workspace
    const uint4* safe16;    // 16 zero bytes in device memory
    uint32_t* meta;
    uint32_t* vals;
    uint32_t* bucket;
    uint32_t* rank;
};
size_t wide_workspace_bytes(uint32_t cap);
size_t wide_scratch_words(uint64_t xs_bytes, uint64_t ys_bytes, uint32_t pairs);
cudaError_t wide_launch(WideDev d, void* workspace, int sms, cudaStream_t stream);

}  // namespace wlcs

namespace wlcs {

// One bit-parallel fill problem of the strip kernel (DEVICE pointers): all
// rows of `coded` against the column string whose match masks are `pmg`.
struct FillProblem {
    const uint4* coded;     // pre-coded rows (pair_code_rows): plane 0, chunk 0
    int64_t plane;          // uint4 stride between the 4 coded planes
    int64_t cstride;        // uint4 stride between chunks
    int64_t rows;
    const uint32_t* pmg;    // global match masks [sigma][W]
    int64_t W;              // words per row = ceil(cols / 32)
    int64_t cols;
    int nstrips;            // ceil(W / (32 K))
    int nchunks;            // 16-row chunks of the row string
    uint32_t* carry;        // [nstrips][cwords] carry words, zero-initialised
    int64_t cwords;         // carry-row stride: round_up(nchunks, 4) + 16
    uint32_t* v_out;        // optional: final V words [>= W]
    unsigned long long* zeros;  // optional: LCS accumulator
    uint32_t* rows_out;     // optional: bit rows, diagonal layout (traceback)
    int64_t Mpad;           // nchunks * 16
    int64_t Dpad;           // diagonals per strip in rows_out = Mpad + 512
    // column split across GPUs: carries of the slice's first strip come from
    // ext_in (written by the neighbour GPU), the last strip's go to ext_out
    // (the neighbour's inbox, a peer pointer); both [cwords] words, zeroed
    const uint32_t* ext_in;
    uint32_t* ext_out;
    // banded (bounded-memory) traceback:
    const uint32_t* v_in;   // optional: V words before the first row (a checkpoint); null = ones
    uint32_t* ckpt_out;     // optional: V after every ckpt_chunks * 16 rows, [c - 1][W] for c >= 1
    int ckpt_chunks;
    int64_t walk_row0;      // global DP row of this problem's row 0 (walk's diagonal guess)
    int64_t walk_mtot;      // rows of the whole pair (walk's diagonal guess)
    int32_t* walk_entry;    // optional (device): entry column at the problem's last row, in:
                            // the walk's exit column at its first row, out; null = N
    unsigned long long* walk_place;  // optional (device): {LCS length, bytes already emitted
                                     // by lower bands}; the walk writes its bytes before them
};

// One strip-kernel launch: up to kMaxProblems problems sharing the column
// alphabet (1 = plain fill, 2 = bidirectional split, 2G = the column split of
// G slices played inside one launch).  CTA b serves problem b % nprob only and
// takes that problem's strips from ticket[b % nprob] in increasing order, so
// every problem has its own pool of warps: a strip waits only on an earlier
// strip of its own pool (already running) or on the neighbouring slice's last
// strip, whose pool is never starved by this one (liveness with more strips
// than resident warps).
constexpr int kMaxProblems = 8;
struct PairDev {
    FillProblem prob[kMaxProblems];
    int nprob;
    uint32_t code_stride;   // smem bytes per code record (set by pair_fill)
    uint32_t pm_warp_bytes; // smem bytes of the match masks (set by pair_fill)
    int max_ctas;           // optional grid cap (0 = resident warps); tests force pools < strips
    const uint8_t* colp0;   // column string of problem 0 (alphabet scan)
    const uint16_t* map;    // 256 byte -> code map of the column alphabet
    int sigma;              // codes incl. the zero row
    uint32_t* ticket;       // per-problem strip ticket counters [kMaxProblems], zeroed
    uint32_t* error;        // zeroed; set when a carry poll times out (watchdog)
    uint32_t* sink;         // scratch the strip kernel's non-publishing lanes store to
                            // (>= kPairSinkWords words)
    const uint4* safe16;    // 16 zero bytes in device memory
};

constexpr int kPairSinkWords = 1 << 20;  // >= grid * block threads of the strip kernel

cudaError_t pair_prepare(PairDev& d, uint32_t* present256, uint16_t* map256, uint32_t* sigma_dev,
                         cudaStream_t stream, int* sigma_host);
cudaError_t pair_build_pm(const uint8_t* colp, int64_t cols, const uint16_t* map, int sigma,
                          int64_t W, uint32_t* pmg, cudaStream_t stream);
int64_t pair_code_plane(int nchunks);  // uint4 entries per coded plane (with padding)
cudaError_t pair_code_rows(const uint8_t* row, int64_t rows, bool reverse, const uint16_t* map,
                           int K, FillProblem& P, uint4* coded_base, cudaStream_t stream);
cudaError_t pair_reverse(const uint8_t* src, int64_t n, uint8_t* dst, cudaStream_t stream);
cudaError_t pair_split_combine(const uint32_t* vf, const uint32_t* vr, int64_t W, int64_t N,
                               uint32_t* scratch, unsigned long long* best, cudaStream_t stream);
int pair_smem_bytes(int K, int sigma);

cudaError_t pair_fill(const PairDev& d, int K, bool store, int sms, cudaStream_t stream);
// The reference's DpTable / BacktrackTable from the stored bit rows.
cudaError_t pair_tables(const PairDev& d, int K, uint32_t* dp, uint8_t* back,
                        cudaStream_t stream);
size_t pair_walk_scratch_bytes(int64_t rows);
// Exact traceback; out receives the subsequence in FORWARD order.
cudaError_t pair_walk(const PairDev& d, int K, const uint8_t* x, uint8_t* out,
                      unsigned long long* out_len, void* scratch, uint32_t* misses,
                      cudaStream_t stream);

}  // namespace wlcs

namespace wlcs {

// ---- cell-wavefront variant (wavefront.cu) ----
constexpr int kWaveMaxCols = 2048;  // batch kernel: shorter string per pair

struct WaveBatchDev {
    const uint8_t* xs;
    const uint64_t* xoff;
    const uint8_t* ys;
    const uint64_t* yoff;
    uint32_t* out;
    uint32_t pairs;
    uint32_t* counter;         // pair ticket (zeroed)
    uint32_t* overflow_count;  // pairs whose shorter string exceeds kWaveMaxCols
    uint32_t* overflow;        // their indices
};

struct WavePairDev {
    const uint8_t* rowp;  // rows (m bytes)
    int64_t m;
    const uint8_t* colp;  // columns (n bytes)
    int64_t n;
    uint32_t* bnd;        // [nbuf][bstride] ring of boundary rows (value << 8 | tag), zeroed
    int64_t bstride;      // >= n + 64
    uint32_t nbuf;        // >= 2
    uint32_t* ticket;     // band ticket (zeroed)
    uint32_t* out;        // LCS length
    uint32_t* error;      // watchdog flag (zeroed): a hand-off word never arrived
    int R;                // rows per virtual lane (wave_pair_rows): bands of 64 R rows
};

// ---- row-band decomposition through seaweed combing (seaweed.cu) ----
struct SeaDev {
    const uint8_t* rowp;    // rows (m bytes)
    const int64_t* row_lo;  // [bands + 1] band row bounds (device)
    const uint8_t* colp;    // columns (n bytes)
    int64_t n;
    uint32_t* v;            // [bands][n] column seaweeds (scratch)
    uint32_t* e;            // [bands][n] exit column of each top seaweed (n = right side)
};
// Combs every band (one launch, bands concurrent), then composes the bands
// top to bottom through their DP boundaries; *out (device) = the length.
// t0, t1: n + 1 words each.
cudaError_t seaweed_bands(const SeaDev& d, int bands, uint32_t* t0, uint32_t* t1,
                          uint32_t* out, cudaStream_t stream);

// ---- the reference's block-kernel contract on the device (tiles.cu) ----
// Tile of h x w cells from its north row (w + 1 values, corner first) and
// west column (h values); cv / bv receive the tile's cells and arrows.
cudaError_t tile_fill(const uint8_t* d_x, const uint8_t* d_y, const uint32_t* d_north,
                      const uint32_t* d_west, uint32_t* d_cv, uint8_t* d_bv, int h, int w,
                      cudaStream_t stream);

size_t wave_batch_smem();
cudaError_t wave_batch_launch(const WaveBatchDev& d, int sms, cudaStream_t stream);
int wave_pair_rows(int64_t m, int sms);
int64_t wave_pair_bands(int64_t m, int R);
cudaError_t wave_pair_launch(const WavePairDev& d, int sms, cudaStream_t stream);

}  // namespace wlcs
