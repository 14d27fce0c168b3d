// bitpar_pair.cu -- single-pair bit-parallel LCS fill (configs C1, C3, C4, C5)
// and the exact device traceback.
//
// Replaces, for ONE (possibly huge) pair, the reference's
//   lcs_fill_parallel   proj/src/parallel.cpp:251-274  (std::thread wavefront)
//   lcs_length          proj/src/serial.cpp:32-34
//   traceback           proj/src/serial.cpp:36-61
// without materialising DpTable / BacktrackTable (5*M*N bytes).
//
// Fill ("strip kernel"): the column string is cut into strips of 32*K words;
// one warp owns one strip and streams all rows, 16 rows per step.  Inside the
// warp the 32 lanes form a skewed carry pipeline (lane l works on chunk t-l,
// carries of 16 rows travel as one mask via __shfl_up_sync).  Between strips
// the carry masks of lane 31 go through global memory as self-validating
// words (see pair_strip_kernel).  Strips are handed out by an atomic ticket in
// increasing order, so a strip only ever waits on a strip that is already
// running (no co-residency assumption).
//
// Length of a long pair: bidirectional split (Hirschberg's lemma).  The top
// half of the rows runs forward and the bottom half runs on the reversed
// strings, as two problems of ONE launch (twice the strips in flight, half the
// sequential row chain); L = max_k F[k] + R[k] over the middle row.
//
// Traceback: with STORE the fill also writes every row's V words into
// rows_out (diagonal layout, see pair_row_index).  The walk applies the
// reference rule (serial.cpp:44-58 with cell.hpp:30-38) in bit form:
//   x_i == y_j                 -> Diag  (emit x_i)
//   bit j-1 of V_i is 0 (H=1)  -> Up     (then c[i-1][j] = c[i][j] > c[i][j-1])
//   otherwise                  -> Left
// so per row it only needs the highest set bit of (PM[x_i] | ~V_i) at or
// below column j: one row per iteration instead of one cell.
#include <cstdio>
#include <cstdlib>

#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {


__global__ void pair_alphabet_kernel(const uint8_t* colp, int64_t cols, uint32_t* present) {
    __shared__ uint32_t seen[256];
    seen[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += int64_t(gridDim.x) * blockDim.x)
        seen[colp[j]] = 1;
    __syncthreads();
    if (seen[threadIdx.x]) present[threadIdx.x] = 1;
}

// One warp: present[256] -> map[256] (codes 1..sigma-1, 0 = absent) and sigma.
// Codes are 16-bit: all 256 byte values plus the zero row need 257 codes.
__global__ void pair_codes_kernel(const uint32_t* present, uint16_t* map, uint32_t* sigma) {
    const uint32_t lane = threadIdx.x;
    uint32_t cnt = 0;
    for (int b = 0; b < 8; ++b) cnt += present[lane * 8 + b] ? 1u : 0u;
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
        if (int(lane) >= o) incl += v;
    }
    uint32_t code = incl - cnt + 1;
    for (int b = 0; b < 8; ++b) map[lane * 8 + b] = present[lane * 8 + b] ? uint16_t(code++) : 0;
    if (lane == 31) *sigma = incl + 1;
}

// Global match masks pmg[code][W]; one thread per word.
__global__ void pair_pm_kernel(const uint8_t* colp, int64_t cols, const uint16_t* map, int sigma,
                               int64_t W, uint32_t* pmg) {
    const int64_t w = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= W) return;
    for (int c = 0; c < sigma; ++c) pmg[int64_t(c) * W + w] = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t j = w * 32 + b;
        if (j >= cols) break;
        const int c = map[colp[j]];
        pmg[int64_t(c) * W + w] |= 1u << b;
    }
}

// Bit rows for the traceback, stored along the lane pipeline's diagonals so
// every store instruction of a warp is one contiguous 128*K-byte run: lane l
// of strip s holds word group g = 32 s + l, and at step t all lanes of the warp
// are on diagonal d = row + 16 l = 16 t + r.  Index of word k of group g at
// string row q:  ((s * Dpad + q + 16 l) * 32 + l) * K + k   (pair_row_index).
__host__ __device__ __forceinline__ int64_t pair_row_index(int64_t q, int64_t w, int K,
                                                           int64_t Dpad) {
    const int64_t g = w / K, s = g >> 5, l = g & 31;
    return ((s * Dpad + q + 16 * l) * 32 + l) * K + (w - g * K);
}

template <int K, bool STORE>
struct StoreHook {
    uint32_t* base;  // rows_out + ((s * Dpad) * 32 + l) * K
    int64_t dlo;     // diagonal of row 0 of the current step (16 t)
    __device__ __forceinline__ void operator()(int r, bool valid, const uint32_t* V) const {
        if constexpr (STORE) {
            if (valid) {
                uint32_t* p = base + (dlo + r) * (32 * K);
                if constexpr (K == 8) {
                    reinterpret_cast<uint4*>(p)[0] = make_uint4(V[0], V[1], V[2], V[3]);
                    reinterpret_cast<uint4*>(p)[1] = make_uint4(V[4], V[5], V[6], V[7]);
                } else if constexpr (K == 4) {
                    reinterpret_cast<uint4*>(p)[0] = make_uint4(V[0], V[1], V[2], V[3]);
                } else if constexpr (K == 2) {
                    reinterpret_cast<uint2*>(p)[0] = make_uint2(V[0], V[1]);
                } else {
                    p[0] = V[0];
                }
            }
        }
    }
};

// System-scope variant for the carry words that cross GPUs (column split:
// the producer writes into the consumer's memory over NVLink / P2P).
__device__ __forceinline__ uint4 ld_relaxed_sys_v4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
// gpu-scope relaxed vector load of four carry words (a strong load: the
// producer's relaxed stores and this poll do not race).  No "memory" clobber:
// the words validate themselves, so other accesses may move across the poll.
__device__ __forceinline__ uint4 ld_relaxed_gpu_v4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Stores without a "memory" clobber (self-validating words: the compiler may
// move other accesses across them).
__device__ __forceinline__ void st_relaxed_gpu_nb(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ void st_relaxed_sys_nb(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

constexpr uint32_t kCarryValid = 0x10000u;  // carry words: valid flag | 16-row mask
// re-polls of one carry group before a strip gives up (about 10-30 s of L2 /
// NVLink round trips: far beyond any legitimate wait, which is bounded by the
// producer's own fill time)
constexpr uint32_t kPollLimit = 1u << 24;

// Row coding: entry i = map[row byte i] (the row's match-mask record in the
// strip's shared-memory table is at code * code_stride).  Rows
// outside [0, rows) -- the lane pipeline's prologue/epilogue chunks -31 ..
// nchunks + 30 and the tail of the last chunk -- are 0 (code 0 = all-zero
// masks = identity row, also carry-neutral), so the strip kernel needs no
// row-validity masks.  Layout: 4 planes of uint4; plane j holds entries
// 4j..4j+3 of every chunk, chunk ch at index ch + kPadChunks, so the warp's
// j-th LDG.128 (lanes on chunks t-0 .. t-31) is one contiguous 512-byte run.
// With `reverse` the row string is coded back to front.
constexpr int kPadChunks = 56;  // >= 31 (lane skew) + 3 (group rounding) + kCodeAhead + kCodeL2Ahead
constexpr int kCodeAhead = 4;   // code prefetch distance in steps (registers)
constexpr int kCodeL2Ahead = 12;  // L2 prefetch distance in steps beyond the register ring

struct Codes {
    uint4 a, b, c, d;  // rows 0-3, 4-7, 8-11, 12-15 of a chunk
};

__global__ void pair_code_rows_kernel(const uint8_t* row, int64_t rows, int reverse,
                                      const uint16_t* map, int64_t plane, int64_t cstride,
                                      int64_t nchp, uint32_t* coded /* plane 0, padded chunk 0 */) {
    const int64_t total = nchp * 16;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t chp = e >> 4;
        const int r = int(e & 15);
        const int64_t i = (chp - kPadChunks) * 16 + r;
        uint32_t v = 0;
        if (i >= 0 && i < rows) v = uint32_t(map[row[reverse ? rows - 1 - i : i]]);
        coded[((r >> 2) * plane + chp * cstride) * 4 + (r & 3)] = v;
    }
}

// Strip kernel.  CTA b serves problem q = b % nprob and takes its strips
// from ticket[q] in increasing order, so inside each problem strips start in
// order and a strip only ever waits on a strip that is already running (or, in
// a column split, on the neighbouring slice's last strip, served by another
// pool).
//
// Per step a lane reads its 16-row chunk as 16 codes (4 coalesced LDG.128,
// prefetched kCodeAhead steps ahead) and runs 16 row updates: per row one
// IMAD for the mask address, one LDS, 3 ALU ops per word plus one ALU op and
// one IMAD.X for the carry bit in and out.
//
// Carry handoff between strips: lane 31 of strip s publishes the 16-row carry
// mask of chunk ch as one relaxed 32-bit store (kCarryValid | mask) into a
// zero-initialised buffer -- the data word is its own ready flag, so no fence
// is needed.  Strip s+1 reads the words four chunks at a time with one 16-byte
// relaxed load (gpu scope; sys scope for a neighbour GPU's inbox), the same
// address for the whole warp: a broadcast, so the hand-off code is
// warp-uniform.  The load of group g+1 is issued half way through group g;
// a group with a word still 0 is re-polled.  Inside the warp the carry masks
// move with two shuffles per step (rows 0-7 after row 7, rows 8-15 after row
// 15), so the shuffle latency hides behind row work.
//
// Launch: 1-warp CTAs (one strip each), up to the occupancy limit (more
// warps per CTA were measured: no gain, strips only share sub-partitions).
// MODE: 0 length, 1 store bit rows (traceback / tables / banded bands),
// 3 length keeping a checkpoint V every ckpt_chunks chunks (banded
// traceback, first pass)
template <int K, int MODE>
__global__ void __launch_bounds__(32, 1) pair_strip_kernel(PairDev d) {
    constexpr bool STORE = MODE == 1, CKPT = MODE == 3;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* pm = smem;
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    const uint32_t lane = lane_id();
    const uint32_t lane_off = PmLayout<K>::word_offset(lane, 0);
    uint32_t* sink = d.sink + (int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
    const int q = int(blockIdx.x % uint32_t(d.nprob));
    const FillProblem& P = d.prob[q];
    for (;;) {
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(d.ticket + q, 1u);
        tk = __shfl_sync(kFullMask, tk, 0);
        if (tk >= uint32_t(P.nstrips)) break;
        const uint32_t strip = tk;
        __syncwarp();
        const int64_t g = int64_t(strip) * 32 + lane;  // global lane-group index
        for (int c = 0; c < d.sigma; ++c) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int64_t w = g * K + k;
                const uint32_t v = w < P.W ? __ldg(P.pmg + int64_t(c) * P.W + w) : 0u;
                *reinterpret_cast<uint32_t*>(pm + c * cs + PmLayout<K>::word_offset(lane, k)) = v;
            }
        }
        __syncwarp();

        const int nchunks = P.nchunks;
        const int64_t plane = P.plane;
        uint32_t V[K];
#pragma unroll
        for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
        if constexpr (STORE) {  // a band of the banded traceback starts at a checkpoint
            if (P.v_in) {
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (g * K + k < P.W) V[k] = __ldg(P.v_in + g * K + k);
            }
        }
        // the slice's first strip takes its carries from ext_in and its last
        // strip sends them to ext_out when the pair is split across GPUs
        const bool ext_left = strip == 0 && P.ext_in != nullptr;
        const bool ext_right = strip + 1 == uint32_t(P.nstrips) && P.ext_out != nullptr;
        const bool has_left = strip > 0 || ext_left;
        const bool has_right = strip + 1 < uint32_t(P.nstrips) || ext_right;
        const int64_t cwords = P.cwords;  // carry-row stride (multiple of 4)
        const uint32_t* left_carry =
            ext_left ? P.ext_in : P.carry + int64_t(strip > 0 ? strip - 1 : 0) * cwords;
        uint32_t* my_carry = ext_right ? P.ext_out : P.carry + int64_t(strip) * cwords;
        // the whole warp loads the (same) carry words -- a broadcast, so the
        // hand-off code is warp-uniform (no divergence); lane 0 consumes them
        const bool feeder = has_left;
        auto carry_ld4 = [&](const uint32_t* p) {
            return ext_left ? ld_relaxed_sys_v4(p) : ld_relaxed_gpu_v4(p);
        };
        StoreHook<K, STORE> hook{
            STORE ? P.rows_out + ((int64_t(strip) * P.Dpad) * 32 + lane) * K : nullptr, 0};
        const int T = (nchunks + 31 + 3) & ~3;
        // lane l works on chunk t - l (chunks < 0 / >= nchunks are padding).
        // Register rings, no rotation moves (a move of a register with a load
        // in flight would stall on it): codes of step t live in ring slot
        // t % 4 and are reloaded, 4 steps ahead, right after their rows.
        // Lane 0's chunk is always new data (an L2 round trip), the other
        // lanes re-read what lane l-1 read a step earlier.
        const int64_t cstride = P.cstride;
        const uint4* cp = P.coded - int64_t(lane) * cstride;
        auto load_codes = [&](const uint4* q) {
            return Codes{__ldg(q), __ldg(q + plane), __ldg(q + 2 * plane), __ldg(q + 3 * plane)};
        };
        Codes ring[kCodeAhead];
#pragma unroll
        for (int j = 0; j < kCodeAhead; ++j) ring[j] = load_codes(cp + j * cstride);
        cp += kCodeAhead * cstride;
        // the left strip's carry words: group g+1 (chunks 4g+4 .. 4g+7) is
        // loaded at step 2 of group g, two steps before its value is moved
        // (carry rows are padded by 16 words past the last chunk)
        uint4 cw = make_uint4(0, 0, 0, 0);
        uint4 cw_next = feeder ? carry_ld4(left_carry) : make_uint4(0, 0, 0, 0);
        const uint8_t* pml = pm + lane_off;
        const uint32_t csr = d.code_stride;  // runtime value: address IMAD stays on the FMA pipe
        // carry-in masks of the current step, rows 0-7 / 8-15 at bits 31..24
        // (consumed MSB first); the shuffles of a step's carry-outs are issued
        // mid-step and at step end so their latency hides behind row work
        uint32_t cin_lo = 0, cin_hi = 0;
        for (int tg = 0; tg < T; tg += 4) {
            if (feeder && tg < nchunks) {
                cw = cw_next;
                const int lim = nchunks - tg;  // words at or past nchunks stay 0
                uint32_t spins = 0;
                while ((cw.x == 0u) | (lim > 1 && cw.y == 0u) | (lim > 2 && cw.z == 0u) |
                       (lim > 3 && cw.w == 0u)) {
                    cw = carry_ld4(left_carry + tg);  // not yet published: re-poll
                    if (++spins > kPollLimit) {
                        // watchdog: a producer that never publishes (a dead peer
                        // GPU, a broken inbox) fails the call instead of hanging it
                        if (lane == 0) atomicOr(d.error, 1u);
                        return;
                    }
                }
                prefetch_l2(left_carry + tg + 16);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int t = tg + j;
                const int ch = t - int(lane);
                // the next group's carry words are loaded half way through this
                // group: two steps ahead of their use, yet fresh enough that they
                // are usually published (measured: loading them at the group start
                // found them stale and cost C4 +22%, re-polling synchronously)
                if (j == 2 && feeder && tg < nchunks) cw_next = carry_ld4(left_carry + tg + 4);
                if (lane == 0) {
                    uint32_t fl = j == 0 ? cw.x : j == 1 ? cw.y : j == 2 ? cw.z : cw.w;
                    if (t >= nchunks) fl = 0;  // padding rows take no carry
                    cin_lo = (fl & 0xff00u) << 16;
                    cin_hi = (fl & 0xffu) << 24;
                }
                Codes& rc = ring[j];
                const uint32_t code[16] = {rc.a.x, rc.a.y, rc.a.z, rc.a.w, rc.b.x, rc.b.y,
                                           rc.b.z, rc.b.w, rc.c.x, rc.c.y, rc.c.z, rc.c.w,
                                           rc.d.x, rc.d.y, rc.d.z, rc.d.w};
                if constexpr (STORE) hook.dlo = int64_t(t) * 16;
                const bool valid = ch >= 0 && ch < nchunks;
                uint32_t Pm[16][K];
#pragma unroll
                for (int r = 0; r < 16; ++r) load_pm<K>(pml, code[r] * csr, Pm[r]);
                rc = load_codes(cp);  // step t + 4
                prefetch_l2(cp + kCodeL2Ahead * cstride);  // lane 0's chunk: first touch
                cp += cstride;
                uint32_t cout_lo = 0, cout_hi = 0;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    RowStep<K>::chain(V, Pm[r], cin_lo, cout_lo);
                    hook(r, valid, V);
                }
                const uint32_t nl = __shfl_up_sync(kFullMask, cout_lo, 1);
#pragma unroll
                for (int r = 8; r < 16; ++r) {
                    RowStep<K>::chain(V, Pm[r], cin_hi, cout_hi);
                    hook(r, valid, V);
                }
                const uint32_t nh = __shfl_up_sync(kFullMask, cout_hi, 1);
                {
                    // every lane stores (no divergent branch): lane 31's word
                    // goes to the carry row when it is real, everything else
                    // to the CTA's sink
                    const bool pub = has_right && lane == 31 && valid;
                    uint32_t* dst = pub ? my_carry + ch : sink;
                    const uint32_t word = kCarryValid | (cout_lo << 8) | cout_hi;
                    if (ext_right) st_relaxed_sys_nb(dst, word);  // warp-uniform branch
                    else st_relaxed_gpu_nb(dst, word);
                }
                cin_lo = nl << 24;
                cin_hi = nh << 24;
                if (CKPT && valid && (ch + 1) % P.ckpt_chunks == 0 && ch + 1 < nchunks) {
                    // checkpoint (ch + 1) / ckpt_chunks: V after the chunk's rows
                    uint32_t* c = P.ckpt_out + int64_t((ch + 1) / P.ckpt_chunks - 1) * P.W;
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (g * K + k < P.W) c[g * K + k] = V[k];
                }
            }
        }
        __syncwarp();
        if (P.v_out) {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (g * K + k < P.W) P.v_out[g * K + k] = V[k];
        }
        if (P.zeros) {
            int zeros = lane_zero_count<K>(V, g * K, P.cols);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
            if (lane == 0 && zeros) atomicAdd(P.zeros, (unsigned long long)zeros);
        }
    }
}

// ---- exact reference traceback over the stored bit rows ------------------
//
// Row step: the reference walk (serial.cpp:44-58 with cell.hpp:30-38) inside
// row i, entered at column j, leaves the row at
//   j' = h + 1 - diag,  h = highest set bit <= j-1 of E = PM[x_i] | ~V_i,
//   diag = bit h of PM[x_i]   (no set bit: Left to column 0, j' = 0)
// and emits x_i iff diag.  j' is a monotone (non-decreasing) function of j,
// hence so is the exit column of any block of rows: two walks that meet stay
// together, and a walk entering between two walks that met leaves with them.
//
// Parallel walk (replaces the latency-bound serial walk, one row at a time):
//  1. speculate: every block of kWalkRows rows is walked, in parallel, from
//     kWalkCand candidate entry columns spaced kWalkStride apart around the
//     column where the path would cross if it followed the diagonal;
//  2. resolve (one thread, bottom block first): the true entry of block k is
//     the exit of block k-1; if it lies between two candidates whose walks
//     left the block at the same column, that column is the exit (O(1)),
//     otherwise the block is walked from the true entry until the walk meets
//     a neighbouring candidate's column recorded every kWalkCkpt rows (rare,
//     and short: adjacent walks merge within a few dozen rows);
//  3. emit: every block is walked again, in parallel, from its true entry,
//     flagging the rows that emit;
//  4. the flagged row bytes are compacted in row order (forward string).
constexpr int kWalkRows = 256;  // the largest walk block (R <= kWalkRows)
constexpr int kWalkRowsMin = 64;
constexpr int kWalkCand = 128;   // candidates per block (4 warps)
constexpr int kWalkStride = 16;  // columns between candidates
constexpr int kWalkCkpt = 32;    // rows between recorded candidate columns
constexpr int kWalkNCkpt = kWalkRows / kWalkCkpt;

template <int K>
__device__ __forceinline__ uint32_t walk_code(const FillProblem& P, int64_t q) {
    const uint32_t* c32 = reinterpret_cast<const uint32_t*>(P.coded);
    const int64_t r = q & 15, ch = q >> 4;
    return c32[((r >> 2) * P.plane + ch * P.cstride) * 4 + (r & 3)];
}

// Column entering row q-1 (0-based q: DP row i = q + 1) from column j of row
// i; *diag = emission.
template <int K>
__device__ __forceinline__ int64_t walk_step(const FillProblem& P, uint32_t code, int64_t q,
                                             int64_t j, uint32_t* diag) {
    *diag = 0;
    if (j <= 0) return 0;
    int64_t w = (j - 1) >> 5;
    uint32_t mask = (2u << ((j - 1) & 31)) - 1u;
    const uint32_t* pmrow = P.pmg + int64_t(code) * P.W;
    for (;;) {
        const uint32_t pmw = __ldg(pmrow + w);
        const uint32_t e = (pmw | ~P.rows_out[pair_row_index(q, w, K, P.Dpad)]) & mask;
        if (e) {
            const int b = 31 - __clz(e);
            *diag = (pmw >> b) & 1u;
            return w * 32 + b + 1 - int64_t(*diag);
        }
        if (w == 0) return 0;
        --w;
        mask = 0xffffffffu;
    }
}

__device__ __forceinline__ int64_t walk_guess(int64_t top_i, int64_t M, int64_t N) {
    return (top_i * N + M / 2) / M;  // column of the diagonal at DP row top_i
}
__device__ __forceinline__ int64_t walk_cand(int64_t guess, int l, int64_t N) {
    const int64_t c = guess + int64_t(l - kWalkCand / 2) * kWalkStride;
    return c < 0 ? 0 : (c > N ? N : c);
}

// Warp-cooperative walk of DP rows top, top-1, ..., lo+1 entering row `top`
// at column j.  The serial walk costs one dependent global round trip per
// row; here the warp loads, for the next 32 rows at once (lane l: row top-l),
// the three mask words wt, wt-1, wt-2 under the entry column (E = PM | ~V and
// PM), then steps through the rows in registers, row l's words fetched by
// shuffles (they do not depend on j, so they are issued ahead).  The path
// only moves left, so the 96-column window lasts until it is left (then it is
// reloaded at the current row).  visit(i, j_exit, diag) runs (warp-uniform)
// for every row walked and returns false to stop; once j reaches 0 the
// remaining rows exit at 0 without emitting and are not visited.  Returns the
// block's exit column.
template <int K, typename Visit>
__device__ __forceinline__ int64_t warp_walk(const FillProblem& P, int64_t top, int64_t lo,
                                             int64_t j, Visit visit) {
    const int lane = int(lane_id());
    int64_t i = top;
    bool stop = false;
    // loop and branch conditions go through warp votes: they are warp-uniform
    // by construction, and the votes let the compiler see that (otherwise the
    // shuffles below get the slow collective emulation)
    while (__all_sync(kFullMask, i > lo && j > 0 && !stop)) {
        const int64_t wt = (j - 1) >> 5;
        const int64_t q = i - 1 - lane;  // 0-based row of this lane
        uint32_t E0 = 0, E1 = 0, E2 = 0, Q0 = 0, Q1 = 0, Q2 = 0;
        if (q >= lo) {
            const uint32_t* pmrow = P.pmg + int64_t(walk_code<K>(P, q)) * P.W;
            Q0 = __ldg(pmrow + wt);
            E0 = Q0 | ~P.rows_out[pair_row_index(q, wt, K, P.Dpad)];
            if (wt >= 1) {
                Q1 = __ldg(pmrow + wt - 1);
                E1 = Q1 | ~P.rows_out[pair_row_index(q, wt - 1, K, P.Dpad)];
            }
            if (wt >= 2) {
                Q2 = __ldg(pmrow + wt - 2);
                E2 = Q2 | ~P.rows_out[pair_row_index(q, wt - 2, K, P.Dpad)];
            }
        }
        const int nrows = int(i - lo < 32 ? i - lo : 32);
        int done = 0;
        bool go = true;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) {
            const uint32_t e0 = __shfl_sync(kFullMask, E0, l), e1 = __shfl_sync(kFullMask, E1, l),
                           e2 = __shfl_sync(kFullMask, E2, l);
            const uint32_t q0 = __shfl_sync(kFullMask, Q0, l), q1 = __shfl_sync(kFullMask, Q1, l),
                           q2 = __shfl_sync(kFullMask, Q2, l);
            if (__all_sync(kFullMask, go && l < nrows)) {
                // 32-bit column arithmetic (columns < 2^31)
                const int jm = int(j) - 1;
                const int d = int(wt) - (jm >> 5);  // window word holding column j-1
                const uint32_t top_mask = (2u << (jm & 31)) - 1u;
                // masked words from the entry word down to the window bottom
                const uint32_t a = (d == 0 ? e0 : d == 1 ? e1 : e2) & top_mask;
                const uint32_t b = d == 0 ? e1 : d == 1 ? e2 : 0u;
                const uint32_t c = d == 0 ? e2 : 0u;
                const uint32_t qa = d == 0 ? q0 : d == 1 ? q1 : q2;
                const uint32_t qb = d == 0 ? q1 : d == 1 ? q2 : 0u;
                const uint32_t qc = d == 0 ? q2 : 0u;
                const int wa = int(wt) - d;  // word index of a
                int h = -1;
                uint32_t dg = 0;
                if (d > 2) {
                    go = false;  // entry column left the window: reload here
                } else if (a) {
                    const int bb = 31 - __clz(a);
                    h = wa * 32 + bb;
                    dg = (qa >> bb) & 1u;
                } else if (b) {
                    const int bb = 31 - __clz(b);
                    h = (wa - 1) * 32 + bb;
                    dg = (qb >> bb) & 1u;
                } else if (c) {
                    const int bb = 31 - __clz(c);
                    h = (wa - 2) * 32 + bb;
                    dg = (qc >> bb) & 1u;
                } else if (wt - 2 > 0) {
                    go = false;  // no set bit inside the window, more words below
                }
                if (go) {
                    j = h < 0 ? 0 : int64_t(h + 1 - int(dg));  // no set bit at all: Left to 0
                    done = l + 1;
                    if (!visit(i - l, j, dg)) {
                        stop = true;
                        go = false;
                    } else if (j == 0) {
                        go = false;
                    }
                }
            }
        }
        i -= done;
        if (__all_sync(kFullMask, done == 0 && !stop && i > lo && j > 0)) {
            // the next set bit lies more than the window below the entry:
            // one serial row step (warp-uniform), then a fresh window
            uint32_t dg;
            j = walk_step<K>(P, walk_code<K>(P, i - 1), i - 1, j, &dg);
            if (!visit(i, j, dg)) stop = true;
            --i;
        }
    }
    return j;
}

// 1. one CTA (kWalkCand threads) per block of rows, one thread per candidate
// (thousands of independent walks: the row latency is hidden by parallelism)
constexpr int kWalkWarps = 4;  // warps per CTA of the warp-walk kernels
template <int K, int R>
__global__ void __launch_bounds__(kWalkCand) walk_spec_kernel(PairDev d, int32_t* exits,
                                                              int32_t* ckpt) {
    constexpr int kWalkRows = R;  // rows per block (64, 128 or 256)
    __shared__ uint32_t codes[kWalkRows];
    const FillProblem& P = d.prob[0];
    const int64_t M = P.rows, N = P.cols;
    const int64_t k = blockIdx.x;
    const int64_t top = M - k * kWalkRows;  // DP row of the block's first (bottom) row
    const int64_t lo = top - kWalkRows > 0 ? top - kWalkRows : 0;
    for (int64_t i = top - threadIdx.x; i > lo; i -= blockDim.x)
        codes[top - i] = walk_code<K>(P, i - 1);
    __syncthreads();
    int64_t j = walk_cand(walk_guess(P.walk_row0 + top, P.walk_mtot, N), int(threadIdx.x), N);
    int32_t* ck = ckpt + k * (kWalkNCkpt * kWalkCand) + threadIdx.x;
    for (int64_t i = top; i > lo; --i) {
        uint32_t dg;
        if (j > 0) j = walk_step<K>(P, codes[top - i], i - 1, j, &dg);
        const int64_t done = top - i + 1;  // rows walked so far
        if (done % kWalkCkpt == 0 && done < kWalkRows) ck[(done / kWalkCkpt) * kWalkCand] = int32_t(j);
    }
    exits[k * kWalkCand + threadIdx.x] = int32_t(j);
}

// 2. one warp (sequential over blocks, bottom first); entry[k] = true entry
// column of block k
template <int K, int R>
__global__ void __launch_bounds__(32) walk_resolve_kernel(PairDev d, const int32_t* exits,
                                                          const int32_t* ckpt, int32_t* entry,
                                                          uint32_t* misses) {
    constexpr int kWalkRows = R;
    const FillProblem& P = d.prob[0];
    const int64_t M = P.rows, N = P.cols;
    const int64_t nb = (M + kWalkRows - 1) / kWalkRows;
    const int lane = int(lane_id());
    int64_t j = P.walk_entry ? int64_t(*P.walk_entry) : N;
    uint32_t miss = 0;
    const long long t_start = clock64();
    long long t_miss = 0;
    // candidate exits are staged into shared memory 32 blocks at a time
    // (cp.async, the next group in flight while the current one is used): the
    // bottom-up chain over the blocks reads shared memory, not global
    constexpr int kGroup = 32;
    __shared__ __align__(16) int32_t exs[2][kGroup * kWalkCand];
    __shared__ int64_t gs[2][kGroup];  // the blocks' diagonal guesses
    auto stage = [&](int64_t grp) {
        const int64_t k0 = grp * kGroup;
        if (k0 + lane < nb)
            gs[grp & 1][lane] = walk_guess(P.walk_row0 + M - (k0 + lane) * kWalkRows, P.walk_mtot, N);
        if (k0 < nb) {
            const int64_t n16 = ((nb - k0 < kGroup ? nb - k0 : kGroup) * kWalkCand) / 4;
            const int4* src = reinterpret_cast<const int4*>(exits + k0 * kWalkCand);
            const uint32_t dst = uint32_t(__cvta_generic_to_shared(&exs[grp & 1][0]));
            for (int64_t t = lane; t < n16; t += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(t) * 16u),
                             "l"(src + t)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage(0);
    stage(1);
    for (int64_t k = 0; k < nb; ++k) {
        if (lane == 0) entry[k] = int32_t(j);
        if (k % kGroup == 0) {
            asm volatile("cp.async.wait_group 1;" ::: "memory");  // group k / kGroup landed
            __syncwarp();
        }
        const int32_t* exl = &exs[(k / kGroup) & 1][(k % kGroup) * kWalkCand];
        const int64_t top = M - k * kWalkRows;
        const int64_t lo = top - kWalkRows > 0 ? top - kWalkRows : 0;
        const int64_t g = gs[(k / kGroup) & 1][k % kGroup];
        const int32_t* ex = exits + k * kWalkCand;
        int64_t next = -1;
        // bracketing candidates (candidate columns are non-decreasing in l),
        // l in [l0 - 1, l0 + 1], lowest first: the first that qualifies gives
        // the true exit.  One lane, 32-bit column arithmetic (columns < 2^31):
        // this step is the resolve's serial chain (one per block), so it is
        // kept short -- no ballot, one broadcast
        if (lane == 0) {
            const int gi = int(g), Ni = int(N), ji = int(j);
            auto cand = [&](int l) {
                const int c = gi + (l - kWalkCand / 2) * kWalkStride;
                return c < 0 ? 0 : (c > Ni ? Ni : c);
            };
            // fast path: no clamping around the entry -- l follows from j
            const int c0 = gi - (kWalkCand / 2) * kWalkStride;  // unclamped candidate 0
            const int off = ji - c0;
            const int lf = off >> 4;  // kWalkStride = 16
            if (off >= 0 && lf + 1 < kWalkCand && c0 + lf * kWalkStride > 0 &&
                c0 + (lf + 1) * kWalkStride < Ni) {
                const int32_t ea = exl[lf], eb = exl[lf + 1];
                if ((off & (kWalkStride - 1)) == 0 || ea == eb) next = ea;
            }
            const int l0 = (ji - cand(0)) / kWalkStride;
#pragma unroll
            for (int dl = -1; dl <= 1; ++dl) {
                const int l = l0 + dl;
                if (next < 0 && l >= 0 && l < kWalkCand) {
                    const int ca = cand(l);
                    if (ca == ji) {
                        next = exl[l];
                    } else if (l + 1 < kWalkCand && ca < ji && ji < cand(l + 1) &&
                               exl[l] == exl[l + 1]) {
                        next = exl[l];
                    }
                }
            }
        }
        next = __shfl_sync(kFullMask, next, 0);
        if (__all_sync(kFullMask, next < 0)) {
            // Outside the window or the bracket had not merged at the block's
            // end: walk from the true entry, but stop at the first checkpoint
            // where the walk meets a candidate's recorded column (from there
            // on it IS that candidate's path).
            ++miss;
            const long long t0 = clock64();
            const int32_t* ck = ckpt + k * (kWalkNCkpt * kWalkCand);
            // every checkpoint row is compared against all candidates at once
            // (4 per lane, one ballot): the walk has drifted since its entry
            int64_t hit = -1;
            const int64_t jw = warp_walk<K>(P, top, lo, j, [&](int64_t i, int64_t jx, uint32_t) {
                const int64_t walked = top - i + 1;
                if (walked % kWalkCkpt == 0 && walked < kWalkRows) {
                    const int4 r4 = reinterpret_cast<const int4*>(
                        ck + (walked / kWalkCkpt) * kWalkCand)[lane];
                    const int32_t jv = int32_t(jx);
                    const int sub = r4.x == jv ? 0 : r4.y == jv ? 1 : r4.z == jv ? 2 : r4.w == jv ? 3 : -1;
                    const uint32_t hits = __ballot_sync(kFullMask, sub >= 0);
                    if (hits) {
                        const int src = __ffs(hits) - 1;
                        hit = int64_t(src) * 4 + __shfl_sync(kFullMask, sub, src);
                        return false;
                    }
                }
                return true;
            });
            next = hit >= 0 ? ex[hit] : jw;
            t_miss += clock64() - t0;
        }
        j = next;
        if (k % kGroup == kGroup - 1) {
            __syncwarp();  // everyone done with this buffer before it is refilled
            stage(k / kGroup + 2);
        }
    }
    if (lane == 0) {
        if (P.walk_entry) *P.walk_entry = int32_t(j);  // the next band up enters here
        misses[0] = miss;
        misses[1] = uint32_t(t_miss >> 10);                    // diagnostics: kilocycles in
        misses[2] = uint32_t((clock64() - t_start) >> 10);     // fallback walks / in total
    }
}

// 3. one warp per block: flags[q] = 1 iff row q emits (flags pre-zeroed);
// counts[k]
template <int K, int R>
__global__ void __launch_bounds__(32 * kWalkWarps) walk_emit_kernel(PairDev d, const int32_t* entry,
                                                                    uint8_t* flags,
                                                                    uint32_t* counts) {
    constexpr int kWalkRows = R;
    const FillProblem& P = d.prob[0];
    const int64_t M = P.rows;
    const int64_t nb = (M + kWalkRows - 1) / kWalkRows;
    const int64_t k = int64_t(blockIdx.x) * kWalkWarps + (threadIdx.x >> 5);
    if (__all_sync(kFullMask, k >= nb)) return;
    const int lane = int(lane_id());
    const int64_t top = M - k * kWalkRows;
    const int64_t lo = top - kWalkRows > 0 ? top - kWalkRows : 0;
    uint32_t n = 0;
    warp_walk<K>(P, top, lo, entry[k], [&](int64_t i, int64_t, uint32_t dg) {
        n += dg;
        if (lane == 0 && dg) flags[i - 1] = 1;
        return true;
    });
    if (lane == 0) counts[k] = n;
}

// 4a. one thread: output offsets (forward order = blocks from the top rows)
__global__ void __launch_bounds__(1024) walk_scan_kernel(const uint32_t* counts, int64_t nb,
                                                        uint32_t* offsets,
                                                        unsigned long long* total,
                                                        unsigned long long* place,
                                                        unsigned long long* base) {
    // offsets[k] = bytes emitted by blocks above k (rows nearer the top come
    // later in the walk but earlier in the string): a suffix-exclusive scan,
    // one 1024-thread block (thread t owns positions r = nb-1-k in
    // [t per, (t+1) per)), so the block counts are loaded in parallel
    __shared__ unsigned long long wsum[32];
    const int t = int(threadIdx.x), lane = t & 31, warp = t >> 5;
    const int64_t per = (nb + 1023) / 1024;
    const int64_t r0 = int64_t(t) * per, r1 = r0 + per < nb ? r0 + per : nb;
    unsigned long long local = 0;
    for (int64_t r = r0; r < r1; ++r) local += counts[nb - 1 - r];
    unsigned long long incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long ws = wsum[lane];
        unsigned long long wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(kFullMask, wi, o);
            if (lane >= o) wi += v;
        }
        wsum[lane] = wi - ws;  // exclusive warp offsets
    }
    __syncthreads();
    unsigned long long run = wsum[warp] + incl - local;
    for (int64_t r = r0; r < r1; ++r) {
        const int64_t k = nb - 1 - r;
        offsets[k] = uint32_t(run);
        run += counts[k];
    }
    if (t == 1023) {
        *total = run;
        // banded traceback: this band's bytes end where the lower bands' begin
        unsigned long long b = 0;
        if (place) {
            b = place[0] - place[1] - run;
            place[1] += run;
        }
        *base = b;
    }
}

// 4b. one warp per block writes its emitted bytes in row order: lane t
// takes 8 consecutive rows, a warp scan gives its output position
template <int R>
__global__ void __launch_bounds__(128) walk_write_kernel(const uint8_t* x, int64_t M,
                                                         const uint8_t* flags,
                                                         const uint32_t* offsets,
                                                         const unsigned long long* base,
                                                         uint8_t* out) {
    constexpr int kWalkRows = R;
    constexpr int kPerLane = R / 32;  // consecutive rows per lane
    const int64_t nb = (M + kWalkRows - 1) / kWalkRows;
    const int64_t k = int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5);
    if (__all_sync(kFullMask, k >= nb)) return;
    const int lane = int(lane_id());
    const int64_t top = M - k * kWalkRows;
    const int64_t lo = top - kWalkRows > 0 ? top - kWalkRows : 0;
    const int64_t q0 = lo + kPerLane * lane;
    uint32_t f = 0, n = 0;
#pragma unroll
    for (int r = 0; r < kPerLane; ++r) {
        const bool e = q0 + r < top && flags[q0 + r];
        f |= uint32_t(e) << r;
        n += e;
    }
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += t;
    }
    uint8_t* o = out + *base + offsets[k] + (incl - n);
#pragma unroll
    for (int r = 0; r < kPerLane; ++r)
        if ((f >> r) & 1u) *o++ = x[q0 + r];
}

// ---- the reference's full tables from the stored bit rows ----------------
// DpTable (tables.hpp:20-45): (M+1) x (N+1) uint32, row-major, row/col 0 = 0,
//   c[i][j] = zero bits of V_i below column j   (prefix popcount)
// BacktrackTable (tables.hpp:49-71): M x N arrows, (i-1)*N + (j-1):
//   Diag (0) if x_i == y_j; else Up (1) iff bit j-1 of V_i is 0 (then
//   c[i-1][j] > c[i][j-1]); else Left (2)  -- lcs_cell, cell.hpp:30-38.
// One warp per DP row; a lane expands one 32-column word at a time.
template <int K>
__global__ void __launch_bounds__(32) tables_kernel(PairDev d, uint32_t* dp, uint8_t* back) {
    const FillProblem& P = d.prob[0];
    const int64_t N = P.cols, W = P.W;
    const int64_t i = blockIdx.x;  // DP row 0..M
    const int lane = int(threadIdx.x);
    uint32_t* drow = dp + i * (N + 1);
    if (lane == 0) drow[0] = 0;
    if (i == 0) {
        for (int64_t j = 1 + lane; j <= N; j += 32) drow[j] = 0;
        return;
    }
    const int64_t q = i - 1;
    const uint32_t code = walk_code<K>(P, q);
    const uint32_t* pmrow = P.pmg + int64_t(code) * W;
    uint8_t* brow = back + q * N;
    uint32_t base = 0;  // zeros of the words before this chunk of 32 words
    for (int64_t w0 = 0; w0 < W; w0 += 32) {
        const int64_t w = w0 + lane;
        const int64_t c0 = w * 32;  // first column (0-based) of the word
        const int nbits = w < W ? int(N - c0 < 32 ? N - c0 : 32) : 0;
        uint32_t v = 0xffffffffu, pm = 0;
        if (nbits > 0) {
            v = P.rows_out[pair_row_index(q, w, K, P.Dpad)];
            pm = __ldg(pmrow + w);
        }
        const uint32_t valid = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
        const uint32_t z = __popc(~v & valid);
        uint32_t incl = z;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFullMask, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t before = base + incl - z;
        for (int b = 0; b < nbits; ++b) {
            const uint32_t below = (2u << b) - 1u;  // bits 0..b
            drow[c0 + b + 1] = before + __popc(~v & below);
            brow[c0 + b] = ((pm >> b) & 1u) ? uint8_t(0) : (((v >> b) & 1u) ? uint8_t(2) : uint8_t(1));
        }
        base += __shfl_sync(kFullMask, incl, 31);
    }
}

// ---- bidirectional split (Hirschberg's lemma) -----------------------------
// L = max_k  F[k] + R[k],  F[k] = c_top[mid][k] = zeros of Vf below k,
// R[k] = LCS(x[mid:], y[k:]) = zeros of Vr below N - k (Vr: reversed strings).
__global__ void __launch_bounds__(1024) split_prefix_kernel(const uint32_t* vf, const uint32_t* vr,
                                                            int64_t W, uint32_t* pf, uint32_t* pr) {
    __shared__ uint32_t warp_f[32], warp_r[32];
    const int tid = threadIdx.x;
    const int64_t per = (W + 1023) / 1024;
    const int64_t w0 = tid * per, w1 = min(W, w0 + per);
    uint32_t sf = 0, sr = 0;
    for (int64_t w = w0; w < w1; ++w) {
        sf += __popc(~vf[w]);
        sr += __popc(~vr[w]);
    }
    uint32_t inf = sf, inr = sr;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(kFullMask, inf, o), b = __shfl_up_sync(kFullMask, inr, o);
        if (lane >= o) {
            inf += a;
            inr += b;
        }
    }
    if (lane == 31) {
        warp_f[warp] = inf;
        warp_r[warp] = inr;
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t a = warp_f[lane], b = warp_r[lane], ia = a, ib = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(kFullMask, ia, o), y = __shfl_up_sync(kFullMask, ib, o);
            if (lane >= o) {
                ia += x;
                ib += y;
            }
        }
        warp_f[lane] = ia - a;
        warp_r[lane] = ib - b;
    }
    __syncthreads();
    uint32_t rf = warp_f[warp] + inf - sf, rr = warp_r[warp] + inr - sr;
    for (int64_t w = w0; w < w1; ++w) {
        pf[w] = rf;
        pr[w] = rr;
        rf += __popc(~vf[w]);
        rr += __popc(~vr[w]);
    }
}

__device__ __forceinline__ uint32_t zeros_below(const uint32_t* v, const uint32_t* pre,
                                                int64_t k) {
    if (k <= 0) return 0;
    const int64_t w = (k - 1) >> 5;
    const int b = int((k - 1) & 31);  // bits 0..b of word w count
    const uint32_t m = b == 31 ? 0xffffffffu : ((2u << b) - 1u);
    return pre[w] + __popc(~v[w] & m);
}

__global__ void split_combine_kernel(const uint32_t* vf, const uint32_t* vr, const uint32_t* pf,
                                     const uint32_t* pr, int64_t N, unsigned long long* best) {
    uint32_t m = 0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k <= N;
         k += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t f = zeros_below(vf, pf, k);
        const uint32_t r = zeros_below(vr, pr, N - k);
        m = max(m, f + r);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(kFullMask, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(best, (unsigned long long)m);
}

__global__ void reverse_kernel(const uint8_t* src, int64_t n, uint8_t* dst) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[n - 1 - i] = src[i];
}

}  // namespace

cudaError_t pair_prepare(PairDev& d, uint32_t* present256, uint16_t* map256, uint32_t* sigma_dev,
                         cudaStream_t stream, int* sigma_host) {
    cudaError_t e = cudaMemsetAsync(present256, 0, 256 * sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    const int64_t blocks64 = (d.prob[0].cols + 255) / 256;
    const int blocks = int(blocks64 > 1024 ? 1024 : (blocks64 < 1 ? 1 : blocks64));
    pair_alphabet_kernel<<<blocks, 256, 0, stream>>>(d.colp0, d.prob[0].cols, present256);
    pair_codes_kernel<<<1, 32, 0, stream>>>(present256, map256, sigma_dev);
    e = cudaMemcpyAsync(sigma_host, sigma_dev, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    d.map = map256;
    d.sigma = *sigma_host;
    return cudaGetLastError();
}

cudaError_t pair_build_pm(const uint8_t* colp, int64_t cols, const uint16_t* map, int sigma,
                          int64_t W, uint32_t* pmg, cudaStream_t stream) {
    const int64_t blocks = (W + 255) / 256;
    pair_pm_kernel<<<int(blocks), 256, 0, stream>>>(colp, cols, map, sigma, W, pmg);
    return cudaGetLastError();
}

cudaError_t pair_reverse(const uint8_t* src, int64_t n, uint8_t* dst, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int64_t b = (n + 255) / 256;
    reverse_kernel<<<int(b > 4096 ? 4096 : b), 256, 0, stream>>>(src, n, dst);
    return cudaGetLastError();
}

cudaError_t pair_split_combine(const uint32_t* vf, const uint32_t* vr, int64_t W, int64_t N,
                               uint32_t* scratch /* 2 * W */, unsigned long long* best,
                               cudaStream_t stream) {
    split_prefix_kernel<<<1, 1024, 0, stream>>>(vf, vr, W, scratch, scratch + W);
    const int64_t b = (N + 1 + 255) / 256;
    split_combine_kernel<<<int(b > 2048 ? 2048 : b), 256, 0, stream>>>(vf, vr, scratch,
                                                                     scratch + W, N, best);
    return cudaGetLastError();
}

int pair_code_stride(int K) { return K > 4 ? 1024 : 128 * (K == 3 ? 4 : K); }

int pair_smem_bytes(int K, int sigma) { return sigma * pair_code_stride(K) + 64; }  // per warp

int64_t pair_code_plane(int nchunks) { return int64_t(nchunks) + 2 * kPadChunks; }

cudaError_t pair_code_rows(const uint8_t* row, int64_t rows, bool reverse, const uint16_t* map,
                           int K, FillProblem& P, uint4* coded_base, cudaStream_t stream) {
    const int64_t nchp = pair_code_plane(P.nchunks);
    P.plane = nchp;  // 4 planes of uint4, one uint4 per chunk and plane
    P.cstride = 1;
    P.coded = coded_base + kPadChunks * P.cstride;
    const int64_t total = nchp * 16;
    const int64_t b = (total + 255) / 256;
    pair_code_rows_kernel<<<int(b > 8192 ? 8192 : b), 256, 0, stream>>>(
        row, rows, reverse ? 1 : 0, map, P.plane, P.cstride, nchp,
        reinterpret_cast<uint32_t*>(coded_base));
    return cudaGetLastError();
}

template <int K, int MODE>
static cudaError_t launch_strip(const PairDev& dev, int sms, cudaStream_t stream) {
    PairDev d = dev;
    d.code_stride = uint32_t(pair_code_stride(K));
    d.pm_warp_bytes = uint32_t(d.sigma * pair_code_stride(K));
    const int smem = pair_smem_bytes(K, d.sigma);
    cudaError_t e = cudaFuncSetAttribute(pair_strip_kernel<K, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_strip_kernel<K, MODE>, 32,
                                                      smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    int strips = 0;
    for (int q = 0; q < d.nprob; ++q) strips += d.prob[q].nstrips;
    int grid = strips;
    if (grid > sms * occ) grid = sms * occ;
    if (d.max_ctas > 0 && grid > d.max_ctas) grid = d.max_ctas;
    if (grid * 32 > kPairSinkWords) grid = kPairSinkWords / 32;
    if (grid < d.nprob) grid = d.nprob;  // every problem needs a pool of at least one warp
    pair_strip_kernel<K, MODE><<<grid, 32, smem, stream>>>(d);
    return cudaGetLastError();
}

cudaError_t pair_fill(const PairDev& d, int K, bool store, int sms, cudaStream_t stream) {
    const bool ckpt = !store && d.prob[0].ckpt_out != nullptr;
    switch (K * 4 + (store ? 1 : ckpt ? 3 : 0)) {
        case 4: return launch_strip<1, 0>(d, sms, stream);
        case 5: return launch_strip<1, 1>(d, sms, stream);
        case 7: return launch_strip<1, 3>(d, sms, stream);
        case 8: return launch_strip<2, 0>(d, sms, stream);
        case 9: return launch_strip<2, 1>(d, sms, stream);
        case 11: return launch_strip<2, 3>(d, sms, stream);
        case 16: return launch_strip<4, 0>(d, sms, stream);
        case 17: return launch_strip<4, 1>(d, sms, stream);
        case 19: return launch_strip<4, 3>(d, sms, stream);
        case 32: return launch_strip<8, 0>(d, sms, stream);
        case 33: return launch_strip<8, 1>(d, sms, stream);
        case 35: return launch_strip<8, 3>(d, sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

size_t pair_walk_scratch_bytes(int64_t rows) {
    const int64_t nb = (rows + kWalkRowsMin - 1) / kWalkRowsMin;  // any block size R >= 64
    return size_t(nb) * kWalkCand * 4 * (1 + kWalkNCkpt) + size_t(nb) * 12 + size_t(rows) + 128;
}

cudaError_t pair_walk(const PairDev& d, int K, const uint8_t* x, uint8_t* out,
                      unsigned long long* out_len, void* scratch, uint32_t* misses,
                      cudaStream_t stream) {
    const int64_t M = d.prob[0].rows;
    // Block size: each speculative / emit walk is a chain of dependent row
    // steps (an L2 round trip each), so short blocks finish sooner; the
    // resolve is one serial step per block, so long walks want long blocks.
    // Measured (tools/walk_rows_probe.py, lcs_subsequence wall time): 2k rows
    // 0.215 / 0.229 / 0.285 ms at R = 64 / 128 / 256, C1 (10k) 0.563 / 0.464 /
    // 0.512 ms, C3 (100k) 2.93 / 2.75 / 2.73 ms.  WLCS_WALK_ROWS overrides.
    int R = M <= 4096 ? 64 : M <= 65536 ? 128 : 256;
    if (const char* v = getenv("WLCS_WALK_ROWS")) {
        const int f = atoi(v);
        if (f == 64 || f == 128 || f == 256) R = f;
    }
    const int64_t nb = (M + R - 1) / R;
    int32_t* exits = static_cast<int32_t*>(scratch);
    int32_t* ckpt = exits + nb * kWalkCand;
    int32_t* entry = ckpt + nb * kWalkCand * kWalkNCkpt;
    uint32_t* counts = reinterpret_cast<uint32_t*>(entry + nb);
    uint32_t* offsets = counts + nb;
    unsigned long long* base = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(offsets + nb) + 15) & ~uintptr_t(15));
    uint8_t* flags = reinterpret_cast<uint8_t*>(base + 2);
    const int emit_ctas = int((nb + kWalkWarps - 1) / kWalkWarps);
    cudaError_t e = cudaMemsetAsync(flags, 0, size_t(M), stream);
    if (e != cudaSuccess) return e;
    const bool dbg = getenv("WLCS_DEBUG_WALK") != nullptr;
    cudaEvent_t ev[6];
    if (dbg) for (auto& x : ev) cudaEventCreate(&x);
    auto mark = [&](int i) { if (dbg) cudaEventRecord(ev[i], stream); };
    auto run = [&](auto spec, auto resolve, auto emit, auto write) {
        mark(0);
        spec<<<int(nb), kWalkCand, 0, stream>>>(d, exits, ckpt);
        mark(1);
        resolve<<<1, 32, 0, stream>>>(d, exits, ckpt, entry, misses);
        mark(2);
        emit<<<emit_ctas, 32 * kWalkWarps, 0, stream>>>(d, entry, flags, counts);
        mark(3);
        walk_scan_kernel<<<1, 1024, 0, stream>>>(counts, nb, offsets, out_len,
                                              d.prob[0].walk_place, base);
        write<<<emit_ctas, 128, 0, stream>>>(x, M, flags, offsets, base, out);
        mark(4);
        if (dbg) {
            cudaEventSynchronize(ev[4]);
            float t[4];
            for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
            uint32_t ms[3] = {0, 0, 0};
            cudaMemcpy(ms, misses, sizeof(ms), cudaMemcpyDeviceToHost);
            fprintf(stderr,
                    "wlcs walk ms: spec %.3f resolve %.3f emit %.3f scan+write %.3f; blocks %lld, "
                    "resolve misses %u (%u of %u kcycles)\n",
                    t[0], t[1], t[2], t[3], (long long)nb, ms[0], ms[1], ms[2]);
        }
        return cudaGetLastError();
    };
#define WLCS_WALK_CASE(KK, RR)                                                              \
    if (K == KK && R == RR)                                                                 \
        return run(walk_spec_kernel<KK, RR>, walk_resolve_kernel<KK, RR>,                   \
                   walk_emit_kernel<KK, RR>, walk_write_kernel<RR>);
    WLCS_WALK_CASE(1, 64) WLCS_WALK_CASE(1, 128) WLCS_WALK_CASE(1, 256)
    WLCS_WALK_CASE(2, 64) WLCS_WALK_CASE(2, 128) WLCS_WALK_CASE(2, 256)
    WLCS_WALK_CASE(4, 64) WLCS_WALK_CASE(4, 128) WLCS_WALK_CASE(4, 256)
    WLCS_WALK_CASE(8, 64) WLCS_WALK_CASE(8, 128) WLCS_WALK_CASE(8, 256)
#undef WLCS_WALK_CASE
    return cudaErrorInvalidValue;
}

cudaError_t pair_tables(const PairDev& d, int K, uint32_t* dp, uint8_t* back,
                        cudaStream_t stream) {
    const int64_t rows = d.prob[0].rows + 1;
    switch (K) {
        case 1: tables_kernel<1><<<int(rows), 32, 0, stream>>>(d, dp, back); break;
        case 2: tables_kernel<2><<<int(rows), 32, 0, stream>>>(d, dp, back); break;
        case 4: tables_kernel<4><<<int(rows), 32, 0, stream>>>(d, dp, back); break;
        case 8: tables_kernel<8><<<int(rows), 32, 0, stream>>>(d, dp, back); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace wlcs
