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

__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr uint32_t kCarryValid = 0x10000u;  // carry words: valid flag | 16-row mask
constexpr int kPairWarps = 4;               // max warps per CTA

// Row coding: entry i = map[row byte i] (the row's match-mask record in the
// strip's shared-memory table is at code * code_stride).  Rows
// outside [0, rows) -- the lane pipeline's prologue/epilogue chunks -31 ..
// nchunks + 30 and the tail of the last chunk -- are 0 (code 0 = all-zero
// masks = identity row, also carry-neutral), so the strip kernel needs no
// row-validity masks.  Layout: 4 planes of uint4; plane j holds entries
// 4j..4j+3 of every chunk, chunk ch at index ch + kPadChunks, so the warp's
// j-th LDG.128 (lanes on chunks t-0 .. t-31) is one contiguous 512-byte run.
// With `reverse` the row string is coded back to front.
constexpr int kPadChunks = 32;

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

// Strip kernel.  Tickets t = 0, 1, ... map to (problem t % nprob, strip
// t / nprob), so inside each problem strips start in order and a strip only
// ever waits on a strip that is already running.
//
// Per step a lane reads its 16-row chunk as 16 pre-coded offsets (4
// coalesced LDG.128, prefetched one step ahead) and runs 16 row updates: per row one IADD3 for
// the address, one LDS for the masks, 3 ALU ops per word plus two for the
// carry bit in and out.
//
// Carry handoff between strips: lane 31 of strip s publishes the 16-row carry
// mask of chunk ch as one relaxed 32-bit store (kCarryValid | mask) into a
// zero-initialised buffer -- the data word is its own ready flag, so no fence
// is needed.  Strip s+1 reads the words in windows, the
// next window prefetched while the current one is consumed (`win` chunks, 16 by default); a word that was
// still 0 when loaded is re-polled.  (A per-step ring refill was tried: its
// pending load blocks the next step's shuffle of the ring register.)
//
// CTAs are persistent with kPairWarps independent warps, one per SM
// sub-partition, so no strip shares an ALU pipe with another strip (a strip
// on a shared sub-partition would run at half speed and throttle every strip
// downstream of it).
template <int K, bool STORE>
__global__ void __launch_bounds__(32 * kPairWarps) pair_strip_kernel(PairDev d) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* pm = smem + (threadIdx.x >> 5) * uint32_t(d.sigma) * PmLayout<K>::code_stride;
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    const uint32_t lane = lane_id();
    const uint32_t lane_off = PmLayout<K>::word_offset(lane, 0);
    for (;;) {
        uint32_t tk = 0;
        if (lane == 0) tk = atomicAdd(d.ticket, 1u);
        tk = __shfl_sync(kFullMask, tk, 0);
        if (tk >= uint32_t(d.nprob * d.prob[0].nstrips)) break;
        const FillProblem& P = d.prob[tk % uint32_t(d.nprob)];
        const uint32_t strip = tk / uint32_t(d.nprob);
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
        const bool has_left = strip > 0;
        const bool has_right = strip + 1 < uint32_t(P.nstrips);
        const uint32_t* left_carry = P.carry + int64_t(has_left ? strip - 1 : 0) * nchunks;
        uint32_t* my_carry = P.carry + int64_t(strip) * nchunks;
        const int win = d.carry_win;
        // carry windows of `win` chunks: lanes 0..win-1 hold the words
        // of the current window (cur_in) and of the next one (nxt_in)
        auto carry_word = [&](int ch) -> uint32_t {
            return (has_left && int(lane) < win && ch < nchunks)
                       ? ld_relaxed_gpu(left_carry + ch)
                       : kCarryValid;
        };
        uint32_t cur_in = carry_word(int(lane)), nxt_in = carry_word(win + int(lane));
        uint32_t cout = 0;
        StoreHook<K, STORE> hook{
            STORE ? P.rows_out + ((int64_t(strip) * P.Dpad) * 32 + lane) * K : nullptr, 0};
        const int T = nchunks + 31;
        // lane l works on chunk t - l (chunks < 0 / >= nchunks are padding);
        // codes are prefetched two steps ahead
        const int64_t cstride = P.cstride;
        const uint4* cp = P.coded - int64_t(lane) * cstride;
        uint4 a0 = __ldg(cp), a1 = __ldg(cp + plane), a2 = __ldg(cp + 2 * plane),
              a3 = __ldg(cp + 3 * plane);
        cp += cstride;
        uint4 b0 = __ldg(cp), b1 = __ldg(cp + plane), b2 = __ldg(cp + 2 * plane),
              b3 = __ldg(cp + 3 * plane);
        const uint8_t* pml = pm + lane_off;
        const uint32_t csr = d.code_stride;  // runtime value: address IMAD stays on the FMA pipe
        for (int t = 0; t < T; ++t) {
            uint32_t from_left = 0;
            if (has_left && t < nchunks) {
                if ((t & (win - 1)) == 0) {
                    if (t > 0) {
                        cur_in = nxt_in;
                        nxt_in = carry_word(t + win + int(lane));
                    }
                    // wait for the current window (normally already published)
                    while (__any_sync(kFullMask, cur_in == 0u))
                        if (cur_in == 0u) cur_in = carry_word(t + int(lane));
                }
                from_left = __shfl_sync(kFullMask, cur_in, t & (win - 1));
            }
            const int ch = t - int(lane);
            cp += cstride;
            const uint4 n0 = __ldg(cp), n1 = __ldg(cp + plane), n2 = __ldg(cp + 2 * plane),
                        n3 = __ldg(cp + 3 * plane);
            uint32_t cin = __shfl_up_sync(kFullMask, cout, 1);
            if (lane == 0) cin = from_left & 0xffffu;
            cin <<= 16;
            cout = 0;
            const uint32_t code[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                                       a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
            if constexpr (STORE) hook.dlo = int64_t(t) * 16;
            const bool valid = ch >= 0 && ch < nchunks;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                row_update<true, K>(V, pml, code[r] * csr, cin, cout);
                hook(r, valid, V);
            }
            if (has_right && lane == 31 && valid) st_relaxed_gpu(my_carry + ch, kCarryValid | cout);
            a0 = b0; a1 = b1; a2 = b2; a3 = b3;
            b0 = n0; b1 = n1; b2 = n2; b3 = n3;
        }
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

// Exact reference traceback over stored bit rows (one thread).
// out receives the subsequence in REVERSE order; *out_len its length.
template <int K>
__global__ void pair_walk_kernel(PairDev d, const uint8_t* x, uint8_t* out,
                                 unsigned long long* out_len) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const FillProblem& P = d.prob[0];
    int64_t i = P.rows, j = P.cols;  // 1-based DP coordinates
    unsigned long long len = 0;
    const int64_t W = P.W;
    while (i > 0 && j > 0) {
        const int64_t q = i - 1;  // string index of row i
        const uint32_t code = d.map[x[q]];
        const uint32_t* pmrow = P.pmg + int64_t(code) * W;
        int64_t w = (j - 1) >> 5;
        int b = int((j - 1) & 31);
        uint32_t v = P.rows_out[pair_row_index(q, w, K, P.Dpad)];
        uint32_t pmw = __ldg(pmrow + w);
        uint32_t e = (pmw | ~v) & (b == 31 ? 0xffffffffu : ((2u << b) - 1u));
        while (e == 0 && w > 0) {
            --w;
            v = P.rows_out[pair_row_index(q, w, K, P.Dpad)];
            pmw = __ldg(pmrow + w);
            e = pmw | ~v;
        }
        if (e == 0) break;  // Left all the way to column 0
        b = 31 - __clz(e);
        const int64_t jj = w * 32 + b + 1;  // event column
        if ((pmw >> b) & 1u) {
            out[len++] = x[q];
            i -= 1;
            j = jj - 1;
        } else {
            i -= 1;
            j = jj;
        }
    }
    *out_len = len;
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

int pair_smem_bytes(int K, int sigma) { return sigma * pair_code_stride(K); }  // per warp

int64_t pair_code_plane(int nchunks) { return int64_t(nchunks) + 2 * kPadChunks; }

cudaError_t pair_code_rows(const uint8_t* row, int64_t rows, bool reverse, const uint16_t* map,
                           int K, FillProblem& P, uint4* coded_base, cudaStream_t stream) {
    const int64_t nchp = pair_code_plane(P.nchunks);
    const char* env = std::getenv("WLCS_PAIR_LAYOUT");
    if (env && *env == '1') {  // chunk-contiguous
        P.plane = 1;
        P.cstride = 4;
    } else {  // planes
        P.plane = nchp;
        P.cstride = 1;
    }
    P.coded = coded_base + kPadChunks * P.cstride;
    const int64_t total = nchp * 16;
    const int64_t b = (total + 255) / 256;
    pair_code_rows_kernel<<<int(b > 8192 ? 8192 : b), 256, 0, stream>>>(
        row, rows, reverse ? 1 : 0, map, P.plane, P.cstride, nchp,
        reinterpret_cast<uint32_t*>(coded_base));
    return cudaGetLastError();
}

template <int K, bool STORE>
static cudaError_t launch_strip(const PairDev& d, int sms, cudaStream_t stream) {
    const_cast<PairDev&>(d).code_stride = uint32_t(pair_code_stride(K));
    const char* wenv = std::getenv("WLCS_PAIR_WIN");
    int win = wenv && *wenv ? std::atoi(wenv) : 16;
    if (win != 4 && win != 8 && win != 16 && win != 32) win = 16;
    const_cast<PairDev&>(d).carry_win = win;
    const char* env = std::getenv("WLCS_PAIR_WPC");
    int wpc = env && *env ? std::atoi(env) : 1;
    if (wpc < 1 || wpc > kPairWarps) wpc = 1;
    const int smem = wpc * pair_smem_bytes(K, d.sigma);
    cudaError_t e = cudaFuncSetAttribute(pair_strip_kernel<K, STORE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_strip_kernel<K, STORE>, 32 * wpc,
                                                      smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    const int strips = d.nprob * d.prob[0].nstrips;
    int grid = (strips + wpc - 1) / wpc;
    if (grid > sms * occ) grid = sms * occ;
    pair_strip_kernel<K, STORE><<<grid, 32 * wpc, smem, stream>>>(d);
    return cudaGetLastError();
}

cudaError_t pair_fill(const PairDev& d, int K, bool store, int sms, cudaStream_t stream) {
    switch (K * 2 + (store ? 1 : 0)) {
        case 2: return launch_strip<1, false>(d, sms, stream);
        case 3: return launch_strip<1, true>(d, sms, stream);
        case 4: return launch_strip<2, false>(d, sms, stream);
        case 5: return launch_strip<2, true>(d, sms, stream);
        case 8: return launch_strip<4, false>(d, sms, stream);
        case 9: return launch_strip<4, true>(d, sms, stream);
        case 16: return launch_strip<8, false>(d, sms, stream);
        case 17: return launch_strip<8, true>(d, sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t pair_walk(const PairDev& d, int K, const uint8_t* x, uint8_t* out_rev,
                      unsigned long long* out_len, cudaStream_t stream) {
    switch (K) {
        case 1: pair_walk_kernel<1><<<1, 32, 0, stream>>>(d, x, out_rev, out_len); break;
        case 2: pair_walk_kernel<2><<<1, 32, 0, stream>>>(d, x, out_rev, out_len); break;
        case 4: pair_walk_kernel<4><<<1, 32, 0, stream>>>(d, x, out_rev, out_len); break;
        case 8: pair_walk_kernel<8><<<1, 32, 0, stream>>>(d, x, out_rev, out_len); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace wlcs
