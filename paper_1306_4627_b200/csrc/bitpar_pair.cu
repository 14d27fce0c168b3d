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
// the carry masks of lane 31 go through global memory: strip s publishes
// progress[s] with st.release.gpu every 8 chunks, strip s+1 polls it with
// ld.acquire.gpu and reads the masks with ld.global.cg.  Strips are handed out
// by an atomic ticket in increasing order, so a strip only ever waits on a
// strip that is already running (no co-residency assumption).
//
// Traceback: with STORE the fill also writes every row's V words into
// rows_out laid out [lane-group g][row][K] (a lane's K words of consecutive
// rows are adjacent, which is what the walk reads).  The walk applies the
// reference rule (serial.cpp:44-58 with cell.hpp:30-38) in bit form:
//   x_i == y_j                 -> Diag  (emit x_i)
//   bit j-1 of V_i is 0 (H=1)  -> Up     (then c[i-1][j] = c[i][j] > c[i][j-1])
//   otherwise                  -> Left
// so per row it only needs the highest set bit of (PM[x_i] | ~V_i) at or
// below column j: one row per iteration instead of one cell.
#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kCarryBatch = 8;  // chunks fetched / published per handshake

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

template <int K, bool STORE>
struct StoreHook {
    uint32_t* base;  // rows_out + (g * Mpad) * K
    int64_t lo;      // string row index of row 0 of the chunk
    int64_t rows;
    __device__ __forceinline__ void operator()(int r, bool valid, const uint32_t* V) const {
        if constexpr (STORE) {
            if (valid) {
                uint32_t* p = base + (lo + r) * K;
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

template <int K, bool STORE>
__global__ void __launch_bounds__(32) pair_strip_kernel(PairDev d) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* map = reinterpret_cast<uint16_t*>(smem);
    uint8_t* pm = smem + 512;
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    const uint32_t lane = lane_id();
    const int a_r = int(reinterpret_cast<uintptr_t>(d.rowp) & 15u);
    const uint8_t* rstart = d.rowp - a_r;
    const int nchunks = d.nchunks;
    const uint32_t lane_off = PmLayout<K>::word_offset(lane, 0);

    for (;;) {
        uint32_t strip = 0;
        if (lane == 0) strip = atomicAdd(d.ticket, 1u);
        strip = __shfl_sync(kFullMask, strip, 0);
        if (strip >= uint32_t(d.nstrips)) break;
        __syncwarp();
        reinterpret_cast<uint4*>(map)[lane] = reinterpret_cast<const uint4*>(d.map)[lane];
        const int64_t g = int64_t(strip) * 32 + lane;  // global lane-group index
        for (int c = 0; c < d.sigma; ++c) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int64_t w = g * K + k;
                const uint32_t v = w < d.W ? __ldg(d.pmg + int64_t(c) * d.W + w) : 0u;
                *reinterpret_cast<uint32_t*>(pm + c * cs + PmLayout<K>::word_offset(lane, k)) = v;
            }
        }
        __syncwarp();

        uint32_t V[K];
#pragma unroll
        for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
        const bool has_left = strip > 0;
        const bool has_right = strip + 1 < uint32_t(d.nstrips);
        const uint32_t* left_carry = d.carry + int64_t(strip - (has_left ? 1 : 0)) * nchunks;
        uint32_t* my_carry = d.carry + int64_t(strip) * nchunks;
        uint32_t inbuf = 0;
        uint32_t cout = 0;
        StoreHook<K, STORE> hook{STORE ? d.rows_out + g * d.Mpad * K : nullptr, 0, d.rows};
        const int T = nchunks + 31;
        // lane l works on chunk t - l: at t = 0 only lane 0 has a real chunk
        uint32_t vm = (lane == 0 && nchunks > 0) ? chunk_valid_mask(-a_r, d.rows) : 0u;
        uint4 cur = fetch_chunk(rstart, -int(lane), vm, d.row_lo, d.row_hi, d.safe16);
        for (int t = 0; t < T; ++t) {
            if (has_left && (t % kCarryBatch) == 0 && t < nchunks) {
                const int need = min(t + kCarryBatch, nchunks);
                if (lane == 0) {
                    while (int(ld_acquire_gpu(d.progress + strip - 1)) < need) {
                    }
                }
                __syncwarp();
                inbuf = (int(lane) < kCarryBatch && t + int(lane) < nchunks)
                            ? __ldcg(left_carry + t + lane)
                            : 0u;
            }
            const int ch = t - int(lane);
            const int64_t lo = int64_t(ch) * 16 - a_r;
            const uint32_t vm_next =
                (ch + 1 >= 0 && ch + 1 < nchunks) ? chunk_valid_mask(lo + 16, d.rows) : 0u;
            const uint4 nxt = fetch_chunk(rstart, ch + 1, vm_next, d.row_lo, d.row_hi, d.safe16);
            uint32_t cin = __shfl_up_sync(kFullMask, cout, 1);
            const uint32_t from_left = __shfl_sync(kFullMask, inbuf, t % kCarryBatch);
            if (lane == 0) cin = (has_left && t < nchunks) ? from_left : 0u;
            cin <<= 16;
            cout = 0;
            hook.lo = lo;
            uint32_t off[16];
            if (__all_sync(kFullMask, vm == 0xffffu)) {
                chunk_offsets(cur, map, cs, lane_off, off);
            } else {
                chunk_offsets_masked(cur, vm, map, cs, lane_off, off);
            }
            rows16<true, K>(V, pm, off, vm, cin, cout, hook);
            if (has_right && lane == 31 && ch >= 0 && ch < nchunks) {
                my_carry[ch] = cout;
                if (((ch + 1) % kCarryBatch) == 0 || ch + 1 == nchunks)
                    st_release_gpu(d.progress + strip, uint32_t(ch + 1));
            }
            cur = nxt;
            vm = vm_next;
        }
        int zeros = lane_zero_count<K>(V, g * K, d.cols);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
        if (lane == 0 && zeros) atomicAdd(d.zeros, (unsigned long long)zeros);
    }
}

// Exact reference traceback over stored bit rows (one thread).
// out receives the subsequence in REVERSE order; *out_len its length.
template <int K>
__global__ void pair_walk_kernel(PairDev d, const uint8_t* x, uint8_t* out,
                                 unsigned long long* out_len) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t i = d.rows, j = d.cols;  // 1-based DP coordinates
    unsigned long long len = 0;
    const int64_t W = d.W;
    while (i > 0 && j > 0) {
        const int64_t q = i - 1;  // string index of row i
        const uint32_t code = d.map[x[q]];
        const uint32_t* pmrow = d.pmg + int64_t(code) * W;
        int64_t w = (j - 1) >> 5;
        int b = int((j - 1) & 31);
        // V_i word w lives at rows_out[((w / K) * Mpad + q) * K + w % K]
        uint32_t v = d.rows_out[((w / K) * d.Mpad + q) * K + (w % K)];
        uint32_t pmw = __ldg(pmrow + w);
        uint32_t e = (pmw | ~v) & (b == 31 ? 0xffffffffu : ((2u << b) - 1u));
        while (e == 0 && w > 0) {
            --w;
            v = d.rows_out[((w / K) * d.Mpad + q) * K + (w % K)];
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

}  // namespace

cudaError_t pair_prepare(PairDev& d, uint32_t* present256, uint16_t* map256, uint32_t* sigma_dev,
                         cudaStream_t stream, int* sigma_host) {
    cudaError_t e = cudaMemsetAsync(present256, 0, 256 * sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    const int64_t blocks64 = (d.cols + 255) / 256;
    const int blocks = int(blocks64 > 1024 ? 1024 : (blocks64 < 1 ? 1 : blocks64));
    pair_alphabet_kernel<<<blocks, 256, 0, stream>>>(d.colp, d.cols, present256);
    pair_codes_kernel<<<1, 32, 0, stream>>>(present256, map256, sigma_dev);
    e = cudaMemcpyAsync(sigma_host, sigma_dev, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return e;
    d.map = map256;
    d.sigma = *sigma_host;
    return cudaGetLastError();
}

cudaError_t pair_build_pm(const PairDev& d, cudaStream_t stream) {
    const int64_t blocks = (d.W + 255) / 256;
    pair_pm_kernel<<<int(blocks), 256, 0, stream>>>(d.colp, d.cols, d.map, d.sigma, d.W,
                                                   const_cast<uint32_t*>(d.pmg));
    return cudaGetLastError();
}

int pair_smem_bytes(int K, int sigma) {
    const int cs = K > 4 ? 1024 : 128 * (K == 3 ? 4 : K);
    return 512 + sigma * cs;
}

template <int K, bool STORE>
static cudaError_t launch_strip(const PairDev& d, int sms, cudaStream_t stream) {
    const int smem = pair_smem_bytes(K, d.sigma);
    cudaError_t e = cudaFuncSetAttribute(pair_strip_kernel<K, STORE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_strip_kernel<K, STORE>, 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    int grid = sms * occ;
    if (grid > d.nstrips) grid = d.nstrips;
    pair_strip_kernel<K, STORE><<<grid, 32, smem, stream>>>(d);
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
