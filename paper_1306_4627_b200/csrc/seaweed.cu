// seaweed.cu -- row-band decomposition of one pair through semi-local LCS
// (seaweed combing), the prototype of the split that lets the ROWS of a long
// pair run in parallel.
//
// The reference fills one table row after row (proj/src/serial.cpp:11-30,
// parallel.cpp:172-226); every row depends on the one above, which caps the
// strong scaling of a single pair.  Semi-local LCS removes that dependency:
//
//  * Seaweed combing of a band of rows a (m_b rows) against all columns b
//    (n): seaweeds enter on the left (row i, numbered m_b - 1 - i, i.e. bottom
//    to top) and on the top (column j, numbered m_b + j); in every cell the
//    row's and the column's seaweeds swap places iff the symbols match or they
//    have already crossed (h > v), otherwise they cross.  Each band is combed
//    independently -- concurrently -- from this canonical start.
//  * Top seaweed k leaves the band at the bottom of column e_k >= k, or on the
//    right (e_k = n).  The band's string-substring LCS is then
//        H(i, j) = LCS(a, b[i, j)) = (j - i) - #{k in [i, j) : e_k < j}.
//  * Bands compose through the DP boundary: the bottom row C of a band under
//    the top row T is C[j] = max_{i <= j} T[i] + H(i, j), and the pair's
//    length is the last band's C[n].
//
// Prototype status: the combing is cell by cell (one warp per band, an
// anti-diagonal wavefront over 32 R rows at a time), the combine is the
// direct O(n^2) max-plus product.  Both are exact (tests/test_seaweed.py and
// the -m gpu parity test against the oracle); neither is the fast form (a
// bit-parallel combing and an O(n log n) Monge / steady-ant combine).
#include "wlcs_common.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kSeaR = 8;                  // rows per lane
constexpr uint32_t kSeaNoRow = 0x100u;   // code of a padding row: never matches a byte

__device__ __forceinline__ void st_global_u32_if(bool pred, uint32_t* p, uint32_t val) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.u32 [%1], %2;\n\t}" ::"r"(
            uint32_t(pred)),
        "l"(p), "r"(val)
        : "memory");
}

// One warp per band; sub-bands of 32 R rows in sequence, the column seaweeds
// v[] handed from one sub-band to the next through global memory.
__global__ void __launch_bounds__(32) seaweed_band_kernel(SeaDev d) {
    const int band = int(blockIdx.x);
    const int lane = int(lane_id());
    const int64_t r0 = d.row_lo[band], r1 = d.row_lo[band + 1];
    const int64_t mb = r1 - r0, n = d.n;
    uint32_t* v = d.v + int64_t(band) * n;
    uint32_t* e = d.e + int64_t(band) * n;
    for (int64_t j = lane; j < n; j += 32) v[j] = uint32_t(mb + j);
    __syncwarp();
    for (int64_t s0 = 0; s0 < mb; s0 += 32 * kSeaR) {
        uint32_t h[kSeaR], a[kSeaR];
#pragma unroll
        for (int r = 0; r < kSeaR; ++r) {
            const int64_t i = s0 + int64_t(lane) * kSeaR + r;  // row within the band
            const bool ok = i < mb;
            a[r] = ok ? uint32_t(d.rowp[r0 + i]) : kSeaNoRow;
            h[r] = ok ? uint32_t(mb - 1 - i) : 0u;  // padding rows never swap
        }
        uint32_t pass = 0;  // column seaweed handed down to the next lane
        const int64_t T = n + 31;
        for (int64_t t = 0; t < T; ++t) {
            const uint32_t up = __shfl_up_sync(kFullMask, pass, 1);
            const int64_t j = t - lane;
            const bool valid = j >= 0 && j < n;
            uint32_t s = lane == 0 ? (valid ? v[j] : 0u) : up;
            const uint32_t c = valid ? uint32_t(__ldg(d.colp + j)) : 0x200u;
#pragma unroll
            for (int r = 0; r < kSeaR; ++r) {
                const bool swap = valid && (a[r] == c || h[r] > s);
                const uint32_t hs = h[r];
                h[r] = swap ? s : hs;
                s = swap ? hs : s;
            }
            pass = s;
            // read by lane 0 at step j, written at j + 31; predicated, not
            // branched (a branch would put the next shuffle on its slow path)
            st_global_u32_if(lane == 31 && valid, v + (valid ? j : 0), s);
        }
        __syncwarp();
    }
    // exits of the top seaweeds: bottom column or the right side (n)
    for (int64_t k = lane; k < n; k += 32) e[k] = uint32_t(n);
    __syncwarp();
    for (int64_t j = lane; j < n; j += 32) {
        const uint32_t s = v[j];
        if (s >= uint32_t(mb)) e[s - uint32_t(mb)] = uint32_t(j);
    }
}

// C[j] = max_{i <= j} T[i] + (j - i) - #{k in [i, j) : e_k < j}, j = 0..n.
__global__ void seaweed_combine_kernel(const uint32_t* __restrict__ e, int64_t n,
                                       const uint32_t* __restrict__ T, uint32_t* __restrict__ C) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j > n) return;
    int64_t best = int64_t(T[j]);
    int64_t cnt = 0;
    for (int64_t i = j - 1; i >= 0; --i) {
        cnt += e[i] < uint32_t(j) ? 1 : 0;
        const int64_t val = int64_t(T[i]) + (j - i) - cnt;
        best = val > best ? val : best;
    }
    C[j] = uint32_t(best);
}

}  // namespace

cudaError_t seaweed_bands(const SeaDev& d, int bands, uint32_t* t0, uint32_t* t1,
                          uint32_t* out, cudaStream_t stream) {
    seaweed_band_kernel<<<bands, 32, 0, stream>>>(d);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(t0, 0, size_t(d.n + 1) * 4, stream);
    if (err != cudaSuccess) return err;
    const int threads = 256;
    const int blocks = int((d.n + 1 + threads - 1) / threads);
    for (int b = 0; b < bands; ++b) {
        seaweed_combine_kernel<<<blocks, threads, 0, stream>>>(d.e + int64_t(b) * d.n, d.n, t0,
                                                               t1);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        uint32_t* tmp = t0;
        t0 = t1;
        t1 = tmp;
    }
    return cudaMemcpyAsync(out, t0 + d.n, 4, cudaMemcpyDeviceToDevice, stream);
}

}  // namespace wlcs
