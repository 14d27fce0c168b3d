// wavefront.cu -- the cell-wavefront fill variant (WLCS_VARIANT_WAVEFRONT).
//
// Same integer result as the bit-parallel variant and as the reference's
// cell recurrence (proj/src/serial.cpp:16-30, cell.hpp:20-38):
//   c[i][j] = x_i == y_j ? c[i-1][j-1] + 1 : max(c[i-1][j], c[i][j-1])
// evaluated branch-free with the Blackwell DPX three-way max as
//   c = __vimax3_s32(up, left, diag + match)
// (diag + match is one add-with-carry of the row's match bit)
// (valid because c[i-1][j-1] + 1 >= max(up, left) on a match and
// c[i-1][j-1] <= max(up, left) always).
//
// Tiling: a warp sweeps a band of 32*R rows (R consecutive rows per lane)
// across all columns as an anti-diagonal wavefront -- lane l works on column
// t - l at step t.  The bottom-row value of lane l-1 (the "up" of lane l's
// first row) and the column byte travel down the warp in ONE packed
// __shfl_up_sync per step ((value << 8) | byte); inside a lane the R rows
// pass values in registers.  The match bits of a lane's R rows against a
// column byte come from a per-lane 256-entry table in shared memory (one LDS
// per step instead of R compares).  Band b+1 takes its top boundary from the
// bottom row of band b.
//
//  * batch kernel: one warp per pair, bands processed in sequence by the same
//    warp; the column string and the boundary row live in the warp's shared
//    memory (column string = the shorter string, <= kWaveMaxCols bytes;
//    longer pairs are listed for the single-pair kernel);
//  * pair kernel: bands of one pair run concurrently on many warps; band b
//    publishes its bottom row as self-validating words (value << 8 | tag)
//    into a ring of boundary rows, band b+1 reads them in windows of 32
//    columns, one window ahead (same hand-off scheme as the strip kernel).
#include "wlcs_common.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kWaveR = 8;           // rows per lane
constexpr int kWaveBand = 32 * kWaveR;
constexpr int kWaveWarps = 4;       // warps per CTA (batch kernel)
constexpr int kWaveTab = 32 * 256;     // per-warp match table bytes: [lane][byte] -> R-bit row mask


// Steps of one band: lane l owns rows i0 + R l + r and, at step t, the two
// columns 2(t - l) and 2(t - l) + 1 (two columns per step halve the per-step
// work of the shuffle, the bounds tests and the boundary hand-off).
// Prov(t, upA, yA, upB, yB) is called by the whole warp at step t and sets,
// for lane 0 (columns 2t, 2t+1), the top boundary c[i0-1][.] (0 for the first
// band) and the column bytes; BottomFn(j, v) receives c[i0 + 32R - 1][j] from
// lane 31.  Returns, in every lane, the final value of row `want_row` (0 if
// not in this band).
template <typename Prov, typename BottomFn>
__device__ __forceinline__ int32_t sweep_band(const uint8_t* rowp, int64_t i0, int64_t m,
                                              int64_t n, uint8_t* tab, Prov prov,
                                              BottomFn bottom, int64_t want_row) {
    const int lane = int(lane_id());
    // lane's match table: tab[lane][c] bit 7-r = (x_{i0 + R lane + r} == c)
    uint8_t* mt = tab + lane * 256;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 64; ++k) reinterpret_cast<uint32_t*>(mt)[k] = 0u;
#pragma unroll
    for (int r = 0; r < kWaveR; ++r) {
        const int64_t i = i0 + int64_t(lane) * kWaveR + r;
        if (i < m) mt[rowp[i]] |= uint8_t(0x80u >> r);  // row r at bit 7 - r
    }
    __syncwarp();
    int32_t left[kWaveR];
#pragma unroll
    for (int r = 0; r < kWaveR; ++r) left[r] = 0;
    int32_t prev_up = 0;  // c[top-1][j-1] of this lane's first row
    uint32_t sendA = 0, sendB = 0;
    const int n2 = int((n + 1) >> 1);  // column pairs (n < 2^31)
    const int T = n2 + 31;
    // one column: 8 rows, each match bit shifted into the carry flag so that
    // diag + match is one add-with-carry
    auto column = [&](int32_t up, uint32_t y) {
        uint32_t mm = uint32_t(mt[y]) << 24;
        int32_t u = up, dg = prev_up;
#pragma unroll
        for (int r = 0; r < kWaveR; ++r) {
            int32_t dm;
            asm("{\n\tadd.cc.u32 %0, %0, %0;\n\taddc.u32 %1, %2, 0;\n\t}"
                : "+r"(mm), "=r"(dm)
                : "r"(dg));
            const int32_t v = __vimax3_s32(u, left[r], dm);
            dg = left[r];
            left[r] = v;
            u = v;
        }
        prev_up = up;
        return u;
    };
    for (int t = 0; t < T; ++t) {
        const uint32_t ra = __shfl_up_sync(kFullMask, sendA, 1);
        const uint32_t rb = __shfl_up_sync(kFullMask, sendB, 1);
        const int jp = t - lane;  // column pair
        int32_t upA0, upB0;
        uint32_t yA0, yB0;
        prov(t, upA0, yA0, upB0, yB0);
        const int32_t upA = lane == 0 ? upA0 : int32_t(ra >> 8);
        const uint32_t yA = lane == 0 ? yA0 : (ra & 0xffu);
        const int32_t upB = lane == 0 ? upB0 : int32_t(rb >> 8);
        const uint32_t yB = lane == 0 ? yB0 : (rb & 0xffu);
        if (unsigned(jp) < unsigned(n2)) {
            const int64_t ja = 2 * int64_t(jp);
            const int32_t ua = column(upA, yA);
            sendA = (uint32_t(ua) << 8) | yA;
            if (lane == 31) bottom(ja, ua);
            if (ja + 1 < n) {  // false only for the last pair of an odd n
                const int32_t ub = column(upB, yB);
                sendB = (uint32_t(ub) << 8) | yB;
                if (lane == 31) bottom(ja + 1, ub);
            }
        }
    }
    int32_t res = 0;
    const int64_t k = want_row - i0;
    if (k >= 0 && k < kWaveBand) {
        const int owner = int(k / kWaveR), rr = int(k % kWaveR);
        int32_t mine = left[0];
#pragma unroll
        for (int r = 1; r < kWaveR; ++r)
            if (r == rr) mine = left[r];
        res = __shfl_sync(kFullMask, mine, owner);
    }
    return res;
}

// ---------------------------------------------------------------- batch
__global__ void __launch_bounds__(32 * kWaveWarps) wave_batch_kernel(WaveBatchDev d) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = int(threadIdx.x >> 5);
    const int lane = int(lane_id());
    uint8_t* base = smem + warp * (kWaveMaxCols * 5 + kWaveTab);
    int32_t* bnd = reinterpret_cast<int32_t*>(base);
    uint8_t* cs = base + kWaveMaxCols * 4;
    uint8_t* tab = base + kWaveMaxCols * 5;
    for (;;) {
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(d.counter, 1u);
        p = __shfl_sync(kFullMask, p, 0);
        if (p >= d.pairs) break;
        const uint64_t xo = d.xoff[p], xn = d.xoff[p + 1] - xo;
        const uint64_t yo = d.yoff[p], yn = d.yoff[p + 1] - yo;
        // length is symmetric: columns = the shorter string
        const bool x_cols = xn < yn;
        const uint8_t* rowp = x_cols ? d.ys + yo : d.xs + xo;
        const uint8_t* colp = x_cols ? d.xs + xo : d.ys + yo;
        const int64_t m = int64_t(x_cols ? yn : xn), n = int64_t(x_cols ? xn : yn);
        if (m == 0 || n == 0) {
            if (lane == 0) d.out[p] = 0;
            continue;
        }
        if (n > kWaveMaxCols) {
            if (lane == 0) d.overflow[atomicAdd(d.overflow_count, 1u)] = p;
            continue;
        }
        __syncwarp();
        for (int64_t k = lane; k < n; k += 32) cs[k] = colp[k];
        __syncwarp();
        int32_t res = 0;
        for (int64_t i0 = 0; i0 < m; i0 += kWaveBand) {
            const bool first = i0 == 0;
            const int32_t v = sweep_band(
                rowp, i0, m, n, tab,
                [&](int t, int32_t& upA, uint32_t& yA, int32_t& upB, uint32_t& yB) {
                    const int64_t ja = 2 * int64_t(t);
                    const bool ina = lane == 0 && ja < n, inb = lane == 0 && ja + 1 < n;
                    upA = (ina && !first) ? bnd[ja] : 0;
                    yA = ina ? uint32_t(cs[ja]) : 0u;
                    upB = (inb && !first) ? bnd[ja + 1] : 0;
                    yB = inb ? uint32_t(cs[ja + 1]) : 0u;
                },
                [&](int64_t j, int32_t v) { bnd[j] = v; }, m - 1);
            if (i0 + kWaveBand >= m) res = v;
            __syncwarp();
        }
        if (lane == 0) d.out[p] = uint32_t(res);
    }
}

// ----------------------------------------------------------- single pair
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(32) wave_pair_kernel(WavePairDev d) {
    __shared__ __align__(16) uint8_t tab[kWaveTab];
    const int lane = int(lane_id());
    const int64_t n = d.n, m = d.m;
    const uint32_t nbands = uint32_t((m + kWaveBand - 1) / kWaveBand);
    for (;;) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(d.ticket, 1u);
        b = __shfl_sync(kFullMask, b, 0);
        if (b >= nbands) break;
        const int64_t i0 = int64_t(b) * kWaveBand;
        const bool first = b == 0, last = b + 1 == nbands;
        // ring of nbuf boundary rows; words are (value << 8) | tag with the
        // writer's generation tag, so stale words of an earlier band are
        // recognised without re-zeroing (a band b+nbuf-1 that reuses band b-1's
        // row writes column j only after band b has read it: band b+k reaches
        // column j no earlier than 31 k steps after band b)
        const uint32_t prev_tag = first ? 0u : ((b - 1) / d.nbuf) % 255u + 1u;
        const uint32_t my_tag = (b / d.nbuf) % 255u + 1u;
        const uint32_t* above = d.bnd + int64_t(first ? 0 : (b - 1) % d.nbuf) * d.bstride;
        uint32_t* below = d.bnd + int64_t(b % d.nbuf) * d.bstride;
        // windows of 32 columns: lane k holds column base + k (boundary word
        // and column byte) for the current and the next window
        auto load_win = [&](int64_t base, uint32_t& w, uint32_t& c) {
            const int64_t jj = base + lane;
            w = (!first && jj < n) ? ld_relaxed(above + jj) : prev_tag;
            c = jj < n ? uint32_t(d.colp[jj]) : 0u;
        };
        uint32_t cw, cc, nw, nc;
        load_win(0, cw, cc);
        load_win(32, nw, nc);
        const int32_t v = sweep_band(
            d.rowp, i0, m, n, tab,
            [&](int t, int32_t& upA, uint32_t& yA, int32_t& upB, uint32_t& yB) {
                const int64_t ja = 2 * int64_t(t);  // columns ja, ja + 1 (same window)
                if ((ja & 31) == 0 && ja < n) {
                    if (ja > 0) {
                        cw = nw;
                        cc = nc;
                        load_win(ja + 32, nw, nc);
                    }
                    // wait until band b-1 has published the whole window
                    while (__any_sync(kFullMask, (cw & 0xffu) != prev_tag))
                        if ((cw & 0xffu) != prev_tag) cw = ld_relaxed(above + ja + lane);
                }
                const int la = int(ja & 31);
                const uint32_t wa = __shfl_sync(kFullMask, cw, la);
                const uint32_t ca = __shfl_sync(kFullMask, cc, la);
                const uint32_t wb = __shfl_sync(kFullMask, cw, la + 1);
                const uint32_t cb = __shfl_sync(kFullMask, cc, la + 1);
                upA = (first || ja >= n) ? 0 : int32_t(wa >> 8);
                yA = ca;
                upB = (first || ja + 1 >= n) ? 0 : int32_t(wb >> 8);
                yB = cb;
            },
            [&](int64_t j, int32_t val) {
                if (!last) st_relaxed(below + j, (uint32_t(val) << 8) | my_tag);
            },
            m - 1);
        if (last && lane == 0) *d.out = uint32_t(v);
    }
}

}  // namespace

size_t wave_batch_smem() { return size_t(kWaveWarps) * (kWaveMaxCols * 5 + kWaveTab); }

cudaError_t wave_batch_launch(const WaveBatchDev& d, int sms, cudaStream_t stream) {
    const int smem = int(wave_batch_smem());
    cudaError_t e = cudaFuncSetAttribute(wave_batch_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave_batch_kernel, 32 * kWaveWarps,
                                                      smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    int64_t grid = int64_t(sms) * occ;
    const int64_t need = (int64_t(d.pairs) + kWaveWarps - 1) / kWaveWarps;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    wave_batch_kernel<<<int(grid), 32 * kWaveWarps, smem, stream>>>(d);
    return cudaGetLastError();
}

int64_t wave_pair_bands(int64_t m) { return (m + kWaveBand - 1) / kWaveBand; }

cudaError_t wave_pair_launch(const WavePairDev& d, int sms, cudaStream_t stream) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave_pair_kernel, 32, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    int64_t grid = int64_t(sms) * (occ < 8 ? occ : 8);
    const int64_t bands = wave_pair_bands(d.m);
    if (grid > bands) grid = bands;
    wave_pair_kernel<<<int(grid), 32, 0, stream>>>(d);
    return cudaGetLastError();
}

}  // namespace wlcs
