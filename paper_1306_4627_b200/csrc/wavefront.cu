// wavefront.cu -- the cell-wavefront fill variant (WLCS_VARIANT_WAVEFRONT).
//
// Same integer result as the bit-parallel variant and as the reference's
// cell recurrence (proj/src/serial.cpp:16-30, cell.hpp:20-38):
//   c[i][j] = x_i == y_j ? c[i-1][j-1] + 1 : max(c[i-1][j], c[i][j-1])
//
// Cells are packed two per 32-bit register (16x2) and updated with the DPX
// SIMD three-way max, three ALU instructions per PAIR of cells:
//   d = x ^ y                        (LOP3; per half 0 iff the codes match)
//   t = diag + 0x00010001 - d        (IADD3; per half diag + 1 - d)
//   c = vimax3_u16x2(up, left, t)    (VIMNMX3.U16x2)
// On a match t = diag + 1, the reference's value; on a mismatch t <= diag,
// and diag <= max(up, left) always, so t never wins.  The halves never borrow
// from each other because every stored value is >= kOff > max d, and never
// overflow because values are stored tile-relative (below).
//
// Tiling: a warp sweeps a band of 64 R rows as 64 "virtual lanes" of R
// consecutive rows: lane l holds virtual lane l in the low halves of its
// registers and virtual lane l + 32 in the high halves.  At step t lane l
// works on column t - l (low) and t - l - 32 (high), so both halves are
// independent cells -- an anti-diagonal wavefront 64 deep.  The bottom value
// and the column code of each virtual lane travel to the next one in two
// __shfl_sync per step; lane 0's high half takes lane 31's low half, lane 0's
// low half takes the band's top boundary.  Columns before a virtual lane's
// start carry a sentinel code that never matches, so no cell needs masking;
// after the last column the state provably stops changing.
//
// Tile-relative values: stored = c - G with a warp-uniform base G (32-bit,
// absolute values only on band borders).  The values one warp holds at a step
// span at most ~64 R + 64, so the pair kernel re-bases every 8192 steps
// (G += the warp's minimum - kOff) and the 16-bit halves never overflow.
//
//  * batch kernel: one warp per pair (columns = the shorter string <=
//    kWaveMaxCols, in the warp's shared memory with the boundary row between
//    bands); R chosen per pair so that the bands cover the rows tightly;
//  * pair kernel: bands of one pair run concurrently on many warps; band b
//    publishes its bottom row as self-validating words (value << 8 | tag)
//    into a ring of boundary rows, band b+1 reads them in windows of 32
//    columns, one window ahead (same hand-off scheme as the strip kernel).
#include "wlcs_common.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr uint32_t kOff = 1024;           // stored value of c = 0 at the start
constexpr uint32_t kOff2 = kOff * 0x10001u;
constexpr uint32_t kSentinel = 0x100u;    // column code of no column
constexpr uint32_t kNoRow = 0x1ffu;       // row code past the last row
constexpr int kWaveWarps = 4;             // warps per CTA (batch kernel)
constexpr int kRebaseMask = 8191;
// Build-time switches; the defaults are the measured best, the others are kept
// so that the A/B rows of DESIGN.md section 4 can be re-run (tools/exp_build.sh)
#ifndef WLCS_WAVE_SLEEP_NS
#define WLCS_WAVE_SLEEP_NS 200
#endif
#ifndef WLCS_WAVE_PF_STEP
#define WLCS_WAVE_PF_STEP 24
#endif
#ifndef WLCS_WAVE_MAX2
#define WLCS_WAVE_MAX2 0
#endif
#ifndef WLCS_WAVE_PAIR_WARPS
#define WLCS_WAVE_PAIR_WARPS 4
#endif

// One packed cell pair.  WLCS_WAVE_MAX2: the three-way max as two two-way
// VIMNMX.16x2, which also issue on the FMA pipe (the ALU pipe keeps LOP3 and
// IADD3); otherwise one VIMNMX3.U16x2 (ALU pipe only).  The second max is the
// signed form so that ptxas does not fuse the pair back into VIMNMX3 (stored
// values stay below 2^15: kOff + band + re-base period).
__device__ __forceinline__ uint32_t cell2(uint32_t up, uint32_t left, uint32_t diag,
                                          uint32_t x, uint32_t y) {
    const uint32_t tt = diag + 0x10001u - (x ^ y);
#if WLCS_WAVE_MAX2
    const uint32_t q = __vmaxu2(left, tt);
    uint32_t v;
    asm("max.s16x2 %0, %1, %2;" : "=r"(v) : "r"(q), "r"(up));
    return v;
#else
    return __vimax3_u16x2(up, left, tt);
#endif
}

// Steps of one band, in windows of 32 steps.  Win(t0, G) is called by the
// whole warp at the start of every window (the provider's hand-off waits and
// conversions), Mid(t0) WLCS_WAVE_PF_STEP steps into it (the next window's
// loads: late enough that the band above has usually written them, early
// enough to land before they are needed); Prov(t) then returns, for lane 0 at step t, the
// packed word (stored top boundary << 16) | code: the top boundary c[i0-1][t]
// as c - G and the code of column t (kSentinel for t >= n, with a stored top
// value in [kOff / 2, the last real one]).  Bottom(t, u, G) is called by
// every lane at every step with its packed values u; lane 31's high half is
// c[i0 + 64R - 1][t - 63] - G (meaningful for 0 <= t - 63 < n); the callee
// stores it without a divergent branch (a branch around the store would put
// the next step's shuffles on their slow path).  G changes only between
// windows.  Returns, in every lane, the final value of row want_row (0 if not
// in this band).
template <int R, bool REBASE, typename Win, typename Mid, typename Prov, typename BottomFn>
__device__ __forceinline__ int32_t sweep_band(const uint8_t* rowp, int64_t i0, int64_t m,
                                              int64_t n, Win win, Mid mid, Prov prov,
                                              BottomFn bottom, int64_t want_row) {
    const int lane = int(lane_id());
    uint32_t xr[R];    // row codes: low half virtual lane `lane`, high half lane + 32
    uint32_t left[R];  // current column's values of the R rows (both halves)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t ilo = i0 + int64_t(lane) * R + r, ihi = ilo + 32 * R;
        const uint32_t lo = ilo < m ? uint32_t(rowp[ilo]) : kNoRow;
        const uint32_t hi = ihi < m ? uint32_t(rowp[ihi]) : kNoRow;
        xr[r] = lo | (hi << 16);
        left[r] = kOff2;
    }
    int32_t G = -int32_t(kOff);  // c = stored + G
    uint32_t prev_in = kOff2;     // up value of the previous column = diag of row 0
    uint32_t send_v = kOff2, send_y = kSentinel * 0x10001u;
    const int src = (lane + 31) & 31;
    const int T = int(n) + 63;  // n < 2^24
    auto step = [&](int t) {
        const uint32_t rv = __shfl_sync(kFullMask, send_v, src);
        const uint32_t ry = __shfl_sync(kFullMask, send_y, src);
        const uint32_t pw = prov(t);
        const uint32_t in_v = lane == 0 ? __byte_perm(pw, rv, 0x5432) : rv;
        const uint32_t in_y = lane == 0 ? __byte_perm(pw, ry, 0x5410) : ry;
        uint32_t u = in_v, dg = prev_in;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t v = cell2(u, left[r], dg, xr[r], in_y);
            dg = left[r];
            left[r] = v;
            u = v;
        }
        prev_in = in_v;
        send_v = u;
        send_y = in_y;
        bottom(t, u, G);
    };
    if constexpr (!REBASE) {  // no windows (batch: Win is empty, G constant)
        for (int t = 0; t < T; ++t) step(t);
    } else {
        for (int t0 = 0; t0 < T; t0 += 32) {
            win(t0, G);
            const int t1 = min(t0 + 32, T), tm = min(t0 + WLCS_WAVE_PF_STEP, t1);
            for (int t = t0; t < tm; ++t) step(t);
            mid(t0);
            for (int t = tm; t < t1; ++t) step(t);
            if (((t0 + 32) & kRebaseMask) == 0 && t0 + 32 <= int(n)) {
                // row 0 of a virtual lane is its smallest value; the in-flight
                // values (diag, sends, lane 0's top) are at most 2 below it.  Not
                // in the last window: lane 0's past-the-end top values are a
                // constant kOff / 2 that a re-base would wrap.
                const uint32_t lmin = min(left[0] & 0xffffu, left[0] >> 16);
                const uint32_t wmin = __reduce_min_sync(kFullMask, lmin);
                if (wmin > 2 * kOff) {
                    const uint32_t delta = wmin - kOff;
                    const uint32_t d2 = delta * 0x10001u;
#pragma unroll
                    for (int r = 0; r < R; ++r) left[r] -= d2;
                    prev_in -= d2;
                    send_v -= d2;
                    G += int32_t(delta);
                }
            }
        }
    }
    int32_t res = 0;
    const int64_t k = want_row - i0;
    if (k >= 0 && k < 64 * R) {
        const int vl = int(k / R), rr = int(k % R);
        uint32_t mine = left[0];
#pragma unroll
        for (int r = 1; r < R; ++r)
            if (r == rr) mine = left[r];
        const uint32_t w = __shfl_sync(kFullMask, mine, vl & 31);
        res = int32_t(vl >= 32 ? (w >> 16) : (w & 0xffffu)) + G;
    }
    return res;
}

// Predicated shared store (no branch: see sweep_band).
__device__ __forceinline__ void st_shared_u16_if(bool pred, uint16_t* p, uint32_t v) {
    const uint32_t a = uint32_t(__cvta_generic_to_shared(p));
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
        "@p st.shared.u16 [%1], %2;\n\t}" ::"r"(uint32_t(pred)),
        "r"(a), "h"(uint16_t(v)));
}

// ---------------------------------------------------------------- batch
// Rows per virtual lane for a pair of m rows: the fewest bands of <= 64 * 16
// rows, then the smallest R >= 4 whose bands cover the rows (odd R too unless
// WLCS_WAVE_EVEN_R: at most 63 padding rows per band).
#ifndef WLCS_WAVE_EVEN_R
#define WLCS_WAVE_EVEN_R 0
#endif
__device__ __forceinline__ int batch_rows_per_lane(int64_t m, int64_t& bands) {
    bands = (m + 64 * 16 - 1) / (64 * 16);
    const int64_t per = (m + bands - 1) / bands;
    int R = int((per + 63) / 64);
    if (WLCS_WAVE_EVEN_R) R += R & 1;
    return R < 4 ? 4 : R;
}

// A pair's columns live in the warp's shared memory as packed words
// col[64 + j] = ((c[top][j] - G) << 16) | code(y_j), 64 words of padding on
// both sides (sentinel code, c = 0): lane 0 reads its step's word without
// bounds tests, and lane 31 writes the band's bottom row into the high halves
// (column t - 63 at step t, i.e. word t + 1, already read by this band) for the
// next band -- also without tests, the padding absorbs t - 63 < 0.
template <int R>
__device__ __forceinline__ int32_t batch_pair(const uint8_t* rowp, int64_t m, int64_t n,
                                              uint32_t* col) {
    int32_t res = 0;
    uint16_t* col16 = reinterpret_cast<uint16_t*>(col);
    const bool is31 = lane_id() == 31;
    for (int64_t i0 = 0; i0 < m; i0 += 64 * R) {
        const int32_t v = sweep_band<R, false>(
            rowp, i0, m, n, [](int, int32_t) {}, [](int) {}, [&](int t) { return col[64 + t]; },
            [&](int t, uint32_t u, int32_t) { st_shared_u16_if(is31, col16 + 2 * (t + 1) + 1, u >> 16); },
            m - 1);
        if (i0 + 64 * R >= m) res = v;
        __syncwarp();
    }
    return res;
}

__global__ void __launch_bounds__(32 * kWaveWarps) wave_batch_kernel(WaveBatchDev d) {
    extern __shared__ __align__(16) uint32_t smem_w[];
    const int warp = int(threadIdx.x >> 5);
    const int lane = int(lane_id());
    uint32_t* col = smem_w + warp * (kWaveMaxCols + 128);
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
        for (int k = lane; k < int(n) + 128; k += 32) {
            const int j = k - 64;
            col[k] = (kOff << 16) | ((j >= 0 && j < n) ? uint32_t(colp[j]) : kSentinel);
        }
        __syncwarp();
        int64_t bands;
        const int R = batch_rows_per_lane(m, bands);
        int32_t res;
        switch (R) {
            case 4: res = batch_pair<4>(rowp, m, n, col); break;
            case 5: res = batch_pair<5>(rowp, m, n, col); break;
            case 6: res = batch_pair<6>(rowp, m, n, col); break;
            case 7: res = batch_pair<7>(rowp, m, n, col); break;
            case 8: res = batch_pair<8>(rowp, m, n, col); break;
            case 9: res = batch_pair<9>(rowp, m, n, col); break;
            case 10: res = batch_pair<10>(rowp, m, n, col); break;
            case 11: res = batch_pair<11>(rowp, m, n, col); break;
            case 12: res = batch_pair<12>(rowp, m, n, col); break;
            case 13: res = batch_pair<13>(rowp, m, n, col); break;
            case 14: res = batch_pair<14>(rowp, m, n, col); break;
            case 15: res = batch_pair<15>(rowp, m, n, col); break;
            default: res = batch_pair<16>(rowp, m, n, col); break;
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
__device__ __forceinline__ void st_relaxed_if(bool pred, uint32_t* p, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
        "@p st.relaxed.gpu.global.u32 [%1], %2;\n\t}" ::"r"(uint32_t(pred)),
        "l"(p), "r"(v)
        : "memory");
}

template <int R>
__global__ void __launch_bounds__(32 * WLCS_WAVE_PAIR_WARPS) wave_pair_kernel(WavePairDev d) {
    const int lane = int(lane_id());
    const int64_t n = d.n, m = d.m;
    constexpr int kBand = 64 * R;
    const uint32_t nbands = uint32_t((m + kBand - 1) / kBand);
    for (;;) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(d.ticket, 1u);
        b = __shfl_sync(kFullMask, b, 0);
        if (b >= nbands) break;
        const int64_t i0 = int64_t(b) * kBand;
        const bool first = b == 0, last = b + 1 == nbands;
        // ring of nbuf boundary rows; words are (value << 8) | tag with the
        // writer's generation tag, so stale words of an earlier band are
        // recognised without re-zeroing (a band b+nbuf-1 that reuses band b-1's
        // row writes column j only after band b has read it: band b+k reaches
        // column j no earlier than 64 k steps after band b)
        const uint32_t prev_tag = first ? 0u : ((b - 1) / d.nbuf) % 255u + 1u;
        const uint32_t my_tag = (b / d.nbuf) % 255u + 1u;
        const uint32_t* above = d.bnd + int64_t(first ? 0 : (b - 1) % d.nbuf) * d.bstride;
        uint32_t* below = d.bnd + int64_t(b % d.nbuf) * d.bstride;
        // windows of 32 columns: lane k loads column base + k (boundary word
        // and column byte) of the next window during the current one; at a
        // window's start they become lane 0's packed provider words for its
        // 32 steps
        auto load_win = [&](int64_t base, uint32_t& w, uint32_t& c) {
            const int64_t jj = base + lane;
            w = (!first && jj < n) ? ld_relaxed(above + jj) : prev_tag;
            c = jj < n ? uint32_t(d.colp[jj]) : kSentinel;
        };
        uint32_t nw, nc, pwin = 0;
        bool failed = false;  // warp-uniform: set by the watchdog
        load_win(0, nw, nc);
        const int ni = int(n);
        const int32_t v = sweep_band<R, true>(
            d.rowp, i0, m, n,
            [&](int t0, int32_t G) {
                if (t0 >= ni) {
                    pwin = ((kOff / 2) << 16) | kSentinel;
                    return;
                }
                uint32_t cw = nw;
                const uint32_t cc = nc;
                // wait until band b-1 has published the whole window; a
                // waiting warp sleeps between polls so that it does not take
                // issue slots from the warps that compute
                uint32_t spins = 0;
                while (__any_sync(kFullMask, (cw & 0xffu) != prev_tag)) {
                    __nanosleep(WLCS_WAVE_SLEEP_NS);
                    if ((cw & 0xffu) != prev_tag) cw = ld_relaxed(above + t0 + lane);
                    if (++spins > (1u << 24)) {  // watchdog (~1 min): fail, do not hang
                        if (lane == 0) atomicOr(d.error, 1u);
                        failed = true;
                        break;
                    }
                }
                const int32_t top = first ? 0 : int32_t(cw >> 8);
                pwin = t0 + lane < ni ? (uint32_t(top - G) << 16) | cc
                                      : ((kOff / 2) << 16) | kSentinel;
            },
            [&](int t0) {
                if (t0 + 32 < ni) load_win(t0 + 32, nw, nc);
            },
            [&](int t) { return __shfl_sync(kFullMask, pwin, t & 31); },
            [&](int t, uint32_t u, int32_t G) {
                const int jb = t - 63;
                st_relaxed_if(lane == 31 && !last && jb >= 0, below + jb,
                              (uint32_t(int32_t(u >> 16) + G) << 8) | my_tag);
            },
            m - 1);
        if (failed) return;  // the error word is set; the host reports it
        if (last && lane == 0) *d.out = uint32_t(v);
    }
}

}  // namespace

size_t wave_batch_smem() { return size_t(kWaveWarps) * (kWaveMaxCols + 128) * 4; }

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

// Rows per virtual lane: the tallest bands (least hand-off and pipeline
// fill) that still give every SM about 12 resident warps.
int wave_pair_rows(int64_t m, int sms) {
    for (int R : {16, 8})
        if ((m + 64 * R - 1) / (64 * R) >= int64_t(sms) * 12) return R;
    return 4;
}

int64_t wave_pair_bands(int64_t m, int R) { return (m + 64 * R - 1) / (64 * R); }

template <int R>
cudaError_t wave_pair_launch_r(const WavePairDev& d, int sms, cudaStream_t stream) {
    // CTAs of WLCS_WAVE_PAIR_WARPS one-band warps: a CTA's warps sit on
    // distinct sub-partitions, so bands spread evenly over them
    constexpr int W = WLCS_WAVE_PAIR_WARPS;
    int occ = 0;
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave_pair_kernel<R>, 32 * W, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    int64_t grid = int64_t(sms) * (occ * W < 16 ? occ : 16 / W);
    const int64_t bands = wave_pair_bands(d.m, R);
    const int64_t need = (bands + W - 1) / W;
    if (grid > need) grid = need;
    wave_pair_kernel<R><<<int(grid), 32 * W, 0, stream>>>(d);
    return cudaGetLastError();
}

cudaError_t wave_pair_launch(const WavePairDev& d, int sms, cudaStream_t stream) {
    switch (d.R) {
        case 16: return wave_pair_launch_r<16>(d, sms, stream);
        case 8: return wave_pair_launch_r<8>(d, sms, stream);
        case 4: return wave_pair_launch_r<4>(d, sms, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace wlcs
