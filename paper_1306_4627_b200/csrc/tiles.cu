// tiles.cu -- the reference's block-kernel contract on the device.
//
// BlockArgs (proj/include/wavelcs/kernels.hpp:14-33): fill the tile
// [i_first, i_last] x [j_first, j_last] of the caller's DpTable / BacktrackTable
// given its final north row (i_first - 1) and west column (j_first - 1); the
// cells follow lcs_cell (cell.hpp:30-38) exactly, arrows included, as the
// reference's scalar kernel does (kernels_scalar.cpp:5-17).  This is the
// plugin-level entry (compute_block, resolve_kernel(...)(args)); whole-table
// fills never go tile by tile (they expand the bit-parallel rows, bitpar_pair.cu
// tables_kernel).
//
// One CTA sweeps the tile in bands of blockDim.x rows: thread t owns row
// r0 + t and visits column k = s - t at step s (an anti-diagonal wavefront).
// The only value that crosses threads is `up` (thread t-1's cell of the same
// column, one step earlier), passed through a two-slot shared-memory row;
// `diag` is the `up` a thread read one step earlier and `left` its own last
// cell.  The band's top row comes from the north border (band 0) or from the
// previous band's last row in the output.
#include <cstdint>

#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr uint8_t kDiag = 0, kUp = 1, kLeft = 2;  // Arrow (cell.hpp:16-20)

__global__ void __launch_bounds__(1024) tile_fill_kernel(const uint8_t* xs, const uint8_t* ys,
                                                         const uint32_t* north, const uint32_t* west,
                                                         uint32_t* cv, uint8_t* bv, int h, int w) {
    __shared__ uint32_t up_buf[2][1024];
    const int t = threadIdx.x, T = blockDim.x;
    for (int r0 = 0; r0 < h; r0 += T) {
        const int i = r0 + t;  // tile row of this thread (0-based)
        const bool row_ok = i < h;
        const int rows = h - r0 < T ? h - r0 : T;
        const uint8_t xi = row_ok ? xs[i] : 0;
        uint32_t left = row_ok ? west[i] : 0u;
        // diag of column 0: the cell above the west border
        uint32_t diag = (t == 0) ? (r0 == 0 ? north[0] : west[r0 - 1]) : (row_ok ? west[i - 1] : 0u);
        const int steps = rows + w - 1;
        for (int s = 0; s < steps; ++s) {
            const int k = s - t;
            if (row_ok && k >= 0 && k < w) {
                uint32_t up;
                if (t == 0) up = r0 == 0 ? north[k + 1] : cv[size_t(r0 - 1) * w + k];
                else up = up_buf[(s - 1) & 1][t - 1];
                uint32_t v;
                uint8_t a;
                if (xi == ys[k]) {
                    v = diag + 1;
                    a = kDiag;
                } else if (up > left) {
                    v = up;
                    a = kUp;
                } else {
                    v = left;
                    a = kLeft;
                }
                cv[size_t(i) * w + k] = v;
                bv[size_t(i) * w + k] = a;
                up_buf[s & 1][t] = v;
                left = v;
                diag = up;
            }
            __syncthreads();
        }
    }
}

}  // namespace

cudaError_t tile_fill(const uint8_t* d_x, const uint8_t* d_y, const uint32_t* d_north,
                      const uint32_t* d_west, uint32_t* d_cv, uint8_t* d_bv, int h, int w,
                      cudaStream_t stream) {
    if (h <= 0 || w <= 0) return cudaSuccess;
    int threads = ((h + 31) / 32) * 32;
    if (threads > 1024) threads = 1024;
    tile_fill_kernel<<<1, threads, 0, stream>>>(d_x, d_y, d_north, d_west, d_cv, d_bv, h, w);
    return cudaGetLastError();
}

}  // namespace wlcs
