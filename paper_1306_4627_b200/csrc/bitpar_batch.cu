// bitpar_batch.cu -- batched bit-parallel LCS lengths (BASELINE config C2).
//
// Replaces, for many independent pairs at once, the reference's length path
//   lcs_length -> lcs_fill_serial -> fill_block_scalar
//   (proj/src/serial.cpp:11-34, proj/src/kernels_scalar.cpp:5-17)
// and its wavefront-parallel fill (proj/src/parallel.cpp:251-274), which the
// reference can only apply one pair at a time (proj/src/bench.cpp:77-129).
//
// Design (DESIGN.md section "Batch kernel"):
//  * plan:   one thread per pair picks the roles (the shorter string becomes
//            the bit-vector "column" string -- LCS length is symmetric,
//            SPEC.md:82), its word count W = ceil(cols/32) and a lane shape
//            (S lanes per pair, K <= 8 words per lane, S*K >= W); a radix sort
//            groups pairs by shape and orders them by decreasing row count.
//  * main:   persistent 1-warp CTAs pull tasks (32/S pairs of one shape) from
//            an atomic counter.  Per task the warp builds, in shared memory, a
//            byte->code map of the task's column alphabet and the match masks
//            PM[code][word] (layout [code][word/4][lane][4] so that every
//            LDS.128 of a warp is bank-conflict free), then streams the row
//            strings 16 rows (one aligned 16-byte chunk) per step.  Each row
//            costs AND + IADD3.X + LOP3 per 32 cells (rowstep.cuh).  With S>1
//            the S lanes of a pair form a skewed pipeline: lane s works on
//            chunk t-s and receives the 16 per-row carries of lane s-1 as one
//            16-bit mask through __shfl_up_sync.
//  * result: LCS = zero bits of V below column `cols`, reduced over the
//            pair's S lanes.
#include <cub/device/device_radix_sort.cuh>

#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kMaxK = 8;
constexpr int kNumClasses = 6 * kMaxK;        // S in {1,2,4,8,16,32} x K in 1..8
constexpr int kMapBytes = 256;
constexpr uint32_t kNoKey = 0xffffffffu;

// meta[] layout (uint32): per-order counts, pair starts, task starts (+total),
// then the task counter and the overflow count.
constexpr int kMetaCount = 0;
constexpr int kMetaPairStart = kNumClasses;
constexpr int kMetaTaskStart = 2 * kNumClasses;          // kNumClasses + 1 entries
constexpr int kMetaCounter = 3 * kNumClasses + 1;
constexpr int kMetaOverflow = 3 * kNumClasses + 2;

__device__ __forceinline__ int class_of(int sidx, int k) { return sidx * kMaxK + (k - 1); }

__global__ void batch_plan_kernel(BatchDev d) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= d.pairs) return;
    const uint64_t m = d.xoff[p + 1] - d.xoff[p];
    const uint64_t n = d.yoff[p + 1] - d.yoff[p];
    const uint64_t cols = m < n ? m : n;
    const uint64_t rows = m < n ? n : m;
    uint32_t key = kNoKey;
    if (cols == 0) {
        d.out[p] = 0;  // empty input: length 0 (proj/tests/test_parallel.cpp:236-242)
    } else {
        const uint64_t w = (cols + 31) / 32;
        if (w > uint64_t(32 * kMaxK)) {
            // Longer than one warp can hold: routed to the single-pair strip kernel.
            const uint32_t i = atomicAdd(d.meta + kMetaOverflow, 1u);
            d.overflow[i] = p;
        } else {
            int sidx = 0;
            while ((uint64_t(kMaxK) << sidx) < w) ++sidx;
            const int s = 1 << sidx;
            const int k = int((w + s - 1) / s);
            const int order = kNumClasses - 1 - class_of(sidx, k);
            const uint32_t r = rows > 0xffffffull ? 0xffffffu : uint32_t(rows);
            key = (uint32_t(order) << 24) | (0xffffffu - r);
            atomicAdd(d.meta + kMetaCount + order, 1u);
        }
    }
    d.keys_in[p] = key;
    d.vals_in[p] = p;
}

__global__ void batch_tasks_kernel(BatchDev d) {
    if (threadIdx.x != 0) return;
    uint32_t ps = 0, ts = 0;
    for (int o = 0; o < kNumClasses; ++o) {
        const int c = kNumClasses - 1 - o;
        const uint32_t per_task = 32u >> (c / kMaxK);
        const uint32_t cnt = d.meta[kMetaCount + o];
        d.meta[kMetaPairStart + o] = ps;
        d.meta[kMetaTaskStart + o] = ts;
        ps += cnt;
        ts += (cnt + per_task - 1) / per_task;
    }
    d.meta[kMetaTaskStart + kNumClasses] = ts;
}

// One warp task: pairs [first, last) of the sorted order, all of shape (S, K).
template <int S, int K>
__device__ __noinline__ void run_task(const BatchDev& d, uint32_t first, uint32_t last,
                                      uint8_t* smem) {
    const uint32_t lane = lane_id();
    const int seg = int(lane) / S;
    const int s = int(lane) % S;
    const uint32_t idx = first + uint32_t(seg);
    const bool active = idx < last;
    const uint32_t pair = active ? d.vals[idx] : 0u;

    // Roles: the shorter string is the column (bit-vector) string.
    const uint8_t* colp = d.xs;
    const uint8_t* rowp = d.xs;
    const uint8_t *col_lo = d.xs, *col_hi = d.xs, *row_lo = d.xs, *row_hi = d.xs;
    int64_t cols = 0, rows = 0;
    if (active) {
        const uint64_t xo = d.xoff[pair], yo = d.yoff[pair];
        const int64_t m = int64_t(d.xoff[pair + 1] - xo);
        const int64_t n = int64_t(d.yoff[pair + 1] - yo);
        if (n <= m) {
            colp = d.ys + yo; cols = n; col_lo = d.ys; col_hi = d.ys + d.ys_bytes;
            rowp = d.xs + xo; rows = m; row_lo = d.xs; row_hi = d.xs + d.xs_bytes;
        } else {
            colp = d.xs + xo; cols = m; col_lo = d.xs; col_hi = d.xs + d.xs_bytes;
            rowp = d.ys + yo; rows = n; row_lo = d.ys; row_hi = d.ys + d.ys_bytes;
        }
    }

    uint8_t* map = smem;
    uint8_t* pm = smem + kMapBytes;

    __syncwarp();
    reinterpret_cast<uint2*>(map)[lane] = make_uint2(0u, 0u);
    __syncwarp();

    // ---- column alphabet of this task -> dense codes 1..sigma-1 (0 = no match)
    const int64_t c0 = int64_t(32 * K) * s;
    int64_t c1 = c0 + 32 * K;
    if (c1 > cols) c1 = cols;
    const int64_t clen = c1 > c0 ? c1 - c0 : 0;
    const uint8_t* cbase = colp + c0;
    const int a_c = int(reinterpret_cast<uintptr_t>(cbase) & 15u);
    const uint8_t* cstart = cbase - a_c;
    const int nch = clen > 0 ? int((a_c + clen + 15) / 16) : 0;
    const int nch_max = warp_max(nch);
    for (int ch = 0; ch < nch_max; ++ch) {
        if (ch < nch) {
            const uint4 c = load_chunk16(cstart + 16 * ch, col_lo, col_hi);
            const uint32_t vm = chunk_valid_mask(int64_t(ch) * 16 - a_c, clen);
#pragma unroll
            for (int r = 0; r < 16; ++r)
                if ((vm >> r) & 1u) map[chunk_byte(c, r)] = 1;
        }
    }
    __syncwarp();
    {
        const uint2 f = reinterpret_cast<const uint2*>(map)[lane];
        uint32_t cnt = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) cnt += ((f.x >> (8 * b)) & 0xffu) ? 1u : 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b) cnt += ((f.y >> (8 * b)) & 0xffu) ? 1u : 0u;
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
            if (int(lane) >= o) incl += v;
        }
        uint32_t code = incl - cnt + 1;
        uint32_t ox = 0, oy = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((f.x >> (8 * b)) & 0xffu) ox |= (code++) << (8 * b);
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((f.y >> (8 * b)) & 0xffu) oy |= (code++) << (8 * b);
        const uint32_t sigma = __shfl_sync(kFullMask, incl, 31) + 1;  // + the zero row
        if (sigma > 256u || sigma * PmLayout<K>::code_stride > uint32_t(d.pm_bytes)) {
            // Alphabet too large for this warp's shared-memory slice.
            if (active && s == 0) {
                const uint32_t i = atomicAdd(d.meta + kMetaOverflow, 1u);
                d.overflow[i] = pair;
            }
            return;
        }
        reinterpret_cast<uint2*>(map)[lane] = make_uint2(ox, oy);
        uint4* pm4 = reinterpret_cast<uint4*>(pm);
        for (uint32_t i = lane; i < sigma * (PmLayout<K>::code_stride / 16); i += 32)
            pm4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // ---- match masks: bit (j - c0) of the lane's K words for every column j.
    for (int ch = 0; ch < nch_max; ++ch) {
        if (ch < nch) {
            const uint4 c = load_chunk16(cstart + 16 * ch, col_lo, col_hi);
            const int jr0 = ch * 16 - a_c;
            const uint32_t vm = chunk_valid_mask(jr0, clen);
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if ((vm >> r) & 1u) {
                    const int jr = jr0 + r;
                    const int w = jr >> 5;
                    const uint32_t code = map[chunk_byte(c, r)];
                    uint32_t* wp = reinterpret_cast<uint32_t*>(
                        pm + code * PmLayout<K>::code_stride + PmLayout<K>::word_offset(lane, w));
                    *wp |= 1u << (jr & 31);
                }
            }
        }
    }
    __syncwarp();

    // ---- row sweep
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int a_r = int(reinterpret_cast<uintptr_t>(rowp) & 15u);
    const uint8_t* rstart = rowp - a_r;
    const int nrch = rows > 0 ? int((rows + a_r + 15) / 16) : 0;
    const int T = warp_max(nrch) + S - 1;
    const uint32_t lane_off = PmLayout<K>::word_offset(lane, 0);
    uint32_t cout = 0;
    for (int t = 0; t < T; ++t) {
        const int ch = t - s;
        const int64_t lo = int64_t(ch) * 16 - a_r;
        const bool full = ch >= 0 && lo >= 0 && lo + 16 <= rows;
        uint32_t cin = 0;
        if constexpr (S > 1) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        const uint32_t vm = ch >= 0 ? chunk_valid_mask(lo, rows) : 0u;
        sweep_chunk<(S > 1), K>(__all_sync(kFullMask, full), V, map, pm, lane_off,
                                rstart + int64_t(ch) * 16, row_lo, row_hi, vm, cin, cout,
                                NoRowHook{});
    }

    // ---- LCS = zero bits of V below `cols`
    int zeros = lane_zero_count<K>(V, int64_t(s) * K, cols);
#pragma unroll
    for (int o = S / 2; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
    if (active && s == 0) d.out[pair] = uint32_t(zeros);
}

#define WLCS_TASK_CASE(SIDX, KK)                                            \
    case SIDX * kMaxK + (KK - 1):                                           \
        run_task<(1 << SIDX), KK>(d, first, last, smem);                    \
        break;

__global__ void __launch_bounds__(32) batch_main_kernel(BatchDev d) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = lane_id();
    const uint32_t* count = d.meta + kMetaCount;
    const uint32_t* pair_start = d.meta + kMetaPairStart;
    const uint32_t* task_start = d.meta + kMetaTaskStart;
    const uint32_t total = task_start[kNumClasses];
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(d.meta + kMetaCounter, 1u);
        t = __shfl_sync(kFullMask, t, 0);
        if (t >= total) break;
        const bool le0 = task_start[lane] <= t;
        const bool le1 = lane + 32 < kNumClasses && task_start[lane + 32] <= t;
        const int order = __popc(__ballot_sync(kFullMask, le0)) +
                          __popc(__ballot_sync(kFullMask, le1)) - 1;
        const int c = kNumClasses - 1 - order;
        const uint32_t per_task = 32u >> (c / kMaxK);
        const uint32_t first = pair_start[order] + (t - task_start[order]) * per_task;
        const uint32_t end = pair_start[order] + count[order];
        const uint32_t last = first + per_task < end ? first + per_task : end;
        switch (c) {
            WLCS_TASK_CASE(0, 1) WLCS_TASK_CASE(0, 2) WLCS_TASK_CASE(0, 3) WLCS_TASK_CASE(0, 4)
            WLCS_TASK_CASE(0, 5) WLCS_TASK_CASE(0, 6) WLCS_TASK_CASE(0, 7) WLCS_TASK_CASE(0, 8)
            WLCS_TASK_CASE(1, 5) WLCS_TASK_CASE(1, 6) WLCS_TASK_CASE(1, 7) WLCS_TASK_CASE(1, 8)
            WLCS_TASK_CASE(2, 5) WLCS_TASK_CASE(2, 6) WLCS_TASK_CASE(2, 7) WLCS_TASK_CASE(2, 8)
            WLCS_TASK_CASE(3, 5) WLCS_TASK_CASE(3, 6) WLCS_TASK_CASE(3, 7) WLCS_TASK_CASE(3, 8)
            WLCS_TASK_CASE(4, 5) WLCS_TASK_CASE(4, 6) WLCS_TASK_CASE(4, 7) WLCS_TASK_CASE(4, 8)
            WLCS_TASK_CASE(5, 5) WLCS_TASK_CASE(5, 6) WLCS_TASK_CASE(5, 7) WLCS_TASK_CASE(5, 8)
            default:
                break;  // unreachable: S >= 2 always has K >= 5
        }
    }
}
#undef WLCS_TASK_CASE

}  // namespace

size_t batch_workspace_bytes(uint32_t pairs, size_t* cub_bytes) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, int(pairs));
    *cub_bytes = (tb + 255) & ~size_t(255);
    const size_t arrays = size_t(pairs) * 4 * 5 + 256 * 4;  // keys/vals x2, overflow, meta
    return *cub_bytes + ((arrays + 255) & ~size_t(255));
}

int batch_smem_per_cta(int pm_bytes) { return kMapBytes + pm_bytes; }

// Launch the whole batch on `stream`.  Device pointers only.  Returns the
// number of pairs routed to the per-pair path in *overflow_count (host value,
// requires one small D2H copy and a stream sync).
cudaError_t batch_launch(BatchDev d, void* workspace, size_t cub_bytes, int sms,
                         cudaStream_t stream) {
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    void* cub_tmp = ws;
    uint32_t* arr = reinterpret_cast<uint32_t*>(ws + cub_bytes);
    d.keys_in = arr;
    d.vals_in = arr + d.pairs;
    d.keys = arr + 2 * size_t(d.pairs);
    d.vals = arr + 3 * size_t(d.pairs);
    d.overflow = arr + 4 * size_t(d.pairs);
    d.meta = arr + 5 * size_t(d.pairs);
    cudaError_t e = cudaMemsetAsync(d.meta, 0, 256 * sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    if (d.pairs == 0) return cudaSuccess;
    batch_plan_kernel<<<(d.pairs + 255) / 256, 256, 0, stream>>>(d);
    size_t tb = cub_bytes;
    e = cub::DeviceRadixSort::SortPairs(cub_tmp, tb, d.keys_in, d.keys, d.vals_in, d.vals,
                                        int(d.pairs), 0, 32, stream);
    if (e != cudaSuccess) return e;
    batch_tasks_kernel<<<1, 32, 0, stream>>>(d);
    const int smem = batch_smem_per_cta(d.pm_bytes);
    e = cudaFuncSetAttribute(batch_main_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, batch_main_kernel, 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    batch_main_kernel<<<sms * occ, 32, smem, stream>>>(d);
    return cudaGetLastError();
}

uint32_t* batch_overflow_count_ptr(void* workspace, size_t cub_bytes, uint32_t pairs) {
    uint32_t* arr = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + cub_bytes);
    return arr + 5 * size_t(pairs) + kMetaOverflow;
}

uint32_t* batch_overflow_list_ptr(void* workspace, size_t cub_bytes, uint32_t pairs) {
    uint32_t* arr = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + cub_bytes);
    return arr + 4 * size_t(pairs);
}

}  // namespace wlcs
