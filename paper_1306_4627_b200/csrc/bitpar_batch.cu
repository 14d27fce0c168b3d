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
//            (S lanes per pair, K <= 8 words per lane, S*K >= W).  A counting
//            sort (plan -> scan -> scatter) groups pairs by shape and, inside
//            a shape, by decreasing 16-row chunk count, so the pairs of one
//            warp task end on the same step.
//  * main:   persistent 1-warp CTAs pull tasks (32/S pairs of one shape) from
//            an atomic counter.  Per task the warp builds, in shared memory, a
//            byte->code map of the task's column alphabet and the match masks
//            PM[code][word] (sweep.cuh layouts: every warp-wide PM load is
//            bank-conflict free), then streams the row strings one aligned
//            16-byte chunk (16 rows) per step, prefetching the next chunk.
//            Each row costs AND + IADD3.X + LOP3 per 32 cells (rowstep.cuh).
//            With S>1 the S lanes of a pair form a skewed pipeline: lane s
//            works on chunk t-s and receives the 16 per-row carries of lane
//            s-1 as one 16-bit mask through __shfl_up_sync.
//  * result: LCS = zero bits of V below column `cols`, reduced over the
//            pair's S lanes.
#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kMaxK = 8;
constexpr int kNumClasses = 6 * kMaxK;   // S in {1,2,4,8,16,32} x K in 1..8
constexpr int kChunkBuckets = 128;       // chunk-count buckets per class (clamped)
constexpr int kBuckets = kNumClasses * kChunkBuckets;
constexpr int kMapBytes = 256;
constexpr uint32_t kNoBucket = 0xffffffffu;

// meta[] layout (uint32)
constexpr int kMetaCount = 0;                            // per order
constexpr int kMetaPairStart = kNumClasses;              // per order
constexpr int kMetaTaskStart = 2 * kNumClasses;          // per order, + total
constexpr int kMetaCounter = 3 * kNumClasses + 1;
constexpr int kMetaOverflow = 3 * kNumClasses + 2;
constexpr int kMetaSafe16 = 240;                          // 16 zero bytes (fetch_chunk)
constexpr int kMetaWords = 256;
// workspace (uint32): meta[256] | hist[kBuckets] | cursor[kBuckets] |
//                     bucket[pairs] | vals[pairs] | overflow[pairs]
constexpr size_t kWsHist = kMetaWords;
constexpr size_t kWsCursor = kWsHist + kBuckets;
constexpr size_t kWsPairs = kWsCursor + kBuckets;

__device__ __forceinline__ int class_of(int sidx, int k) { return sidx * kMaxK + (k - 1); }

__global__ void __launch_bounds__(256) batch_plan_kernel(BatchDev d, uint32_t* hist,
                                                         uint32_t* bucket) {
    __shared__ uint32_t local[kBuckets];
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) local[i] = 0;
    __syncthreads();
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < d.pairs) {
        const uint64_t m = d.xoff[p + 1] - d.xoff[p];
        const uint64_t n = d.yoff[p + 1] - d.yoff[p];
        const uint64_t cols = m < n ? m : n;
        const uint64_t rows = m < n ? n : m;
        uint32_t b = kNoBucket;
        if (cols == 0) {
            d.out[p] = 0;  // empty input: length 0 (proj/tests/test_parallel.cpp:236-242)
        } else {
            const uint64_t w = (cols + 31) / 32;
            if (w > uint64_t(32 * kMaxK)) {
                // Wider than one warp can hold: routed to the single-pair strip kernel.
                const uint32_t i = atomicAdd(d.meta + kMetaOverflow, 1u);
                d.overflow[i] = p;
            } else {
                int sidx = 0;
                while ((uint64_t(kMaxK) << sidx) < w) ++sidx;
                const int s = 1 << sidx;
                const int k = int((w + s - 1) / s);
                const int order = kNumClasses - 1 - class_of(sidx, k);
                uint64_t nch = (rows + 15) / 16;
                if (nch > kChunkBuckets - 1) nch = kChunkBuckets - 1;
                b = uint32_t(order * kChunkBuckets + (kChunkBuckets - 1 - int(nch)));
                atomicAdd(&local[b], 1u);
            }
        }
        bucket[p] = b;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
        if (local[i]) atomicAdd(hist + i, local[i]);
}

// One CTA: exclusive scan of the bucket histogram -> cursors, per-class pair
// ranges and the task table.
__global__ void __launch_bounds__(1024) batch_scan_kernel(BatchDev d, const uint32_t* hist,
                                                          uint32_t* cursor) {
    constexpr int kPer = kBuckets / 1024;  // 6
    __shared__ uint32_t warp_sums[32];
    const int tid = threadIdx.x;
    uint32_t v[kPer];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        v[i] = hist[tid * kPer + i];
        sum += v[i];
    }
    uint32_t incl = sum;
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t ws = warp_sums[lane];
        uint32_t wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFullMask, wi, o);
            if (lane >= o) wi += t;
        }
        warp_sums[lane] = wi - ws;
    }
    __syncthreads();
    uint32_t run = warp_sums[warp] + incl - sum;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        cursor[tid * kPer + i] = run;
        run += v[i];
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t ts = 0;
        for (int o = 0; o < kNumClasses; ++o) {
            const int c = kNumClasses - 1 - o;
            const uint32_t per_task = 32u >> (c / kMaxK);
            const uint32_t start = cursor[o * kChunkBuckets];
            const uint32_t end = o + 1 < kNumClasses ? cursor[(o + 1) * kChunkBuckets]
                                                     : cursor[kBuckets - 1] + hist[kBuckets - 1];
            d.meta[kMetaCount + o] = end - start;
            d.meta[kMetaPairStart + o] = start;
            d.meta[kMetaTaskStart + o] = ts;
            ts += (end - start + per_task - 1) / per_task;
        }
        d.meta[kMetaTaskStart + kNumClasses] = ts;
    }
}

__global__ void __launch_bounds__(256) batch_scatter_kernel(BatchDev d, const uint32_t* bucket,
                                                            uint32_t* cursor) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= d.pairs) return;
    const uint32_t b = bucket[p];
    if (b == kNoBucket) return;
    d.vals[atomicAdd(cursor + b, 1u)] = p;
}

// Per-lane view of its pair inside a task.
struct LanePair {
    const uint8_t* colp;  // column (bit-vector) string = the shorter one
    const uint8_t* rowp;
    const uint8_t *col_lo, *col_hi, *row_lo, *row_hi;
    int cols;             // <= 8192 in the batch path
    int64_t rows;
};

__device__ __forceinline__ LanePair lane_pair(const BatchDev& d, bool active, uint32_t pair) {
    LanePair p{d.xs, d.xs, d.xs, d.xs, d.xs, d.xs, 0, 0};
    if (active) {
        const uint64_t xo = d.xoff[pair], yo = d.yoff[pair];
        const int64_t m = int64_t(d.xoff[pair + 1] - xo);
        const int64_t n = int64_t(d.yoff[pair + 1] - yo);
        if (n <= m) {
            p.colp = d.ys + yo; p.cols = int(n); p.col_lo = d.ys; p.col_hi = d.ys + d.ys_bytes;
            p.rowp = d.xs + xo; p.rows = m; p.row_lo = d.xs; p.row_hi = d.xs + d.xs_bytes;
        } else {
            p.colp = d.xs + xo; p.cols = int(m); p.col_lo = d.xs; p.col_hi = d.xs + d.xs_bytes;
            p.rowp = d.ys + yo; p.rows = n; p.row_lo = d.ys; p.row_hi = d.ys + d.ys_bytes;
        }
    }
    return p;
}

// Builds the task's byte -> code map and match masks in shared memory.  K is
// a runtime value here (one copy of this code for every lane shape).
// Returns sigma (codes incl. the zero row) or 0 when the task's alphabet does
// not fit the warp's shared-memory slice; *zrep receives a byte value absent
// from the alphabet, replicated x4 (used to blank invalid rows).
__device__ __forceinline__ uint32_t build_task(const BatchDev& d, const LanePair& p, int K, int s,
                                            uint8_t* smem, uint32_t* zrep) {
    const uint32_t lane = lane_id();
    uint8_t* map = smem;
    uint8_t* pm = smem + kMapBytes;
    const bool wide = K > 4;
    const uint32_t cs = wide ? 1024u : 128u * uint32_t(K == 3 ? 4 : K);
    const uint32_t ls = wide ? 16u : 4u * uint32_t(K == 3 ? 4 : K);

    __syncwarp();
    reinterpret_cast<uint2*>(map)[lane] = make_uint2(0u, 0u);
    __syncwarp();

    // The lane's columns: [c0, c0 + clen) of its pair's column string, read in
    // 16-byte aligned chunks.
    const int c0 = 32 * K * s;
    const int clen = max(min(c0 + 32 * K, p.cols) - c0, 0);
    const uint8_t* cbase = p.colp + c0;
    const int a_c = int(reinterpret_cast<uintptr_t>(cbase) & 15u);
    const uint8_t* cstart = cbase - a_c;
    const int nch = clen > 0 ? (a_c + clen + 15) >> 4 : 0;
    const int nch_max = warp_max(nch);
    for (int ch = 0; ch < nch_max; ++ch) {
        const uint32_t vm = ch < nch ? valid_mask16(ch * 16 - a_c, clen) : 0u;
        const uint4 c = fetch_chunk(cstart, ch, vm, p.col_lo, p.col_hi, d.safe16);
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if ((vm >> r) & 1u) map[chunk_byte(c, r)] = 1;
    }
    __syncwarp();
    uint32_t sigma;
    {
        const uint2 f = reinterpret_cast<const uint2*>(map)[lane];
        uint32_t present = 0;  // bit b: byte 8*lane + b present
#pragma unroll
        for (int b = 0; b < 4; ++b) present |= (((f.x >> (8 * b)) & 0xffu) ? 1u : 0u) << b;
#pragma unroll
        for (int b = 0; b < 4; ++b) present |= (((f.y >> (8 * b)) & 0xffu) ? 1u : 0u) << (b + 4);
        const uint32_t cnt = __popc(present);
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
            if ((present >> b) & 1u) ox |= (code++) << (8 * b);
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if ((present >> (b + 4)) & 1u) oy |= (code++) << (8 * b);
        sigma = __shfl_sync(kFullMask, incl, 31) + 1;  // + the zero row
        if (sigma > 256u || sigma * cs > uint32_t(d.pm_bytes)) return 0u;
        // an absent byte value (exists: at most 255 are present)
        const uint32_t absent = ~present & 0xffu;
        const uint32_t has = __ballot_sync(kFullMask, absent != 0u);
        const int zl = __ffs(has) - 1;
        const uint32_t zb = __shfl_sync(kFullMask, uint32_t(8 * lane) + __ffs(absent) - 1, zl);
        *zrep = zb * 0x01010101u;
        reinterpret_cast<uint2*>(map)[lane] = make_uint2(ox, oy);
        uint4* pm4 = reinterpret_cast<uint4*>(pm);
        for (uint32_t i = lane; i < sigma * (cs / 16); i += 32) pm4[i] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();

    // Match masks: bit (j - c0) of the lane's K words for every column j.  A
    // 16-column chunk touches at most two words: A (its first column's) and B.
    for (int ch = 0; ch < nch_max; ++ch) {
        const int jr0 = ch * 16 - a_c;
        const uint32_t vm = ch < nch ? valid_mask16(jr0, clen) : 0u;
        const uint4 c = fetch_chunk(cstart, ch, vm, p.col_lo, p.col_hi, d.safe16);
        const int sh0 = jr0 & 31;
        const int w0 = jr0 >> 5;
        const int w1 = w0 + 1;
        const uint32_t woffA = wide ? uint32_t((w0 >> 2) * 512 + (w0 & 3) * 4) + lane * 16u
                                    : lane * ls + uint32_t(w0 * 4);
        const uint32_t woffB = wide ? uint32_t((w1 >> 2) * 512 + (w1 & 3) * 4) + lane * 16u
                                    : lane * ls + uint32_t(w1 * 4);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            if ((vm >> r) & 1u) {
                const int t = sh0 + r;
                const uint32_t code = map[chunk_byte(c, r)];
                uint32_t* wp = reinterpret_cast<uint32_t*>(pm + code * cs + (t < 32 ? woffA : woffB));
                *wp |= 1u << (t & 31);
            }
        }
    }
    __syncwarp();
    return sigma;
}

// Row sweep of a task whose masks are built.  S (lanes per pair) is runtime;
// returns the lane's count of zero bits below `cols`.
template <bool CHAIN, int K>
__device__ __forceinline__ int sweep_task(const BatchDev& d, const LanePair& p, int S, int s,
                                       const uint8_t* smem, uint32_t zrep) {
    const uint32_t lane = lane_id();
    const uint8_t* map = smem;
    const uint8_t* pm = smem + kMapBytes;
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int a_r = int(reinterpret_cast<uintptr_t>(p.rowp) & 15u);
    const uint8_t* rstart = p.rowp - a_r;
    const int nrch = p.rows > 0 ? int((p.rows + a_r + 15) / 16) : 0;
    const int T = warp_max(nrch) + S - 1;
    const uint32_t lane_off = PmLayout<K>::word_offset(lane, 0);
    uint32_t cout = 0;
    uint32_t vm = chunk_valid_mask(int64_t(-s) * 16 - a_r, p.rows);
    uint4 cur = fetch_chunk(rstart, -s, vm, p.row_lo, p.row_hi, d.safe16);
    for (int t = 0; t < T; ++t) {
        const int ch = t - s;
        const uint32_t vm_next = chunk_valid_mask(int64_t(ch + 1) * 16 - a_r, p.rows);
        const uint4 nxt = fetch_chunk(rstart, ch + 1, vm_next, p.row_lo, p.row_hi, d.safe16);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        if (!__all_sync(kFullMask, vm == 0xffffu)) cur = sanitize_chunk(cur, vm, zrep);
        uint32_t off[16];
        chunk_offsets(cur, map, cs, lane_off, off);
        rows16<CHAIN, K>(V, pm, off, vm, cin, cout, NoRowHook{});
        cur = nxt;
        vm = vm_next;
    }
    return lane_zero_count<K>(V, int64_t(s) * K, p.cols);
}

#define WLCS_SWEEP_CASE(CH, KK) \
    case (CH) * 8 + (KK - 1):   \
        zeros = sweep_task<CH, KK>(d, p, S, s, smem, zrep); \
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
        const int sidx = c / kMaxK;
        const int K = c % kMaxK + 1;
        const int S = 1 << sidx;
        const uint32_t per_task = 32u >> sidx;
        const uint32_t first = pair_start[order] + (t - task_start[order]) * per_task;
        const uint32_t end = pair_start[order] + count[order];
        const uint32_t last = first + per_task < end ? first + per_task : end;

        const int seg = int(lane) >> sidx;
        const int s = int(lane) & (S - 1);
        const uint32_t idx = first + uint32_t(seg);
        const bool active = idx < last;
        const uint32_t pair = active ? d.vals[idx] : 0u;
        const LanePair p = lane_pair(d, active, pair);
        uint32_t zrep = 0;
        if (build_task(d, p, K, s, smem, &zrep) == 0u) {
            // Alphabet too large for this warp's shared-memory slice.
            if (active && s == 0) d.overflow[atomicAdd(d.meta + kMetaOverflow, 1u)] = pair;
            continue;
        }
        int zeros = 0;
        switch ((S > 1 ? 8 : 0) + (K - 1)) {
            WLCS_SWEEP_CASE(0, 1) WLCS_SWEEP_CASE(0, 2) WLCS_SWEEP_CASE(0, 3)
            WLCS_SWEEP_CASE(0, 4) WLCS_SWEEP_CASE(0, 5) WLCS_SWEEP_CASE(0, 6)
            WLCS_SWEEP_CASE(0, 7) WLCS_SWEEP_CASE(0, 8)
            WLCS_SWEEP_CASE(1, 5) WLCS_SWEEP_CASE(1, 6) WLCS_SWEEP_CASE(1, 7)
            WLCS_SWEEP_CASE(1, 8)
            default:
                break;  // unreachable: S >= 2 always has K >= 5
        }
        for (int o = S >> 1; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
        if (active && s == 0) d.out[pair] = uint32_t(zeros);
    }
}
#undef WLCS_SWEEP_CASE

}  // namespace

size_t batch_workspace_bytes(uint32_t pairs, size_t* aux_bytes) {
    *aux_bytes = 0;
    return (kWsPairs + 3 * size_t(pairs)) * sizeof(uint32_t);
}

int batch_smem_per_cta(int pm_bytes) { return kMapBytes + pm_bytes; }

// Enqueue the whole batch on `stream` (device pointers only).  Pairs routed to
// the single-pair path are listed in the workspace (batch_overflow_*_ptr).
// Optional events bracket the main kernel (bench.py's roofline timing).
cudaError_t batch_launch(BatchDev d, void* workspace, size_t /*aux_bytes*/, int sms,
                         cudaStream_t stream, cudaEvent_t ev_main0, cudaEvent_t ev_main1) {
    uint32_t* ws = static_cast<uint32_t*>(workspace);
    d.meta = ws;
    d.safe16 = reinterpret_cast<const uint4*>(ws + kMetaSafe16);
    uint32_t* hist = ws + kWsHist;
    uint32_t* cursor = ws + kWsCursor;
    uint32_t* bucket = ws + kWsPairs;
    d.vals = bucket + d.pairs;
    d.overflow = d.vals + d.pairs;
    cudaError_t e = cudaMemsetAsync(ws, 0, kWsCursor * sizeof(uint32_t), stream);  // meta + hist
    if (e != cudaSuccess) return e;
    if (d.pairs == 0) return cudaSuccess;
    const int blocks = int((d.pairs + 255) / 256);
    batch_plan_kernel<<<blocks, 256, 0, stream>>>(d, hist, bucket);
    batch_scan_kernel<<<1, 1024, 0, stream>>>(d, hist, cursor);
    batch_scatter_kernel<<<blocks, 256, 0, stream>>>(d, bucket, cursor);
    const int smem = batch_smem_per_cta(d.pm_bytes);
    e = cudaFuncSetAttribute(batch_main_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, batch_main_kernel, 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    if (ev_main0) cudaEventRecord(ev_main0, stream);
    batch_main_kernel<<<sms * occ, 32, smem, stream>>>(d);
    if (ev_main1) cudaEventRecord(ev_main1, stream);
    return cudaGetLastError();
}

uint32_t* batch_overflow_count_ptr(void* workspace, size_t, uint32_t) {
    return static_cast<uint32_t*>(workspace) + kMetaOverflow;
}

uint32_t* batch_overflow_list_ptr(void* workspace, size_t, uint32_t pairs) {
    return static_cast<uint32_t*>(workspace) + kWsPairs + 2 * size_t(pairs);
}

}  // namespace wlcs
