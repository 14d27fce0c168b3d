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
//            (S lanes per pair, K <= kmax words per lane -- 10 by default --,
//            S*K >= W; 5-8 word pairs take S = 2).  A counting sort (plan +
//            scatter: one cooperative launch with a grid barrier before the
//            bucket scan, or two kernels when the grid does not fit at once)
//            groups pairs by shape in queue order -- decreasing K, then S:
//            the longest tasks first, half-length ones last -- and, inside a
//            shape, by decreasing 16-row chunk count, so the pairs of one warp
//            task end on the same step.
//  * main:   persistent 1-warp CTAs pull tasks (32/S pairs of one shape) from
//            an atomic counter.  Per task the warp builds, in shared memory, a
//            byte->code map of the task's column alphabet (reused from the
//            previous task when it covers the new columns; a warp's first task
//            samples it from its lanes' first 32 column bytes) and the match
//            masks PM[code][word] (bit planes by PRMT + delta swaps; sweep.cuh
//            layouts: every warp-wide PM load is bank-conflict free), then
//            streams the row strings one aligned 16-byte chunk (16 rows) per
//            step, prefetching the next chunk.  Each row costs a DP4A (map
//            address, FMA pipe), the map and mask loads, and AND + IADD3.X +
//            LOP3 per 32 cells (rowstep.cuh).
//            With S>1 the S lanes of a pair form a skewed pipeline: lane s
//            works on chunk t-s and receives the 16 per-row carries of lane
//            s-1 as one 16-bit mask through __shfl_up_sync.
//  * result: LCS = zero bits of V below column `cols`, reduced over the
//            pair's S lanes.
#include <cstdlib>

#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kMaxK = 12;
#ifdef WLCS_BATCH_TRACE
// Diagnostic build only (tools/trace_probe.py): per task the globaltimer at
// its start and end, smid << 32 | build ns, (16 S + K) << 32 | max rows.
constexpr int kTraceMax = 1 << 15;
__device__ unsigned long long g_trace[kTraceMax][4];
__device__ unsigned int g_trace_n;
#endif
constexpr int kNumClasses = 6 * kMaxK;   // S in {1,2,4,8,16,32} x K in 1..12
constexpr int kChunkBuckets = 128;       // chunk-count buckets per class (clamped)
constexpr int kBuckets = kNumClasses * kChunkBuckets;
constexpr int kTableSlots = (kNumClasses + 31) / 32;  // task-table entries per lane
// per-warp shared memory before the masks: map [256] (byte -> code) | zmap [256]
// (all zero: the map of chunks outside a row string) | inv [16 x u16] (low-
// nibble presence per high nibble of the map's bytes) | pad
constexpr int kMapBytes = 576;
constexpr uint32_t kZmapOff = 256, kInvOff = 512;
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
//                     bucket[pairs] | vals[pairs] | overflow[pairs] | rank[pairs]
constexpr size_t kWsHist = kMetaWords;
constexpr size_t kWsCursor = kWsHist + kBuckets;
constexpr size_t kWsPairs = kWsCursor + kBuckets;

__device__ __forceinline__ int class_of(int sidx, int k) { return sidx * kMaxK + (k - 1); }

// Queue order of the lane-shape classes: decreasing K (words per lane: a
// task's duration is about K x its rows, whatever its S), then decreasing S
// -- the longest tasks first, and one sweep variant hot in the I-cache at a
// time (S = 2 and S = 4 share the chain variant of a K).  Pairs of 5-8 words
// take the S = 2, K <= 4 shape (half-length tasks) so the queue ends short.
#ifndef WLCS_BATCH_FINE_TAIL
#define WLCS_BATCH_FINE_TAIL 1
#endif
#ifndef WLCS_BATCH_FINE_MAXW
#define WLCS_BATCH_FINE_MAXW 8
#endif
__device__ __forceinline__ int order_of_class(int c) {
    const int k = c % kMaxK + 1, sidx = c / kMaxK;
    return (kMaxK - k) * 6 + (5 - sidx);
}
__device__ __forceinline__ int class_of_order(int o) {
    const int k = kMaxK - o / 6, sidx = 5 - o % 6;
    return class_of(sidx, k);
}

// Bucket (lane shape x row-chunk count, in queue order) of entry i and its
// rank inside the block's count of that bucket (shared-memory atomics on
// `local`); kNoBucket for empty pairs (answered here) and for pairs routed to
// the second pass.
__device__ __forceinline__ void plan_pair(const BatchDev& d, uint32_t i, uint32_t p, uint32_t* local,
                                          uint32_t& b, uint32_t& r) {
    b = kNoBucket;
    r = 0;
    if (i < d.pairs) {
        const uint64_t m = d.xoff[p + 1] - d.xoff[p];
        const uint64_t n = d.yoff[p + 1] - d.yoff[p];
        const uint64_t cols = m < n ? m : n;
        const uint64_t rows = m < n ? n : m;
        if (cols == 0) {
            d.out[p] = 0;  // empty input: length 0 (proj/tests/test_parallel.cpp:236-242)
        } else {
            const uint64_t w = (cols + 31) / 32;
            const uint64_t kmax = uint64_t(d.kmax);
            if (w > 32 * kmax || rows > (uint64_t(1) << 30)) {
                // Wider than one warp's lane shapes: the second pass (bitpar_wide.cu)
                // sweeps it in column blocks -- or, when the host holds the
                // offsets, the single-pair strip kernel (long_to_host).
                if (!(d.long_to_host && w > 32 * kmax)) {
                    const uint32_t i = atomicAdd(d.meta + kMetaOverflow, 1u);
                    d.overflow[i] = p;
                }
            } else {
                int sidx = 0;
                while ((kmax << sidx) < w) ++sidx;
                if (WLCS_BATCH_FINE_TAIL && sidx == 0 && w >= 5 && w <= WLCS_BATCH_FINE_MAXW) sidx = 1;
                const int s = 1 << sidx;
                const int k = int((w + s - 1) / s);
                const int order = order_of_class(class_of(sidx, k));
                uint64_t nch = (rows + 15) / 16;
                if (nch > kChunkBuckets - 1) nch = kChunkBuckets - 1;
                b = uint32_t(order * kChunkBuckets + (kChunkBuckets - 1 - int(nch)));
                r = atomicAdd(&local[b], 1u);
            }
        }
    }
}

// One thread per pair.  Besides the bucket it records the pair's rank inside
// its bucket: a block-local rank (shared-memory atomics) plus the block's base
// in that bucket (one global atomic per block and bucket), so the scatter
// needs no atomics.
constexpr int kPlanThreads = 1024;  // fewer blocks: fewer bucket flushes / global atomics
__global__ void __launch_bounds__(kPlanThreads) batch_plan_kernel(BatchDev d, uint32_t* hist,
                                                         uint32_t* bucket, uint32_t* rank) {
    // programmatic dependent launch: the scatter kernel may launch now; it
    // waits (griddepcontrol.wait) for this grid's hist / bucket / rank
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t local[kBuckets];
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) local[i] = 0;
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t p = i < d.pairs ? (d.ids ? d.ids[i] : i) : 0u;
    uint32_t b = kNoBucket, r = 0;
    plan_pair(d, i, p, local, b, r);
    __syncthreads();
    {
        // block base inside every bucket: the kBuckets / kPlanThreads returning
        // atomics of a thread are issued back to back (all in flight at once)
        constexpr int kPer = kBuckets / kPlanThreads;
        static_assert(kBuckets % kPlanThreads == 0, "bucket split");
        uint32_t c[kPer], base[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) c[k] = local[threadIdx.x + k * kPlanThreads];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            base[k] = c[k] ? atomicAdd(hist + threadIdx.x + k * kPlanThreads, c[k]) : 0u;
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (c[k]) local[threadIdx.x + k * kPlanThreads] = base[k];
    }
    __syncthreads();
    if (i < d.pairs) {
        bucket[i] = b;
        rank[i] = b == kNoBucket ? 0u : local[b] + r;
    }
}

// Exclusive scan of the bucket histogram into shared memory (every scatter
// block does it: 9216 counts, cheaper than a separate single-block launch);
// block 0 also writes the per-order pair ranges and the task table.
__device__ __forceinline__ void scan_buckets(const BatchDev& d, const uint32_t* hist,
                                             uint32_t* cursor, bool bookkeeping) {
    constexpr int kPer = kBuckets / 1024;
    static_assert(kBuckets % 1024 == 0, "scan split");
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t order_start[kNumClasses + 1];
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
        const int b = tid * kPer + i;
        if (b % kChunkBuckets == 0) order_start[b / kChunkBuckets] = run;
        cursor[b] = run;
        run += v[i];
    }
    if (tid == 1023) order_start[kNumClasses] = run;
    __syncthreads();
    if (bookkeeping && warp == 0) {
        // orders 3*lane .. 3*lane+2: counts, starts, task counts, then an
        // exclusive scan of the task counts in order
        uint32_t nt[kTableSlots], tsum = 0;
#pragma unroll
        for (int q = 0; q < kTableSlots; ++q) {
            const int o = lane * kTableSlots + q;
            nt[q] = 0;
            if (o < kNumClasses) {
                const uint32_t per_task = 32u >> (class_of_order(o) / kMaxK);
                const uint32_t cnt = order_start[o + 1] - order_start[o];
                d.meta[kMetaCount + o] = cnt;
                d.meta[kMetaPairStart + o] = order_start[o];
                nt[q] = (cnt + per_task - 1) / per_task;
            }
            tsum += nt[q];
        }
        uint32_t ti = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFullMask, ti, o);
            if (lane >= o) ti += t;
        }
        uint32_t ts = ti - tsum;
#pragma unroll
        for (int q = 0; q < kTableSlots; ++q) {
            const int o = lane * kTableSlots + q;
            if (o < kNumClasses) d.meta[kMetaTaskStart + o] = ts;
            ts += nt[q];
        }
        if (lane == 31) d.meta[kMetaTaskStart + kNumClasses] = ti;
    }
}

// 1024-thread blocks, kScatterPairs pairs each: scan, then place every pair
// id at cursor[bucket] + rank.
constexpr int kScatterPairs = 2048;
__global__ void __launch_bounds__(1024) batch_scatter_kernel(BatchDev d, const uint32_t* hist,
                                                             const uint32_t* bucket,
                                                             const uint32_t* rank) {
    __shared__ uint32_t cursor[kBuckets];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the plan kernel's results
    scan_buckets(d, hist, cursor, blockIdx.x == 0);
    const uint32_t i0 = blockIdx.x * uint32_t(kScatterPairs);
    const uint32_t i1 = min(d.pairs, i0 + uint32_t(kScatterPairs));
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const uint32_t b = bucket[i];
        if (b == kNoBucket) continue;
        d.vals[cursor[b] + rank[i]] = d.ids ? d.ids[i] : i;
    }
}

// Plan and scatter in ONE cooperative launch (all blocks co-resident; one
// grid barrier between the bucket counts and the scan): a pair's bucket and
// rank stay in registers, and the main kernel waits on one launch instead of
// two.  Used when the grid fits the device at once (batch_launch); the two
// kernels above are the fallback.
constexpr int kMetaBarrier = 3 * kNumClasses + 3;
__global__ void __launch_bounds__(1024) batch_plan_scatter_kernel(BatchDev d, uint32_t* hist) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t local[kBuckets];
    for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) local[i] = 0;
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t p = i < d.pairs ? (d.ids ? d.ids[i] : i) : 0u;
    uint32_t b = kNoBucket, r = 0;
    plan_pair(d, i, p, local, b, r);
    __syncthreads();
    {
        constexpr int kPer = kBuckets / 1024;
        uint32_t c[kPer], base[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) c[k] = local[threadIdx.x + k * 1024];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            base[k] = c[k] ? atomicAdd(hist + threadIdx.x + k * 1024, c[k]) : 0u;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPer; ++k) local[threadIdx.x + k * 1024] = base[k];
    }
    const uint32_t rk = b == kNoBucket ? 0u : r;  // rank inside the block's run
    __syncthreads();
    const uint32_t blk_base = b == kNoBucket ? 0u : local[b];
    // grid barrier: every block's counts are in hist
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(d.meta + kMetaBarrier, 1u);
        uint32_t seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(d.meta + kMetaBarrier) : "memory");
        } while (seen < gridDim.x);
    }
    __syncthreads();
    scan_buckets(d, hist, local, blockIdx.x == 0);  // local := exclusive bucket starts
    __syncthreads();
    if (b != kNoBucket) d.vals[local[b] + blk_base + rk] = p;
}

// Per-lane view of its pair inside a task.
struct LanePair {
    const uint8_t* colp;  // column (bit-vector) string = the shorter one
    const uint8_t* rowp;
    const uint8_t *col_lo, *col_hi, *row_lo, *row_hi;
    int cols;             // <= 12288 in the batch path
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

// Decoded warp task t: pairs [first, last) of one lane shape (S, K).
struct TaskInfo {
    int sidx, S, K;
    uint32_t first, last;
};

// The task table (per class order: task start, pair start, pair count) is
// constant during the sweep kernel: every lane keeps orders `lane`,
// `lane + 32` and `lane + 64` in registers, so decoding a task is ballots and
// shuffles only.
static_assert(kTableSlots == 3, "task table slots");
struct TaskTable {
    uint32_t ts[kTableSlots], ps[kTableSlots], cn[kTableSlots];
};

__device__ __forceinline__ TaskTable load_task_table(const BatchDev& d, uint32_t lane) {
    const uint32_t* count = d.meta + kMetaCount;
    const uint32_t* pair_start = d.meta + kMetaPairStart;
    const uint32_t* task_start = d.meta + kMetaTaskStart;
    TaskTable tt;
#pragma unroll
    for (int i = 0; i < kTableSlots; ++i) {
        const uint32_t o = lane + 32u * i;
        const bool ok = o < uint32_t(kNumClasses);
        tt.ts[i] = ok ? task_start[o] : 0xffffffffu;
        tt.ps[i] = ok ? pair_start[o] : 0u;
        tt.cn[i] = ok ? count[o] : 0u;
    }
    return tt;
}

__device__ __forceinline__ TaskInfo decode_task(const TaskTable& tt, uint32_t t) {
    int order = -1;
#pragma unroll
    for (int i = 0; i < kTableSlots; ++i) order += __popc(__ballot_sync(kFullMask, tt.ts[i] <= t));
    const int src = order & 31;
    const int slot = order >> 5;
    const uint32_t ts = __shfl_sync(kFullMask, slot == 0 ? tt.ts[0] : slot == 1 ? tt.ts[1] : tt.ts[2], src);
    const uint32_t ps = __shfl_sync(kFullMask, slot == 0 ? tt.ps[0] : slot == 1 ? tt.ps[1] : tt.ps[2], src);
    const uint32_t cn = __shfl_sync(kFullMask, slot == 0 ? tt.cn[0] : slot == 1 ? tt.cn[1] : tt.cn[2], src);
    const int c = class_of_order(order);
    TaskInfo ti;
    ti.sidx = c / kMaxK;
    ti.K = c % kMaxK + 1;
    ti.S = 1 << ti.sidx;
    const uint32_t per_task = 32u >> ti.sidx;
    ti.first = ps + (t - ts) * per_task;
    const uint32_t end = ps + cn;
    ti.last = ti.first + per_task < end ? ti.first + per_task : end;
    return ti;
}

// ---------------------------------------------------------------------------
// Match-mask build (per warp task, in the sweep kernel).
//
// Each lane owns K consecutive words (32*K columns) of its pair's column
// string.  Per word the lane (1) realigns the 32 column bytes out of 16-byte
// aligned chunks (funnel shifts), (2) turns them into 8 bit-planes with four
// 8x8 bit transposes (plane b, bit j = bit b of column j's byte) and marks
// the bytes present.  After the warp's prefix scan has assigned dense codes,
// every code's match mask is the AND over the planes of "plane == bit of the
// code's byte value": a handful of LOP3 per (code, word), written once --
// no read-modify-write, no dependency chains, ALU only.
// The byte -> code map a warp keeps from one task to the next (hm == 0: none).
struct MapState {
    uint32_t hm;     // ballot of present high nibbles (bit 2h)
    uint32_t sigma;  // codes incl. the zero row
    uint32_t zrep;   // a byte absent from the map, replicated x4
};

// Dense codes 1..sigma-1 in byte order (0 = no match) for the byte set
// `present` (lane l holds bytes 8l .. 8l+7 as bits 0..7): writes the
// byte -> code map and the low-nibble presence per high nibble (inv), and
// returns sigma (codes incl. the zero row), the ballot of present high
// nibbles (bit 2h) and a byte absent from the set replicated x4.  False when
// more than 255 codes would be needed.
__device__ __forceinline__ bool assign_codes(uint32_t present, uint32_t map, uint32_t inv,
                                             uint32_t* sigma, uint32_t* hm, uint32_t* zrep) {
    const uint32_t lane = lane_id();
    const uint32_t cnt = __popc(present);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
        if (int(lane) >= o) incl += v;
    }
    *sigma = __shfl_sync(kFullMask, incl, 31) + 1;  // + the zero row
    if (*sigma > 256u) return false;
    uint32_t code = incl - cnt + 1;
    uint32_t ox = 0, oy = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if ((present >> b) & 1u) {
            if (b < 4) ox |= code << (8 * b);
            else oy |= code << (8 * (b - 4));
            ++code;
        }
    }
    // low-nibble presence per high nibble h (lanes 2h, 2h+1 hold bytes 16h..16h+15)
    const uint32_t upper = __shfl_down_sync(kFullMask, present, 1);
    const uint32_t nib16 = present | (upper << 8);
    *hm = __ballot_sync(kFullMask, (lane & 1u) == 0u && nib16 != 0u);
    const uint32_t absent = ~present & 0xffu;  // exists: at most 255 bytes present
    const uint32_t has = __ballot_sync(kFullMask, absent != 0u);
    const uint32_t zb = __shfl_sync(kFullMask, uint32_t(8 * lane) + __ffs(absent) - 1, __ffs(has) - 1);
    *zrep = zb * 0x01010101u;
    __syncwarp();
    sts_v2(map + 8u * lane, ox, oy);
    if ((lane & 1u) == 0u) sts_u16(inv + lane, nib16);
    return true;
}

// Presence flags (one 32-bit word per byte value at `flags`) of the valid
// bytes (bit r of vm) of a 16-byte chunk.
__device__ __forceinline__ void mark_chunk(const uint4& c, uint32_t vm, uint32_t flags) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if ((vm >> r) & 1u) {
            uint32_t a;
            asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(w[r >> 2]), "r"(4u << (8 * (r & 3))), "r"(flags));
            sts_u32(a, 1u);
        }
    }
}

// Builds the task's match masks (and, when needed, its byte -> code map) in
// shared memory.  K is a runtime value and every loop over words / codes is
// rolled: the build is one small piece of code shared by all lane shapes (it
// runs once per task while the sweep code is hot, so its I-cache footprint
// matters).
//
// Map reuse: tasks of one batch usually share their column alphabet (C2: the
// same 20 letters), so the warp first builds the masks with the PREVIOUS
// task's map and checks that every valid column matched one of its codes (the
// OR of the masks equals the valid-column mask).  Only when some column is not
// covered does it run the presence pass and the code scan and build again.
// Codes of the old map absent from this task just get all-zero masks.
//
// Returns sigma (codes incl. the zero row) or 0 when the alphabet does not fit
// the warp's shared-memory slice; *zrep receives a byte value absent from the
// map, replicated x4 (used to blank invalid rows in the sweep).
__device__ __forceinline__ uint32_t build_task(const BatchDev& d, const LanePair& p, int K, int s,
                                               uint32_t sbase, uint32_t* zrep, MapState& st) {
    const uint32_t lane = lane_id();
    const uint32_t map = sbase;           // byte -> code
    const uint32_t inv = sbase + kInvOff;  // u16 low-nibble presence per high nibble
    const uint32_t pm = sbase + uint32_t(kMapBytes);
    const bool wide = pm_slotted(K);
    const uint32_t cs = wide ? 512u * uint32_t((K + 3) / 4) : 128u * pm_lane_words(K);
    const uint32_t ls = wide ? 16u : 4u * pm_lane_words(K);

    // The lane's columns [c0, c0 + clen), read as the 16-byte aligned chunks
    // 0..2K of the region starting a_c bytes before them.
    const int c0 = 32 * K * s;
    const int clen = max(min(c0 + 32 * K, p.cols) - c0, 0);
    const uint8_t* cbase = p.colp + c0;
    const int a_c = int(reinterpret_cast<uintptr_t>(cbase) & 15u);
    const uint8_t* cstart = cbase - a_c;
    const int q = a_c >> 2;
    const uint32_t fs = uint32_t(a_c & 3) * 8u;
    auto chunk = [&](int i) {
        const uint32_t vm = i <= 2 * K ? valid_mask16(16 * i - a_c, clen) : 0u;
        return fetch_chunk(cstart, i, vm, p.col_lo, p.col_hi, d.safe16);
    };
    const int nchk = 2 * K + 1;
    const uint32_t stage = pm + uint32_t(d.pm_bytes) - uint32_t(nchk) * 512u;
    auto staged = [&](int i) {
        return i < nchk ? lds_v4(stage + uint32_t(i) * 512u + lane * 16u) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint32_t sigma = st.sigma, hm = st.hm;
    *zrep = st.zrep;
    // attempt 0: the previous task's map; attempt 2 (a warp's first task): a
    // map sampled from the first 32 column bytes of every lane; attempt 1 (a
    // column byte missing from the map): a fresh map from all columns
    int attempt = (hm != 0u && sigma * cs <= uint32_t(d.pm_bytes)) ? 0 : (hm == 0u ? 2 : 1);
    for (;;) {
        bool use_stage = false;
        if (attempt == 2) {
            const uint32_t flags = pm;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 2; ++i) sts_v4(flags + 16u * (lane * 2 + i), make_uint4(0u, 0u, 0u, 0u));
            const uint4 s0 = chunk(0), s1 = chunk(1);
            const uint32_t v0 = valid_mask16(-a_c, clen), v1 = valid_mask16(16 - a_c, clen);
            __syncwarp();
            mark_chunk(s0, v0, flags);
            mark_chunk(s1, v1, flags);
            __syncwarp();
            const uint4 f0 = lds_v4(flags + 32u * lane);
            const uint4 f1 = lds_v4<16>(flags + 32u * lane);
            const uint32_t present = (f0.x ? 1u : 0u) | (f0.y ? 2u : 0u) | (f0.z ? 4u : 0u) |
                                     (f0.w ? 8u : 0u) | (f1.x ? 16u : 0u) | (f1.y ? 32u : 0u) |
                                     (f1.z ? 64u : 0u) | (f1.w ? 128u : 0u);
            __syncwarp();
            if (!assign_codes(present, map, inv, &sigma, &hm, zrep) ||
                sigma * cs > uint32_t(d.pm_bytes)) {
                attempt = 1;
                continue;
            }
            __syncwarp();
        }
        if (attempt == 1) {
            // presence flags: one 32-bit word per byte value in the (not yet
            // used) PM region -- lanes marking the same byte hit the same word
            const uint32_t flags = pm;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 2; ++i) sts_v4(flags + 16u * (lane * 2 + i), make_uint4(0u, 0u, 0u, 0u));
            // Stage the lane's 2K+1 column chunks in shared memory with cp.async
            // (one exposed global latency per task instead of one per word and
            // pass): at the end of the mask region, [chunk][lane] x 16 bytes.
            bool slow = false;
            for (int i = 0; i < nchk; ++i) {
                const uint8_t* src = cstart + 16 * i;
                const uint32_t vm = valid_mask16(16 * i - a_c, clen);
                const bool inb = src >= p.col_lo && src + 16 <= p.col_hi;
                slow |= vm != 0u && !inb;
                const void* g = (vm != 0u && inb) ? static_cast<const void*>(src)
                                                    : static_cast<const void*>(d.safe16);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 stage + uint32_t(i) * 512u + lane * 16u),
                             "l"(g)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
            if (__any_sync(kFullMask, slow)) {  // a chunk straddles the buffer end (rare)
                for (int i = 0; i < nchk; ++i) {
                    const uint8_t* src = cstart + 16 * i;
                    const uint32_t vm = valid_mask16(16 * i - a_c, clen);
                    if (vm != 0u && !(src >= p.col_lo && src + 16 <= p.col_hi))
                        sts_v4(stage + uint32_t(i) * 512u + lane * 16u,
                               load_chunk16(src, p.col_lo, p.col_hi));
                }
            }
            __syncwarp();  // flags zeroed, stage filled

            // pass 1: mark the bytes present
            {
                uint4 c0v = staged(0), c1v = staged(1), c2v = staged(2);
#pragma unroll 1
                for (int k = 0; k < K; ++k) {
                    const uint4 n1 = staged(2 * k + 3), n2 = staged(2 * k + 4);
                    uint32_t w[8];
                    word_bytes(c0v, c1v, c2v, q, fs, w);
                    const int nv = min(max(clen - 32 * k, 0), 32);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < nv)
                            sts_u32(flags + 4u * __byte_perm(w[j >> 2], 0u, 0x4440u | uint32_t(j & 3)), 1u);
                    c0v = c2v;
                    c1v = n1;
                    c2v = n2;
                }
            }
            __syncwarp();

            // dense codes 1..sigma-1 in byte order (0 = no match), low-nibble
            // presence per high nibble (in the inv region), zrep
            {
                const uint4 f0 = lds_v4(flags + 32u * lane);
                const uint4 f1 = lds_v4<16>(flags + 32u * lane);
                const uint32_t present = (f0.x ? 1u : 0u) | (f0.y ? 2u : 0u) | (f0.z ? 4u : 0u) |
                                         (f0.w ? 8u : 0u) | (f1.x ? 16u : 0u) | (f1.y ? 32u : 0u) |
                                         (f1.z ? 64u : 0u) | (f1.w ? 128u : 0u);  // byte 8*lane + b
                st.hm = 0u;  // the map is about to change
                if (!assign_codes(present, map, inv, &sigma, &hm, zrep) ||
                    sigma * cs > uint32_t(d.pm_bytes))
                    return 0u;
            }
            __syncwarp();
            use_stage = sigma * cs <= uint32_t(d.pm_bytes) - uint32_t(nchk) * 512u;
        }

        // pass 2, two words per iteration (their bit-plane transposes are
        // independent): bit-planes, then every code's match mask = valid
        // columns whose byte equals the code's byte value; `covered` checks
        // that every valid column matched a code of the map
        const uint32_t lane_off = wide ? lane * 16u : lane * ls;
        auto chunk2 = [&](int i) { return use_stage ? staged(i) : chunk(i); };
        auto woff_of = [&](int k) {
            return lane_off + (wide ? uint32_t((k >> 2) * 512 + (k & 3) * 4) : uint32_t(k * 4));
        };
        bool covered = true;
        {
            uint4 c0v = chunk2(0), c1v = chunk2(1), c2v = chunk2(2), c3v = chunk2(3), c4v = chunk2(4);
#pragma unroll 1
            for (int k = 0; k < K; k += 2) {
                const uint4 n1 = chunk2(2 * k + 5), n2 = chunk2(2 * k + 6), n3 = chunk2(2 * k + 7),
                            n4 = chunk2(2 * k + 8);
                uint32_t w0[8], w1[8], P0[8], P1[8];
                word_bytes(c0v, c1v, c2v, q, fs, w0);
                word_bytes(c2v, c3v, c4v, q, fs, w1);
                bit_planes8(w0, P0);
                bit_planes8(w1, P1);
                const bool has1 = k + 1 < K;  // warp-uniform
                const int nv0 = min(max(clen - 32 * k, 0), 32);
                const int nv1 = has1 ? min(max(clen - 32 * (k + 1), 0), 32) : 0;
                const uint32_t vm0 = nv0 >= 32 ? 0xffffffffu : ((1u << nv0) - 1u);
                const uint32_t vm1 = nv1 >= 32 ? 0xffffffffu : ((1u << nv1) - 1u);
                // words k, k+1 (k even) are adjacent and 8-byte aligned in every
                // layout: one STS.64 per code (half the stores, at most 2-way
                // bank conflicts where the 16-byte lane stride gave 4-way)
                uint32_t ca0 = pm + woff_of(k);
                if (has1) sts_v2(ca0, 0u, 0u);  // code 0: the zero row
                else sts_u32(ca0, 0u);
                const uint32_t a0[4] = {~(P0[0] | P0[1]), P0[0] & ~P0[1], ~P0[0] & P0[1], P0[0] & P0[1]};
                const uint32_t b0[4] = {~(P0[2] | P0[3]), P0[2] & ~P0[3], ~P0[2] & P0[3], P0[2] & P0[3]};
                const uint32_t a1[4] = {~(P1[0] | P1[1]), P1[0] & ~P1[1], ~P1[0] & P1[1], P1[0] & P1[1]};
                const uint32_t b1[4] = {~(P1[2] | P1[3]), P1[2] & ~P1[3], ~P1[2] & P1[3], P1[2] & P1[3]};
                uint32_t cov0 = 0, cov1 = 0;
                uint32_t groups = hm;
                while (groups) {  // warp-uniform
                    const uint32_t h = uint32_t(__ffs(groups) - 1) >> 1;
                    groups &= groups - 1u;
                    const uint32_t m4 = 0u - (h & 1u), m5 = 0u - ((h >> 1) & 1u),
                                   m6 = 0u - ((h >> 2) & 1u), m7 = 0u - ((h >> 3) & 1u);
                    const uint32_t hi0 = vm0 & ~((P0[4] ^ m4) | (P0[5] ^ m5) | (P0[6] ^ m6) | (P0[7] ^ m7));
                    const uint32_t hi1 = vm1 & ~((P1[4] ^ m4) | (P1[5] ^ m5) | (P1[6] ^ m6) | (P1[7] ^ m7));
                    const uint32_t nm = lds_u16(inv + 2u * h);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        if ((nm >> (4 * jj)) & 0xfu) {
                            const uint32_t hb0 = hi0 & b0[jj], hb1 = hi1 & b1[jj];
#pragma unroll
                            for (int ii = 0; ii < 4; ++ii) {
                                if ((nm >> (4 * jj + ii)) & 1u) {
                                    ca0 += cs;
                                    const uint32_t mk0 = hb0 & a0[ii], mk1 = hb1 & a1[ii];
                                    cov0 |= mk0;
                                    cov1 |= mk1;
                                    if (has1) sts_v2(ca0, mk0, mk1);
                                    else sts_u32(ca0, mk0);
                                }
                            }
                        }
                    }
                }
                covered = covered && cov0 == vm0 && cov1 == vm1;
                c0v = c4v;
                c1v = n1;
                c2v = n2;
                c3v = n3;
                c4v = n4;
            }
        }
        if (attempt == 1 || __all_sync(kFullMask, covered)) break;
        attempt = 1;
    }
    __syncwarp();
    st.hm = hm;
    st.sigma = sigma;
    st.zrep = *zrep;
    return sigma;
}

// Row sweep of a task whose masks are built.  S (lanes per pair) is runtime;
// returns the lane's count of zero bits below `cols`.
// Generic form: 64-bit chunk bounds and allocation checks every step (tasks
// whose row strings touch the ends of the input buffers).
template <bool CHAIN, int K>
__device__ __noinline__ int sweep_task_generic(const BatchDev& d, const LanePair& p, int S, int s,
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
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const uint32_t lo = h ? cur.z : cur.x;
            const uint32_t hi = h ? cur.w : cur.y;
            rows8<CHAIN, K>(V, map, pm, cs, lane_off, lo, hi, cin, cout);
        }
        cur = nxt;
        vm = vm_next;
    }
    return lane_zero_count<K>(V, int64_t(s) * K, p.cols);
}

// Fast form (every lane's chunks lie inside its buffer): per step one
// 16-byte load of the next chunk and the row updates.  Only the edge steps
// -- before every lane has reached its first full chunk, or after some lane
// has passed its last one -- classify chunks: chunks outside a row string
// read through the all-zero byte -> code table (identity rows) and the two
// partial chunks of a string are sanitized; the steps in between (every
// lane on a full chunk) skip all of it.  Shared memory is addressed through
// one 32-bit base.
template <bool CHAIN, int K>
__device__ __forceinline__ int sweep_task(const BatchDev& d, const LanePair& p, int S, int s,
                                          const uint8_t* smem, uint32_t sbase, uint32_t zrep) {
    const int a_r = int(reinterpret_cast<uintptr_t>(p.rowp) & 15u);
    const uint8_t* rstart = p.rowp - a_r;
    const int rows = int(p.rows);  // < 2^30 in the batch path
    const int nrch = rows > 0 ? (rows + a_r + 15) >> 4 : 0;
    const bool inb =
        nrch == 0 || (rstart >= p.row_lo && rstart + 16 * int64_t(nrch) <= p.row_hi);
    if (!__all_sync(kFullMask, inb)) return sweep_task_generic<CHAIN, K>(d, p, S, s, smem, zrep);
    const uint32_t lane = lane_id();
    const uint32_t map_a = sbase;
    const uint32_t zmap_a = map_a + kZmapOff;  // all zero: every byte -> code 0
    const uint32_t pm_a = map_a + uint32_t(kMapBytes) + PmLayout<K>::word_offset(lane, 0);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int T = warp_max(nrch) + S - 1;
    // steps [t_lo, t_hi): every lane's chunk t - s lies fully inside its string
    // (chunks [a_r ? 1 : 0, (rows + a_r) / 16) are full)
    const int t_lo = warp_max((a_r ? 1 : 0) + s);
    const int t_hi = max(-warp_max(-(((rows + a_r) >> 4) + s)), t_lo);
    uint32_t cout = 0;
    int lo = -16 * s - a_r;  // row index of byte 0 of chunk ch = t - s
    const uint4* cptr = reinterpret_cast<const uint4*>(rstart);
    uint4 cur = __ldg((s == 0 && nrch > 0) ? cptr : d.safe16);
    const uint4* nptr = cptr + (1 - s);  // chunk ch + 1
    for (int t = 0; t < T; ++t) {
        const int ch = t - s;
        const bool nv = unsigned(ch + 1) < unsigned(nrch);
        const uint4 nxt = ldg_l2pf(nv ? nptr : d.safe16);
        ++nptr;
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        uint32_t ma = map_a;
        if (t < t_lo || t >= t_hi) {  // warp-uniform: an edge step
            const bool none = lo >= rows || lo <= -16;
            const bool part = !none && (lo < 0 || lo > rows - 16);
            if (__any_sync(kFullMask, part)) {
                if (part) cur = sanitize_chunk(cur, valid_mask16(lo, rows), zrep);
            }
            if (none) ma = zmap_a;
        }
        uint32_t wlo = cur.x, whi = cur.y;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            rows8_sh<CHAIN, K>(V, ma, pm_a, wlo, whi, cin, cout);
            wlo = cur.z;
            whi = cur.w;
        }
        cur = nxt;
        lo += 16;
    }
    return lane_zero_count<K>(V, int64_t(s) * K, p.cols);
}

#define WLCS_SWEEP_CASE(CH, KK) \
    case (CH) * 16 + (KK - 1):  \
        zeros = sweep_task<CH, KK>(d, p, S, s, smem, sbase, zrep); \
        break;

__global__ void __launch_bounds__(32) batch_main_kernel(BatchDev d) {
    extern __shared__ __align__(16) uint8_t smem[];  // map [256] | inv [256] | PM
    const uint32_t lane = lane_id();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the scatter kernel's task table
    const uint32_t total = d.meta[kMetaTaskStart + kNumClasses];
    const TaskTable tt = load_task_table(d, lane);
    // shared base address, computed once (opaque, so it is not re-derived
    // from SR_CgaCtaId inside the loops)
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    sts_v2(sbase + kZmapOff + 8u * lane, 0u, 0u);  // the all-zero map, once
    MapState mstate{0u, 0u, 0u};                    // no map yet
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(d.meta + kMetaCounter, 1u);
        t = __shfl_sync(kFullMask, t, 0);
        if (t >= total) break;
        const TaskInfo ti = decode_task(tt, t);
        const int K = ti.K;
        const int S = ti.S;
        const int s = int(lane) & (S - 1);
        const uint32_t idx = ti.first + (lane >> ti.sidx);
        const bool active = idx < ti.last;
        const uint32_t pair = active ? d.vals[idx] : 0u;
        const LanePair p = lane_pair(d, active, pair);
#ifdef WLCS_BATCH_TRACE
        unsigned long long trb0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trb0));
#endif
        uint32_t zrep = 0;
        if (build_task(d, p, K, s, sbase, &zrep, mstate) == 0u) {
            // Alphabet too large for this warp's shared-memory slice.
            if (active && s == 0) d.overflow[atomicAdd(d.meta + kMetaOverflow, 1u)] = pair;
            continue;
        }
#ifdef WLCS_BATCH_TRACE
        unsigned long long tr0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
#endif
        int zeros = 0;
        switch ((S > 1 ? 16 : 0) + (K - 1)) {
            WLCS_SWEEP_CASE(0, 1) WLCS_SWEEP_CASE(0, 2) WLCS_SWEEP_CASE(0, 3)
            WLCS_SWEEP_CASE(0, 4) WLCS_SWEEP_CASE(0, 5) WLCS_SWEEP_CASE(0, 6)
            WLCS_SWEEP_CASE(0, 7) WLCS_SWEEP_CASE(0, 8) WLCS_SWEEP_CASE(0, 9)
            WLCS_SWEEP_CASE(0, 10) WLCS_SWEEP_CASE(0, 11) WLCS_SWEEP_CASE(0, 12)
            WLCS_SWEEP_CASE(1, 1) WLCS_SWEEP_CASE(1, 2) WLCS_SWEEP_CASE(1, 3)
            WLCS_SWEEP_CASE(1, 4) WLCS_SWEEP_CASE(1, 5) WLCS_SWEEP_CASE(1, 6)
            WLCS_SWEEP_CASE(1, 7) WLCS_SWEEP_CASE(1, 8) WLCS_SWEEP_CASE(1, 9)
            WLCS_SWEEP_CASE(1, 10) WLCS_SWEEP_CASE(1, 11) WLCS_SWEEP_CASE(1, 12)
            default:
                break;  // unreachable
        }
        for (int o = S >> 1; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
        if (active && s == 0) d.out[pair] = uint32_t(zeros);
#ifdef WLCS_BATCH_TRACE
        {
            unsigned long long tr1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
            const int mr = warp_max(int(p.rows));
            if (lane == 0) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                const unsigned i = atomicAdd(&g_trace_n, 1u);
                if (i < kTraceMax) {
                    g_trace[i][0] = trb0;
                    g_trace[i][1] = tr1;
                    g_trace[i][2] = (uint64_t(smid) << 32) | uint32_t(tr0 - trb0);
                    g_trace[i][3] = (uint64_t(S * 16 + K) << 32) | uint32_t(mr);
                }
            }
        }
#endif
    }
}
#undef WLCS_SWEEP_CASE

}  // namespace

size_t batch_workspace_bytes(uint32_t pairs, int /*pm_bytes*/) {
    return (kWsPairs + 4 * size_t(pairs)) * sizeof(uint32_t);
}

int batch_smem_per_cta(int pm_bytes) { return kMapBytes + pm_bytes; }

// Enqueue the whole batch on `stream` (device pointers only).  Pairs routed to
// the single-pair path are listed in the workspace (batch_overflow_*_ptr).
// Optional events bracket the main kernel (bench.py's roofline timing).
// WLCS_BATCH_TWO_KERNEL_PLAN=1 forces the two-kernel plan (A/B, tests)
static const bool g_no_fused_plan = [] {
    const char* v = std::getenv("WLCS_BATCH_TWO_KERNEL_PLAN");
    return v && v[0] == '1';
}();

cudaError_t batch_launch(BatchDev d, void* workspace, int sms, cudaStream_t stream,
                         cudaEvent_t ev_main0, cudaEvent_t ev_main1) {
    uint32_t* ws = static_cast<uint32_t*>(workspace);
    d.meta = ws;
    d.safe16 = reinterpret_cast<const uint4*>(ws + kMetaSafe16);
    uint32_t* hist = ws + kWsHist;
    uint32_t* bucket = ws + kWsPairs;
    d.vals = bucket + d.pairs;
    d.overflow = d.vals + d.pairs;
    uint32_t* rank = d.overflow + d.pairs;
    cudaError_t e = cudaMemsetAsync(ws, 0, kWsCursor * sizeof(uint32_t), stream);  // meta + hist
    if (e != cudaSuccess) return e;
    if (d.pairs == 0) return cudaSuccess;
    // kernel attributes and the occupancy query once per (thread, device,
    // smem size): fewer driver calls on every launch
    thread_local int cached_dev = -1, cached_smem = -1, cached_occ = 0;
    const int smem = batch_smem_per_cta(d.pm_bytes);
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev != cached_dev || smem != cached_smem) {
        int occ = 0;
        e = cudaFuncSetAttribute(batch_main_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(batch_main_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, batch_main_kernel, 32, smem);
        if (e != cudaSuccess) return e;
        cached_dev = dev;
        cached_smem = smem;
        cached_occ = occ < 1 ? 1 : occ;
    }
    const int occ = cached_occ;
    // plan + scatter: one cooperative launch when all its blocks fit the
    // device at once, else the two kernels (scatter as a programmatic
    // dependent launch of the plan)
    thread_local int cached_fused_dev = -1, cached_fused_blocks = 0;
    if (dev != cached_fused_dev) {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batch_plan_scatter_kernel, 1024, 0);
        if (e != cudaSuccess) return e;
        cached_fused_dev = dev;
        cached_fused_blocks = per_sm * sms;
    }
    const unsigned plan_blocks = unsigned((d.pairs + 1023) / 1024);
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.stream = stream;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    cfg.dynamicSmemBytes = 0;
    cfg.blockDim = dim3(1024);
    bool fused = !g_no_fused_plan && int(plan_blocks) <= cached_fused_blocks;
    if (fused) {
        cudaLaunchAttribute coop[1];
        coop[0].id = cudaLaunchAttributeCooperative;
        coop[0].val.cooperative = 1;
        cudaLaunchConfig_t fc{};
        fc.stream = stream;
        fc.attrs = coop;
        fc.numAttrs = 1;
        fc.gridDim = dim3(plan_blocks);
        fc.blockDim = dim3(1024);
        fc.dynamicSmemBytes = 0;
        e = cudaLaunchKernelEx(&fc, batch_plan_scatter_kernel, d, hist);
        if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
            // the device is shared (its blocks would not all be resident):
            // the two-kernel plan needs no co-residency
            (void)cudaGetLastError();
            fused = false;
        } else if (e != cudaSuccess) {
            return e;
        }
    }
    if (!fused) {
        batch_plan_kernel<<<int((d.pairs + kPlanThreads - 1) / kPlanThreads), kPlanThreads, 0,
                            stream>>>(d, hist, bucket, rank);
        cfg.gridDim = dim3(unsigned((d.pairs + kScatterPairs - 1) / kScatterPairs));
        e = cudaLaunchKernelEx(&cfg, batch_scatter_kernel, d, static_cast<const uint32_t*>(hist),
                               static_cast<const uint32_t*>(bucket),
                               static_cast<const uint32_t*>(rank));
        if (e != cudaSuccess) return e;
    }
    if (ev_main0) {
        // an event between the two kernels ends the overlap: the timed main
        // kernel is launched plainly
        cudaEventRecord(ev_main0, stream);
        batch_main_kernel<<<sms * occ, 32, smem, stream>>>(d);
    } else {
        cfg.gridDim = dim3(unsigned(sms * occ));
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = size_t(smem);
        e = cudaLaunchKernelEx(&cfg, batch_main_kernel, d);
        if (e != cudaSuccess) return e;
    }
    if (ev_main1) cudaEventRecord(ev_main1, stream);
    return cudaGetLastError();
}

#ifdef WLCS_BATCH_TRACE
}  // namespace wlcs
extern "C" int wlcs_debug_batch_trace(unsigned long long* out, unsigned int cap, int reset) {
    unsigned int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, wlcs::g_trace_n, 4);
    if (n > unsigned(wlcs::kTraceMax)) n = wlcs::kTraceMax;
    if (n > cap) n = cap;
    if (out && n) cudaMemcpyFromSymbol(out, wlcs::g_trace, size_t(n) * 32);
    if (reset) {
        const unsigned int z = 0;
        cudaMemcpyToSymbol(wlcs::g_trace_n, &z, 4);
    }
    return int(n);
}
namespace wlcs {
#endif

uint32_t* batch_overflow_count_ptr(void* workspace, uint32_t) {
    return static_cast<uint32_t*>(workspace) + kMetaOverflow;
}

uint32_t* batch_overflow_list_ptr(void* workspace, uint32_t pairs) {
    return static_cast<uint32_t*>(workspace) + kWsPairs + 2 * size_t(pairs);
}

}  // namespace wlcs
