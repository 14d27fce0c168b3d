// bitpar_wide.cu -- second pass of the batched bit-parallel lengths: the pairs
// the first pass (bitpar_batch.cu) lists as overflow, finished on the device
// without a host round trip.
//
// The first pass hands over pairs whose column alphabet does not fit its
// per-warp mask budget and pairs wider than 32 * kmax words.  Here every pair
// runs at one word per lane (K = 1) with the general mask table: 16-bit byte
// -> code map (all 256 byte values plus the zero row fit), 257 code rows of
// 128 bytes.  Pairs of up to 32 words take S = next power of two >= W lanes
// (the first pass's lane pipeline at K = 1); wider pairs take the whole warp
// and sweep the rows once per 1024-column block, left to right: lane 31's
// 16-row carry masks of block b go to a global scratch word per row chunk and
// enter lane 0 in block b + 1 -- the strip hand-off of bitpar_pair.cu, played
// by one warp in sequence (no inter-warp waits).
//
// Enqueued unconditionally after the first pass: the planner reads the
// overflow count on the device, so an empty second pass costs two short
// launches and no synchronisation.  Same integers as lcs_cell
// (proj/include/wavelcs/cell.hpp:30-38) via the Hyyro identity.
#include "sweep.cuh"
#include "wlcs_device.h"

namespace wlcs {
namespace {

constexpr int kWideOrders = 6;      // S = 32, 16, 8, 4, 2, 1 (queue order)
constexpr int kWideChunkBuckets = 128;
constexpr int kWideBuckets = kWideOrders * kWideChunkBuckets;
constexpr int kWideBlockCols = 1024;  // 32 lanes x 1 word
// meta (uint32): task start [7] | pair start [6] | count [6] | ticket
constexpr int kWmTaskStart = 0;
constexpr int kWmPairStart = 8;
constexpr int kWmCount = 16;
constexpr int kWmTicket = 24;
constexpr int kWmSafe16 = 28;  // 16 zero bytes (chunk loads with no valid byte)
constexpr int kWmWords = 32;
// shared memory per warp: map u16[256] | inv u16[16] (+pad) | masks [257][32 lanes]
constexpr uint32_t kWideMapBytes = 1024;
constexpr uint32_t kWideCodeStride = 128;
constexpr int kWideSmem = int(kWideMapBytes) + 257 * int(kWideCodeStride);

struct WidePair {
    const uint8_t* colp;
    const uint8_t* rowp;
    const uint8_t *col_lo, *col_hi, *row_lo, *row_hi;
    int64_t cols, rows;
    int64_t slot;  // first carry-scratch word of the row string's chunk 0
};

__device__ __forceinline__ WidePair wide_pair(const WideDev& d, bool active, uint32_t pair) {
    WidePair p{d.xs, d.xs, d.xs, d.xs, d.xs, d.xs, 0, 0, 0};
    if (!active) return p;
    const uint64_t xo = d.xoff[pair], yo = d.yoff[pair];
    const int64_t m = int64_t(d.xoff[pair + 1] - xo);
    const int64_t n = int64_t(d.yoff[pair + 1] - yo);
    // shorter string = columns (LCS length is symmetric)
    const bool y_cols = n <= m;
    p.colp = y_cols ? d.ys + yo : d.xs + xo;
    p.cols = y_cols ? n : m;
    p.col_lo = y_cols ? d.ys : d.xs;
    p.col_hi = y_cols ? d.ys + d.ys_bytes : d.xs + d.xs_bytes;
    p.rowp = y_cols ? d.xs + xo : d.ys + yo;
    p.rows = y_cols ? m : n;
    p.row_lo = y_cols ? d.xs : d.ys;
    p.row_hi = y_cols ? d.xs + d.xs_bytes : d.ys + d.ys_bytes;
    // chunk ranges of different strings of one buffer overlap in at most one
    // 16-byte chunk: shifting by the pair index makes them disjoint
    const int64_t rchunk = (reinterpret_cast<uintptr_t>(p.rowp) & ~uintptr_t(15)) -
                           reinterpret_cast<uintptr_t>(p.row_lo);
    p.slot = rchunk / 16 + int64_t(pair) +
             (y_cols ? 0 : int64_t(d.xs_bytes / 16) + int64_t(d.pairs_total) + 2);
    return p;
}

// One warp, one planner block: counting sort of the overflow list by (S
// descending, row chunks descending) and the task table.
__global__ void __launch_bounds__(1024) wide_plan_kernel(WideDev d) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the first pass's list and count
    __shared__ uint32_t hist[kWideBuckets];
    __shared__ uint32_t order_start[kWideOrders + 1];
    const int tid = threadIdx.x;
    for (int i = tid; i < kWideBuckets; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    uint32_t n = *d.count;
    if (n > d.cap) n = d.cap;
    for (uint32_t i = tid; i < n; i += blockDim.x) {
        const uint32_t p = d.list[i];
        const uint64_t m = d.xoff[p + 1] - d.xoff[p];
        const uint64_t nn = d.yoff[p + 1] - d.yoff[p];
        const uint64_t cols = m < nn ? m : nn, rows = m < nn ? nn : m;
        const uint64_t w = (cols + 31) / 32;
        int sidx = 0;
        while (sidx < 5 && (uint64_t(1) << sidx) < w) ++sidx;
        uint64_t nch = (rows + 15) / 16;
        if (nch > kWideChunkBuckets - 1) nch = kWideChunkBuckets - 1;
        const uint32_t b = uint32_t((5 - sidx) * kWideChunkBuckets + (kWideChunkBuckets - 1 - int(nch)));
        d.bucket[i] = b;
        d.rank[i] = atomicAdd(&hist[b], 1u);
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of 768 counts by one warp, 24 per lane
        constexpr int kPer = kWideBuckets / 32;
        uint32_t v[kPer], sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            v[k] = hist[tid * kPer + k];
            sum += v[k];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(kFullMask, incl, o);
            if (tid >= o) incl += t;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int b = tid * kPer + k;
            if (b % kWideChunkBuckets == 0) order_start[b / kWideChunkBuckets] = run;
            hist[b] = run;
            run += v[k];
        }
        if (tid == 31) order_start[kWideOrders] = run;
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += blockDim.x) d.vals[hist[d.bucket[i]] + d.rank[i]] = d.list[i];
    if (tid == 0) {
        uint32_t ts = 0;
        for (int o = 0; o < kWideOrders; ++o) {
            const uint32_t cnt = order_start[o + 1] - order_start[o];
            const uint32_t per_task = 32u >> (5 - o);  // order o holds S = 32 >> o
            d.meta[kWmTaskStart + o] = ts;
            d.meta[kWmPairStart + o] = order_start[o];
            d.meta[kWmCount + o] = cnt;
            ts += (cnt + per_task - 1) / per_task;
        }
        d.meta[kWmTaskStart + kWideOrders] = ts;
        d.meta[kWmTicket] = 0;
        for (int k = 0; k < 4; ++k) d.meta[kWmSafe16 + k] = 0;
    }
}

// Per-task mask build for this lane's 32 columns [c0, c0 + 32) of the block
// view `p` (K = 1): presence flags -> dense codes in byte order (16-bit map,
// so 257 codes fit) -> bit-planes -> one mask per present code.
__device__ __forceinline__ void wide_build(const WideDev& d, const WidePair& p, int64_t colbase,
                                           int s, uint32_t sbase) {
    const uint32_t lane = lane_id();
    const uint32_t map = sbase, inv = sbase + 512u, pm = sbase + kWideMapBytes;
    const uint32_t flags = pm;  // 256 presence words, overwritten by the masks below
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i) sts_v4(flags + 16u * (lane * 2 + i), make_uint4(0u, 0u, 0u, 0u));
    const int64_t c0 = colbase + 32 * int64_t(s);
    const int64_t rem = p.cols - c0;
    const int clen = rem <= 0 ? 0 : (rem >= 32 ? 32 : int(rem));
    const uint8_t* cbase = p.colp + (clen ? c0 : 0);
    const int a_c = int(reinterpret_cast<uintptr_t>(cbase) & 15u);
    const uint8_t* cstart = cbase - a_c;
    uint4 ch[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        ch[i] = fetch_chunk(cstart, i, valid_mask16(16 * i - a_c, clen), p.col_lo, p.col_hi,
                            d.safe16);
    uint32_t w[8];
    word_bytes(ch[0], ch[1], ch[2], a_c >> 2, uint32_t(a_c & 3) * 8u, w);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j)
        if (j < clen) sts_u32(flags + 4u * __byte_perm(w[j >> 2], 0u, 0x4440u | uint32_t(j & 3)), 1u);
    __syncwarp();
    uint32_t hm;
    {
        const uint4 f0 = lds_v4(flags + 32u * lane);
        const uint4 f1 = lds_v4<16>(flags + 32u * lane);
        const uint32_t present = (f0.x ? 1u : 0u) | (f0.y ? 2u : 0u) | (f0.z ? 4u : 0u) |
                                 (f0.w ? 8u : 0u) | (f1.x ? 16u : 0u) | (f1.y ? 32u : 0u) |
                                 (f1.z ? 64u : 0u) | (f1.w ? 128u : 0u);
        const uint32_t cnt = __popc(present);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
            if (int(lane) >= o) incl += v;
        }
        uint32_t code = incl - cnt + 1, packed[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            if ((present >> b) & 1u) {
                packed[b >> 1] |= code << (16 * (b & 1));
                ++code;
            }
        }
        const uint32_t upper = __shfl_down_sync(kFullMask, present, 1);
        const uint32_t nib16 = present | (upper << 8);
        hm = __ballot_sync(kFullMask, (lane & 1u) == 0u && nib16 != 0u);
        __syncwarp();
        sts_v4(map + 16u * lane, make_uint4(packed[0], packed[1], packed[2], packed[3]));
        if ((lane & 1u) == 0u) sts_u16(inv + lane, nib16);
    }
    __syncwarp();
    uint32_t P[8];
    bit_planes8(w, P);
    const uint32_t vmask = clen >= 32 ? 0xffffffffu : ((1u << clen) - 1u);
    uint32_t caddr = pm + 4u * lane;
    sts_u32(caddr, 0u);  // code 0: the zero row
    const uint32_t a[4] = {~(P[0] | P[1]), P[0] & ~P[1], ~P[0] & P[1], P[0] & P[1]};
    const uint32_t b4[4] = {~(P[2] | P[3]), P[2] & ~P[3], ~P[2] & P[3], P[2] & P[3]};
    while (hm) {  // warp-uniform: present high nibbles in increasing order
        const uint32_t h = uint32_t(__ffs(hm) - 1) >> 1;
        hm &= hm - 1u;
        const uint32_t hi_acc =
            vmask & ~((P[4] ^ (0u - (h & 1u))) | (P[5] ^ (0u - ((h >> 1) & 1u))) |
                      (P[6] ^ (0u - ((h >> 2) & 1u))) | (P[7] ^ (0u - ((h >> 3) & 1u))));
        const uint32_t nm = lds_u16(inv + 2u * h);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            if ((nm >> (4 * jj)) & 0xfu) {
                const uint32_t hb = hi_acc & b4[jj];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    if ((nm >> (4 * jj + ii)) & 1u) {
                        caddr += kWideCodeStride;
                        sts_u32(caddr, hb & a[ii]);
                    }
                }
            }
        }
    }
    __syncwarp();
}

// Row sweep of one column block at K = 1 with the S-lane carry pipeline;
// lane 0 takes its carries from cin_buf (previous block) and lane S-1 stores
// its carries to cout_buf (next block).  Invalid rows map to code 0.
__device__ __noinline__ int wide_sweep(const WideDev& d, const WidePair& p, int64_t colbase, int S,
                                       int s, uint32_t sbase, const uint16_t* cin_buf,
                                       uint16_t* cout_buf) {
    const uint32_t lane = lane_id();
    const uint16_t* map = reinterpret_cast<const uint16_t*>(
        static_cast<const uint8_t*>(__cvta_shared_to_generic(sbase)));
    const uint8_t* pm = static_cast<const uint8_t*>(__cvta_shared_to_generic(sbase + kWideMapBytes));
    uint32_t V[1] = {0xffffffffu};
    const int a_r = int(reinterpret_cast<uintptr_t>(p.rowp) & 15u);
    const uint8_t* rstart = p.rowp - a_r;
    const int64_t nrch = p.rows > 0 ? (p.rows + a_r + 15) / 16 : 0;
    const int T = warp_max(int(nrch)) + S - 1;
    uint32_t cout = 0;
    for (int t = 0; t < T; ++t) {
        const int ch = t - s;
        const uint32_t vm = chunk_valid_mask(int64_t(ch) * 16 - a_r, p.rows);
        const uint4 cur = fetch_chunk(rstart, ch, vm, p.row_lo, p.row_hi, d.safe16);
        uint32_t cin = __shfl_up_sync(kFullMask, cout, 1, S);
        const bool real = ch >= 0 && int64_t(ch) < nrch;
        if (s == 0) cin = (cin_buf != nullptr && real) ? uint32_t(cin_buf[ch]) : 0u;
        cin <<= 16;
        cout = 0;
        uint32_t off[16];
        chunk_offsets_masked(cur, vm, map, kWideCodeStride, 4u * lane, off);
        rows16<true, 1>(V, pm, off, vm, cin, cout, NoRowHook{});
        if (cout_buf != nullptr && s == S - 1 && real) cout_buf[ch] = uint16_t(cout);
    }
    return lane_zero_count<1>(V, int64_t(s), p.cols - colbase);
}

__global__ void __launch_bounds__(32) wide_kernel(WideDev d) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = lane_id();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the planner's table
    const uint32_t total = d.meta[kWmTaskStart + kWideOrders];
    if (total == 0) return;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    const uint32_t my_ts = lane < uint32_t(kWideOrders) ? d.meta[kWmTaskStart + lane] : 0xffffffffu;
    const uint32_t my_ps = lane < uint32_t(kWideOrders) ? d.meta[kWmPairStart + lane] : 0u;
    const uint32_t my_cn = lane < uint32_t(kWideOrders) ? d.meta[kWmCount + lane] : 0u;
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(d.meta + kWmTicket, 1u);
        t = __shfl_sync(kFullMask, t, 0);
        if (t >= total) break;
        const int order = __popc(__ballot_sync(kFullMask, my_ts <= t)) - 1;
        const uint32_t ts = __shfl_sync(kFullMask, my_ts, order);
        const uint32_t ps = __shfl_sync(kFullMask, my_ps, order);
        const uint32_t cn = __shfl_sync(kFullMask, my_cn, order);
        const int sidx = 5 - order, S = 1 << sidx;
        const uint32_t per_task = 32u >> sidx;
        const uint32_t first = ps + (t - ts) * per_task;
        const uint32_t last = min(first + per_task, ps + cn);
        const int s = int(lane) & (S - 1);
        const uint32_t idx = first + (lane >> sidx);
        const bool active = idx < last;
        const uint32_t pair = active ? d.vals[idx] : 0u;
        const WidePair p = wide_pair(d, active, pair);
        // one block unless the pair is wider than the warp (S = 32 only:
        // then the whole warp holds the one pair and the count is uniform)
        const int64_t words = (p.cols + 31) / 32;
        const int64_t blocks = (S == 32 && words > 32) ? (words + 31) / 32 : 1;
        int zeros = 0;
        for (int64_t b = 0; b < blocks; ++b) {
            const int64_t colbase = b * kWideBlockCols;
            wide_build(d, p, colbase, s, sbase);
            const uint16_t* cin_buf = b > 0 ? d.carry[b & 1] + p.slot : nullptr;
            uint16_t* cout_buf = b + 1 < blocks ? d.carry[(b + 1) & 1] + p.slot : nullptr;
            zeros += wide_sweep(d, p, colbase, S, s, sbase, cin_buf, cout_buf);
            __syncwarp();  // lane 31's carry stores before lane 0's loads of the next block
        }
        for (int o = S >> 1; o >= 1; o >>= 1) zeros += __shfl_xor_sync(kFullMask, zeros, o);
        if (active && s == 0) d.out[pair] = uint32_t(zeros);
    }
}

}  // namespace

size_t wide_workspace_bytes(uint32_t cap) {
    return (size_t(kWmWords) + 3 * size_t(cap)) * sizeof(uint32_t);
}

size_t wide_scratch_words(uint64_t xs_bytes, uint64_t ys_bytes, uint32_t pairs) {
    return size_t(xs_bytes / 16 + ys_bytes / 16) + 2 * size_t(pairs) + 16;
}

cudaError_t wide_launch(WideDev d, void* workspace, int sms, cudaStream_t stream) {
    uint32_t* ws = static_cast<uint32_t*>(workspace);
    d.meta = ws;
    d.safe16 = reinterpret_cast<const uint4*>(ws + kWmSafe16);  // zeroed by the planner
    d.vals = ws + kWmWords;
    d.bucket = d.vals + d.cap;
    d.rank = d.bucket + d.cap;
    thread_local int cached_dev = -1, cached_occ = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev != cached_dev) {
        e = cudaFuncSetAttribute(wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWideSmem);
        if (e != cudaSuccess) return e;
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wide_kernel, 32, kWideSmem);
        if (e != cudaSuccess) return e;
        cached_dev = dev;
        cached_occ = occ < 1 ? 1 : occ;
    }
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.stream = stream;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1024);
    e = cudaLaunchKernelEx(&cfg, wide_plan_kernel, d);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3(unsigned(sms * cached_occ));
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = size_t(kWideSmem);
    e = cudaLaunchKernelEx(&cfg, wide_kernel, d);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace wlcs
