// Microbenchmark: ALU-pipe utilisation of the batch row sweep in isolation
// (the production rows8_sh / RowStep code from csrc/sweep.cuh), without task
// scheduling or mask builds.  Each 1-warp CTA streams a private row string
// (16 rows per step, 16-byte chunk prefetched one step ahead as in
// sweep_task) against random match masks in shared memory; prints the row
// updates' ALU instructions per clock against the 2 per clock per SM peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//        -I../../paper_1306_4627_b200/csrc -o sweep_rate sweep_rate.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "sweep.cuh"

using namespace wlcs;

constexpr int kSigma = 21;
constexpr int kMapBytes = 576;

template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench(const uint8_t* rows, int steps, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    // map: bytes 'A'.. -> codes 1..20 (everything else 0); random masks
    for (int b = lane; b < 256; b += 32) smem[b] = (b >= 65 && b < 65 + kSigma - 1) ? uint8_t(b - 64) : 0;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t map_a = sbase;
    const uint32_t pm_a = sbase + kMapBytes + PmLayout<K>::word_offset(lane, 0);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 ring[AHEAD];
#pragma unroll
    for (int a = 0; a < AHEAD; ++a) ring[a] = ldg_l2pf(rp + a);
    uint32_t cout = 0;
    for (int t = 0; t < steps - AHEAD; ++t) {
        const uint4 cur = ring[0];
#pragma unroll
        for (int a = 0; a + 1 < AHEAD; ++a) ring[a] = ring[a + 1];
        ring[AHEAD - 1] = ldg_l2pf(rp + t + AHEAD);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        uint32_t wlo = cur.x, whi = cur.y;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            rows8_sh<CHAIN, K>(V, map_a, pm_a, wlo, whi, cin, cout);
            wlo = cur.z;
            whi = cur.w;
        }
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}


// Pipelined half-step form: the next half's 8 mask offsets (DP4A, LDS.U8,
// IMAD) and its first two rows' masks are fetched during the current half;
// carries between lanes move once per half and are consumed two halves later
// (the lane skew), so no latency sits at the head of a half.
template <int K>
__device__ __forceinline__ void offsets8(uint32_t* off, uint32_t map_a, uint32_t pm_a, uint32_t lo,
                                         uint32_t hi) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    off[0] = lds_u8(byte_addr<0>(lo, map_a)) * cs + pm_a;
    off[1] = lds_u8(byte_addr<1>(lo, map_a)) * cs + pm_a;
    off[2] = lds_u8(byte_addr<2>(lo, map_a)) * cs + pm_a;
    off[3] = lds_u8(byte_addr<3>(lo, map_a)) * cs + pm_a;
    off[4] = lds_u8(byte_addr<0>(hi, map_a)) * cs + pm_a;
    off[5] = lds_u8(byte_addr<1>(hi, map_a)) * cs + pm_a;
    off[6] = lds_u8(byte_addr<2>(hi, map_a)) * cs + pm_a;
    off[7] = lds_u8(byte_addr<3>(hi, map_a)) * cs + pm_a;
}

template <bool CHAIN, int K>
__device__ __forceinline__ void row_sh(uint32_t* V, const uint32_t* P, uint32_t& cin, uint32_t& cout) {
    if constexpr (CHAIN) RowStep<K>::chain(V, P, cin, cout);
    else RowStep<K>::plain(V, P);
}

template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench2(const uint8_t* rows, int steps, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    for (int b = lane; b < 256; b += 32) smem[b] = (b >= 65 && b < 65 + kSigma - 1) ? uint8_t(b - 64) : 0;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t map_a = sbase;
    const uint32_t pm_a = sbase + kMapBytes + PmLayout<K>::word_offset(lane, 0);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 cur = ldg_l2pf(rp), nxt = ldg_l2pf(rp + 1);
    uint32_t off[8];
    offsets8<K>(off, map_a, pm_a, cur.x, cur.y);
    uint32_t PA[K], PB[K];
    load_pm_sh<K>(off[0], PA);
    load_pm_sh<K>(off[1], PB);
    uint32_t cq0 = 0, cq1 = 0;
    const int halves = 2 * (steps - 2);
    for (int u = 0; u < halves; u += 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t lo_n, hi_n;
            if (h == 0) { lo_n = cur.z; hi_n = cur.w; }
            else { lo_n = nxt.x; hi_n = nxt.y; }
            uint32_t offn[8];
            offsets8<K>(offn, map_a, pm_a, lo_n, hi_n);
            uint32_t cin = 0, cout = 0;
            if constexpr (CHAIN) cin = (h == 0 ? cq0 : cq1) << 24;
            row_sh<CHAIN, K>(V, PA, cin, cout);
            row_sh<CHAIN, K>(V, PB, cin, cout);
#pragma unroll
            for (int r = 2; r < 8; ++r) {
                uint32_t P[K];
                load_pm_sh<K>(off[r], P);
                row_sh<CHAIN, K>(V, P, cin, cout);
            }
            load_pm_sh<K>(offn[0], PA);
            load_pm_sh<K>(offn[1], PB);
#pragma unroll
            for (int r = 0; r < 8; ++r) off[r] = offn[r];
            if constexpr (CHAIN) {
                uint32_t c = __shfl_up_sync(kFullMask, cout, 1, S);
                if (s == 0) c = 0;
                if (h == 0) cq0 = c; else cq1 = c;
            }
            if (h == 1) {
                cur = nxt;
                nxt = ldg_l2pf(rp + u / 2 + 2);
            }
        }
    }
    uint32_t acc = cq0 ^ cq1;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}


// Variant without the byte -> code map lookup: code = byte & 15 (timing
// only), offset = dp4a(w & 0x0f0f0f0f, (cs / 128) << 8r, 0) * 128 + pm_a.
template <int K, int R>
__device__ __forceinline__ uint32_t nomap_off(uint32_t wm, uint32_t pm_a) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t t;
    asm("dp4a.u32.u32 %0, %1, %2, 0;" : "=r"(t) : "r"(wm), "n"((cs / 128) << (8 * R)));
    return t * 128u + pm_a;
}

template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench3(const uint8_t* rows, int steps, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t pm_a = sbase + kMapBytes + PmLayout<K>::word_offset(lane, 0);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 cur = ldg_l2pf(rp);
    uint32_t cout = 0;
    for (int t = 0; t < steps - 1; ++t) {
        const uint4 nxt = ldg_l2pf(rp + t + 1);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        uint32_t wlo = cur.x & 0x0f0f0f0fu, whi = cur.y & 0x0f0f0f0fu;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            uint32_t off[8];
            off[0] = nomap_off<K, 0>(wlo, pm_a); off[1] = nomap_off<K, 1>(wlo, pm_a);
            off[2] = nomap_off<K, 2>(wlo, pm_a); off[3] = nomap_off<K, 3>(wlo, pm_a);
            off[4] = nomap_off<K, 0>(whi, pm_a); off[5] = nomap_off<K, 1>(whi, pm_a);
            off[6] = nomap_off<K, 2>(whi, pm_a); off[7] = nomap_off<K, 3>(whi, pm_a);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                uint32_t P[K];
                load_pm_sh<K>(off[r], P);
                if constexpr (CHAIN) RowStep<K>::chain(V, P, cin, cout);
                else RowStep<K>::plain(V, P);
            }
            wlo = cur.z & 0x0f0f0f0fu;
            whi = cur.w & 0x0f0f0f0fu;
        }
        cur = nxt;
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}

// Register-only row updates (masks rotate through 4 preloaded sets): the
// ALU ceiling of the row-update instruction mix itself.
template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench4(const uint8_t* rows, int steps, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t P[4][K];
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1) ^ uint32_t(rows[lane]);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int k = 0; k < K; ++k) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; P[c][k] = x; }
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    uint32_t cout = 0;
    for (int t = 0; t < steps - 1; ++t) {
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if constexpr (CHAIN) RowStep<K>::chain(V, P[r & 3], cin, cout);
                else RowStep<K>::plain(V, P[r & 3]);
            }
        }
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}

// K = 10 with packed slots: words 0-3 [lane][4] at 0, words 4-7 [lane][4] at
// 512, words 8-9 [lane][2] at 1024 (code stride 1280 as [lane][10]) -> three
// loads per row (LDS.128, LDS.128, LDS.64) instead of five LDS.64.
template <bool CHAIN, int S>
__global__ void __launch_bounds__(32) sweep_bench5(const uint8_t* rows, int steps, uint32_t* out) {
    constexpr int K = 10;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = 1280;
    for (int b = lane; b < 256; b += 32) smem[b] = (b >= 65 && b < 65 + kSigma - 1) ? uint8_t(b - 64) : 0;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t map_a = sbase;
    const uint32_t pm_a = sbase + kMapBytes + lane * 16u;
    const uint32_t pm_b = sbase + kMapBytes + 1024u + lane * 8u;
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 cur = ldg_l2pf(rp);
    uint32_t cout = 0;
    for (int t = 0; t < steps - 1; ++t) {
        const uint4 nxt = ldg_l2pf(rp + t + 1);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        uint32_t wlo = cur.x, whi = cur.y;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            uint32_t code[8];
            code[0] = lds_u8(byte_addr<0>(wlo, map_a)) * cs; code[1] = lds_u8(byte_addr<1>(wlo, map_a)) * cs;
            code[2] = lds_u8(byte_addr<2>(wlo, map_a)) * cs; code[3] = lds_u8(byte_addr<3>(wlo, map_a)) * cs;
            code[4] = lds_u8(byte_addr<0>(whi, map_a)) * cs; code[5] = lds_u8(byte_addr<1>(whi, map_a)) * cs;
            code[6] = lds_u8(byte_addr<2>(whi, map_a)) * cs; code[7] = lds_u8(byte_addr<3>(whi, map_a)) * cs;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                uint32_t P[K];
                const uint4 p0 = lds_v4(code[r] + pm_a);
                const uint4 p1 = lds_v4<512>(code[r] + pm_a);
                const uint2 p2 = lds_v2(code[r] + pm_b);
                P[0] = p0.x; P[1] = p0.y; P[2] = p0.z; P[3] = p0.w;
                P[4] = p1.x; P[5] = p1.y; P[6] = p1.z; P[7] = p1.w;
                P[8] = p2.x; P[9] = p2.y;
                if constexpr (CHAIN) RowStep<K>::chain(V, P, cin, cout);
                else RowStep<K>::plain(V, P);
            }
            wlo = cur.z;
            whi = cur.w;
        }
        cur = nxt;
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}

// Range map (no map lookup): code = min(byte - lo, R - 1) by DP4A + a 16x2
// min (both FMA-pipe capable), offset = code * cs + lane base.
template <int K, int R>
__device__ __forceinline__ uint32_t range_off(uint32_t w, uint32_t neg_lo, uint32_t lim, uint32_t pm_a) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t t;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(w), "n"(1u << (8 * R)), "r"(neg_lo));
    t = __vminu2(t, lim);
    return t * cs + pm_a;
}

template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench6(const uint8_t* rows, int steps, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t pm_a = sbase + kMapBytes + PmLayout<K>::word_offset(lane, 0);
    const uint32_t neg_lo = 0u - 65u, lim = uint32_t(kSigma - 1);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 cur = ldg_l2pf(rp);
    uint32_t cout = 0;
    for (int t = 0; t < steps - 1; ++t) {
        const uint4 nxt = ldg_l2pf(rp + t + 1);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        uint32_t wlo = cur.x, whi = cur.y;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            uint32_t off[8];
            off[0] = range_off<K, 0>(wlo, neg_lo, lim, pm_a); off[1] = range_off<K, 1>(wlo, neg_lo, lim, pm_a);
            off[2] = range_off<K, 2>(wlo, neg_lo, lim, pm_a); off[3] = range_off<K, 3>(wlo, neg_lo, lim, pm_a);
            off[4] = range_off<K, 0>(whi, neg_lo, lim, pm_a); off[5] = range_off<K, 1>(whi, neg_lo, lim, pm_a);
            off[6] = range_off<K, 2>(whi, neg_lo, lim, pm_a); off[7] = range_off<K, 3>(whi, neg_lo, lim, pm_a);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                uint32_t P[K];
                load_pm_sh<K>(off[r], P);
                if constexpr (CHAIN) RowStep<K>::chain(V, P, cin, cout);
                else RowStep<K>::plain(V, P);
            }
            wlo = cur.z;
            whi = cur.w;
        }
        cur = nxt;
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}

// 16-row body per step (one head latency per 16 rows instead of per 8).
template <bool CHAIN, int K, int S, int AHEAD>
__global__ void __launch_bounds__(32) sweep_bench7(const uint8_t* rows, int steps, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t sbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(smem)));
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    for (int b = lane; b < 256; b += 32) smem[b] = (b >= 65 && b < 65 + kSigma - 1) ? uint8_t(b - 64) : 0;
    uint32_t x = 0x9e3779b9u * (blockIdx.x * 32 + lane + 1);
    for (uint32_t i = lane; i < kSigma * cs / 4; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem + kMapBytes)[i] = i < cs / 4 ? 0u : x;
    }
    __syncwarp();
    const uint32_t map_a = sbase;
    const uint32_t pm_a = sbase + kMapBytes + PmLayout<K>::word_offset(lane, 0);
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    const int s = int(lane) & (S - 1);
    const uint4* rp = reinterpret_cast<const uint4*>(rows) + size_t(blockIdx.x * 32 + lane) * steps;
    uint4 cur = ldg_l2pf(rp);
    uint32_t cout = 0;
    for (int t = 0; t < steps - 1; ++t) {
        const uint4 nxt = ldg_l2pf(rp + t + 1);
        uint32_t cin = 0;
        if constexpr (CHAIN) {
            cin = __shfl_up_sync(kFullMask, cout, 1, S);
            if (s == 0) cin = 0;
            cin <<= 16;
            cout = 0;
        }
        const uint32_t w[4] = {cur.x, cur.y, cur.z, cur.w};
        uint32_t off[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            uint32_t a;
            asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(w[r >> 2]), "r"(1u << (8 * (r & 3))), "r"(map_a));
            off[r] = lds_u8(a) * cs + pm_a;
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            uint32_t P[K];
            load_pm_sh<K>(off[r], P);
            if constexpr (CHAIN) RowStep<K>::chain(V, P, cin, cout);
            else RowStep<K>::plain(V, P);
        }
        cur = nxt;
    }
    uint32_t acc = cout;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= V[k];
    out[blockIdx.x * 32 + lane] = acc;
}

template <bool CHAIN, int K, int S, int AHEAD, int PIPE = 0>
void run(const uint8_t* rows, int steps, uint32_t* out, int sms, int warps_per_sm) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    const int smem = kMapBytes + kSigma * cs;
    auto kern = PIPE == 6 ? sweep_bench7<CHAIN, K, S, AHEAD> : PIPE == 5 ? sweep_bench6<CHAIN, K, S, AHEAD> : PIPE == 4 ? sweep_bench5<CHAIN, S> : PIPE == 3 ? sweep_bench4<CHAIN, K, S, AHEAD> : PIPE == 2 ? sweep_bench3<CHAIN, K, S, AHEAD> : PIPE ? sweep_bench2<CHAIN, K, S, AHEAD> : sweep_bench<CHAIN, K, S, AHEAD>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
    const int per_sm = warps_per_sm < occ ? warps_per_sm : occ;
    const int grid = sms * per_sm;
    kern<<<grid, 32, smem>>>(rows, steps, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, 32, smem>>>(rows, steps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double alu = double(grid) * (steps - AHEAD) * 16.0 * (3 * K + (CHAIN ? 1 : 0));
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%s K=%2d chain=%d S=%d ahead=%d warps/SM=%2d (occ %2d, smem %5d): %.3f ms, row-update ALU %.2f /clk/SM = %.1f%% of peak\n",
           PIPE == 6 ? "full16" : PIPE == 5 ? "range" : PIPE == 4 ? "slot3" : PIPE == 3 ? "regs " : PIPE == 2 ? "nomap" : PIPE ? "pipe" : "base", K, int(CHAIN), S, AHEAD, per_sm, occ, smem, ms, alu / cyc / sms, 100.0 * alu / cyc / sms / 2.0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int steps = 400;  // 6400 rows per lane
    const size_t max_grid = size_t(sms) * 16;
    std::vector<uint8_t> h(max_grid * 32 * steps * 16);
    uint32_t x = 12345;
    for (auto& b : h) { x ^= x << 13; x ^= x >> 17; x ^= x << 5; b = uint8_t(65 + x % 20); }
    uint8_t* d;
    uint32_t* out;
    cudaMalloc(&d, h.size());
    cudaMalloc(&out, max_grid * 32 * 4);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    for (int pipe = 0; pipe < 7; ++pipe) {
        if (pipe == 6) {
            run<true, 8, 2, 1, 6>(d, steps, out, sms, 8);
            run<true, 7, 2, 1, 6>(d, steps, out, sms, 8);
            run<true, 6, 4, 1, 6>(d, steps, out, sms, 8);
            run<true, 6, 2, 1, 6>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 6>(d, steps, out, sms, 8);
            run<true, 6, 2, 1, 0>(d, steps, out, sms, 8);
        } else if (pipe == 5) {
            run<false, 10, 1, 1, 5>(d, steps, out, sms, 8);
            run<true, 8, 2, 1, 5>(d, steps, out, sms, 8);
            run<true, 7, 2, 1, 5>(d, steps, out, sms, 8);
            run<true, 6, 4, 1, 5>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 5>(d, steps, out, sms, 8);
        } else if (pipe == 4) {
            run<false, 10, 1, 1, 4>(d, steps, out, sms, 8);
            run<true, 10, 2, 1, 4>(d, steps, out, sms, 8);
        } else if (pipe == 3) {
            run<false, 10, 1, 1, 3>(d, steps, out, sms, 8);
            run<false, 10, 1, 1, 3>(d, steps, out, sms, 16);
            run<true, 8, 2, 1, 3>(d, steps, out, sms, 8);
            run<true, 8, 2, 1, 3>(d, steps, out, sms, 16);
            run<true, 4, 2, 1, 3>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 3>(d, steps, out, sms, 16);
            run<false, 4, 1, 1, 3>(d, steps, out, sms, 8);
            run<false, 4, 1, 1, 3>(d, steps, out, sms, 16);
        } else if (pipe == 2) {
            run<false, 10, 1, 1, 2>(d, steps, out, sms, 8);
            run<true, 10, 2, 1, 2>(d, steps, out, sms, 8);
            run<true, 8, 2, 1, 2>(d, steps, out, sms, 8);
            run<true, 6, 4, 1, 2>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 2>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 2>(d, steps, out, sms, 12);
        } else if (pipe) {
            run<false, 10, 1, 1, 1>(d, steps, out, sms, 8);
            run<false, 9, 1, 1, 1>(d, steps, out, sms, 8);
            run<true, 10, 2, 1, 1>(d, steps, out, sms, 8);
            run<true, 8, 2, 1, 1>(d, steps, out, sms, 8);
            run<true, 7, 2, 1, 1>(d, steps, out, sms, 8);
            run<true, 6, 4, 1, 1>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 1>(d, steps, out, sms, 8);
            run<true, 4, 2, 1, 1>(d, steps, out, sms, 12);
        } else {
            run<false, 10, 1, 1>(d, steps, out, sms, 8);
            run<false, 9, 1, 1>(d, steps, out, sms, 8);
            run<true, 10, 2, 1>(d, steps, out, sms, 8);
            run<true, 8, 2, 1>(d, steps, out, sms, 8);
            run<true, 7, 2, 1>(d, steps, out, sms, 8);
            run<true, 6, 4, 1>(d, steps, out, sms, 8);
            run<true, 4, 2, 1>(d, steps, out, sms, 8);
            run<true, 4, 2, 1>(d, steps, out, sms, 12);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
