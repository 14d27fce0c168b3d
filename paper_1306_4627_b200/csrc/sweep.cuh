// sweep.cuh -- the per-lane row sweep shared by the batch and single-pair
// bit-parallel kernels.
//
// A lane owns K consecutive 32-bit words of the bit vector V (32*K columns)
// and streams the row string one 16-byte chunk (16 rows) per step.  Per row:
//   code = map[byte]           (DP4A address + LDS.U8, per-task byte -> dense code)
//   P    = PM[code][lane][0:K] (one LDS.32/64/128 or two LDS.128)
//   V    = row update          (rowstep.cuh: AND, IADD3.X, LOP3 per word)
// Shared-memory match-mask layout, chosen so every warp-wide PM load is
// bank-conflict free:
//   K <= 4 : [code][lane][K words]               code stride 128*K bytes
//   K 9-10 : [code][lane][10 words]              code stride 1280 bytes
//            (40-byte lane stride: five LDS.64 per row, conflict-free; 17%
//            less than the 3-slot layout, which lets kmax = 10 run 8 warps
//            per SM in 26.25 KB of masks)
//   other K > 4 : [code][ceil(K/4) slot][lane][4 words] code stride 512*ceil(K/4)
#pragma once

#include "rowstep.cuh"
#include "wlcs_common.cuh"

namespace wlcs {

// Words per lane row of the non-slotted layouts (K = 3 and 9 are padded).
__host__ __device__ constexpr uint32_t pm_lane_words(int K) {
    return K == 3 ? 4u : (K == 9 || K == 10) ? 10u : uint32_t(K);
}
__host__ __device__ constexpr bool pm_slotted(int K) { return K > 4 && K != 9 && K != 10; }

template <int K>
struct PmLayout {
    static constexpr int kWide = pm_slotted(K);
    static constexpr uint32_t code_stride =
        kWide ? 512u * uint32_t((K + 3) / 4) : 128u * pm_lane_words(K);
    static constexpr uint32_t lane_stride = kWide ? 16u : 4u * pm_lane_words(K);
    // byte offset of word k of `lane` inside one code row
    __device__ __forceinline__ static uint32_t word_offset(uint32_t lane, int k) {
        return kWide ? uint32_t(k >> 2) * 512u + lane * 16u + uint32_t(k & 3) * 4u
                     : lane * lane_stride + uint32_t(k) * 4u;
    }
};

// Slot i (words 4i .. 4i+3) of a wide row sits at byte offset 512*i.
template <int K>
__device__ __forceinline__ void load_pm(const uint8_t* pm, uint32_t off, uint32_t* P) {
    if constexpr (K == 9 || K == 10) {
#pragma unroll
        for (int i = 0; 2 * i < K; ++i) {
            if (2 * i + 1 < K) {
                const uint2 a = *reinterpret_cast<const uint2*>(pm + off + 8 * i);
                P[2 * i] = a.x; P[2 * i + 1] = a.y;
            } else {
                P[2 * i] = *reinterpret_cast<const uint32_t*>(pm + off + 8 * i);
            }
        }
    } else if constexpr (K >= 4) {
#pragma unroll
        for (int i = 0; 4 * i < K; ++i) {
            const uint8_t* q = pm + off + 512 * i;
            const int n = K - 4 * i < 4 ? K - 4 * i : 4;
            if (n == 4) {
                const uint4 a = *reinterpret_cast<const uint4*>(q);
                P[4 * i] = a.x; P[4 * i + 1] = a.y; P[4 * i + 2] = a.z; P[4 * i + 3] = a.w;
            } else if (n >= 2) {
                const uint2 a = *reinterpret_cast<const uint2*>(q);
                P[4 * i] = a.x; P[4 * i + 1] = a.y;
                if (n == 3) P[4 * i + 2] = *reinterpret_cast<const uint32_t*>(q + 8);
            } else {
                P[4 * i] = *reinterpret_cast<const uint32_t*>(q);
            }
        }
    } else if constexpr (K == 3) {
        const uint2 a = *reinterpret_cast<const uint2*>(pm + off);
        P[0] = a.x; P[1] = a.y;
        P[2] = *reinterpret_cast<const uint32_t*>(pm + off + 8);
    } else if constexpr (K == 2) {
        const uint2 a = *reinterpret_cast<const uint2*>(pm + off);
        P[0] = a.x; P[1] = a.y;
    } else {
        P[0] = *reinterpret_cast<const uint32_t*>(pm + off);
    }
}

template <bool CHAIN, int K>
__device__ __forceinline__ void row_update(uint32_t* V, const uint8_t* pm, uint32_t off,
                                           uint32_t& cin, uint32_t& cout) {
    uint32_t P[K];
    load_pm<K>(pm, off, P);
    if constexpr (CHAIN) {
        RowStep<K>::chain(V, P, cin, cout);
    } else {
        RowStep<K>::plain(V, P);
    }
}

struct NoRowHook {
    __device__ __forceinline__ void operator()(int, bool, const uint32_t*) const {}
};

// A step processes the 16 rows of one chunk in two parts so that only the
// small part has a masked variant (keeps the hot code small for the I-cache):
//  (a) offsets: off[r] = PM byte offset of row r's match masks for this lane
//      (code * code_stride + lane_off; code 0 = all-zero masks = identity row)
//  (b) rows:    16 unrolled row updates reading P from off[r].
template <typename MapT>
__device__ __forceinline__ void chunk_offsets(const uint4& c, const MapT* map, uint32_t cs,
                                              uint32_t lane_off, uint32_t* off) {
#pragma unroll
    for (int r = 0; r < 16; ++r) off[r] = uint32_t(map[chunk_byte(c, r)]) * cs + lane_off;
}

// Rows whose bit in vm is clear become identity rows.
template <typename MapT>
__device__ __forceinline__ void chunk_offsets_masked(const uint4& c, uint32_t vm, const MapT* map,
                                                     uint32_t cs, uint32_t lane_off,
                                                     uint32_t* off) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t code = ((vm >> r) & 1u) ? uint32_t(map[chunk_byte(c, r)]) : 0u;
        off[r] = code * cs + lane_off;
    }
}

// Replaces the bytes of invalid rows by `zrep` (a byte value absent from the
// task's column alphabet, replicated x4) so that they map to code 0.
__device__ __forceinline__ uint4 sanitize_chunk(uint4 c, uint32_t vm, uint32_t zrep) {
    uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m4 = (vm >> (4 * i)) & 0xfu;
        const uint32_t keep = ((m4 * 0x00204081u) & 0x01010101u) * 0xffu;  // bit b -> byte b
        w[i] = (w[i] & keep) | (zrep & ~keep);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}


// hook(r, valid, V) runs after each row (used to store bit rows).
template <bool CHAIN, int K, typename Hook>
__device__ __forceinline__ void rows16(uint32_t* V, const uint8_t* pm, const uint32_t* off,
                                       uint32_t vm, uint32_t& cin, uint32_t& cout,
                                       const Hook& hook) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        row_update<CHAIN, K>(V, pm, off[r], cin, cout);
        hook(r, ((vm >> r) & 1u) != 0u, V);
    }
}

// Half-chunk variant used by the batch sweep: rows 8h..8h+7 of the chunk
// (bytes in lo = word 2h, hi = word 2h+1), emitted once inside a rolled loop
// over the two halves so each sweep instance stays small in the I-cache.
template <bool CHAIN, int K, typename MapT>
__device__ __forceinline__ void rows8(uint32_t* V, const MapT* map, const uint8_t* pm,
                                      uint32_t cs, uint32_t lane_off, uint32_t lo, uint32_t hi,
                                      uint32_t& cin, uint32_t& cout) {
    uint32_t off[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
        off[r] = uint32_t(map[__byte_perm(r < 4 ? lo : hi, 0u, 0x4440u | uint32_t(r & 3))]) * cs +
                 lane_off;
#pragma unroll
    for (int r = 0; r < 8; ++r) row_update<CHAIN, K>(V, pm, off[r], cin, cout);
}

// The 16-byte chunk `ch` of a lane's row string (chunk addresses are 16-byte
// aligned by construction).  The common case is one unconditional LDG.128 the
// compiler can hoist a whole step ahead of its use; straddling chunks take a
// warp-uniform slow path.
__device__ __forceinline__ uint4 fetch_chunk(const uint8_t* rstart, int ch, uint32_t vm,
                                             const uint8_t* alloc_lo, const uint8_t* alloc_hi,
                                             const uint4* safe) {
    const uint8_t* p = rstart + int64_t(ch) * 16;
    bool slow;
    uint4 c = fetch_chunk_fast(p, vm, alloc_lo, alloc_hi, safe, slow);
    if (__any_sync(kFullMask, slow)) {
        if (slow) c = load_chunk16(p, alloc_lo, alloc_hi);
    }
    return c;
}

// ---------------------------------------------------------------------------
// Explicit 32-bit shared-memory addressing.  With generic pointers into the
// dynamic shared window the compiler re-derives the window base
// (S2R SR_CgaCtaId + LEA) inside loops; these keep one base in a register.
// The asm is volatile so loads stay ordered after the stores / __syncwarp()
// of the mask build.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
template <int OFF = 0>
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF = 0>
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+%3];" : "=r"(v.x), "=r"(v.y) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF = 0>
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(uint16_t(v)) : "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// load_pm over a 32-bit shared address (same layouts as load_pm).
template <int K, int I>
__device__ __forceinline__ void load_slot_sh(uint32_t a, uint32_t* P) {
    constexpr int n = K - 4 * I < 4 ? K - 4 * I : 4;
    if constexpr (n == 4) {
        const uint4 x = lds_v4<512 * I>(a);
        P[4 * I] = x.x; P[4 * I + 1] = x.y; P[4 * I + 2] = x.z; P[4 * I + 3] = x.w;
    } else if constexpr (n >= 2) {
        const uint2 x = lds_v2<512 * I>(a);
        P[4 * I] = x.x; P[4 * I + 1] = x.y;
        if constexpr (n == 3) P[4 * I + 2] = lds_u32<512 * I + 8>(a);
    } else {
        P[4 * I] = lds_u32<512 * I>(a);
    }
}

// load_pm over a 32-bit shared address (same layouts as load_pm).
template <int K, int I>
__device__ __forceinline__ void load_pair_sh(uint32_t a, uint32_t* P) {
    if constexpr (2 * I + 1 < K) {
        const uint2 x = lds_v2<8 * I>(a);
        P[2 * I] = x.x; P[2 * I + 1] = x.y;
    } else if constexpr (2 * I < K) {
        P[2 * I] = lds_u32<8 * I>(a);
    }
}

template <int K>
__device__ __forceinline__ void load_pm_sh(uint32_t a, uint32_t* P) {
    if constexpr (K == 9 || K == 10) {
        load_pair_sh<K, 0>(a, P);
        load_pair_sh<K, 1>(a, P);
        load_pair_sh<K, 2>(a, P);
        load_pair_sh<K, 3>(a, P);
        load_pair_sh<K, 4>(a, P);
    } else if constexpr (K >= 4) {
        load_slot_sh<K, 0>(a, P);
        if constexpr (K > 4) load_slot_sh<K, 1>(a, P);
        if constexpr (K > 8) load_slot_sh<K, 2>(a, P);
    } else if constexpr (K == 3) {
        const uint2 x = lds_v2(a);
        P[0] = x.x; P[1] = x.y;
        P[2] = lds_u32<8>(a);
    } else if constexpr (K == 2) {
        const uint2 x = lds_v2(a);
        P[0] = x.x; P[1] = x.y;
    } else {
        P[0] = lds_u32(a);
    }
}

// map_a + byte r of w as ONE instruction on the FMA pipe: dp4a(w, 1 << 8r,
// map_a) = byte_r(w) * 1 + map_a.  The row update saturates the ALU pipe;
// PRMT (byte extract) would be an ALU op per row plus an add
// (tools/micro/byte_extract.cu: DP4A issues on the FMA pipe at the full
// 64 ops/clk/SM, 4.7-cycle latency, like PRMT).
template <int R>
__device__ __forceinline__ uint32_t byte_addr(uint32_t w, uint32_t base) {
    uint32_t a;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(w), "n"(1u << (8 * R)), "r"(base));
    return a;
}

// rows8 over shared addresses: map_a = byte -> code table, pm_a = this
// lane's word 0 of code 0.
template <bool CHAIN, int K>
__device__ __forceinline__ void rows8_sh(uint32_t* V, uint32_t map_a, uint32_t pm_a, uint32_t lo,
                                         uint32_t hi, uint32_t& cin, uint32_t& cout) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    uint32_t off[8];
    off[0] = lds_u8(byte_addr<0>(lo, map_a)) * cs + pm_a;
    off[1] = lds_u8(byte_addr<1>(lo, map_a)) * cs + pm_a;
    off[2] = lds_u8(byte_addr<2>(lo, map_a)) * cs + pm_a;
    off[3] = lds_u8(byte_addr<3>(lo, map_a)) * cs + pm_a;
    off[4] = lds_u8(byte_addr<0>(hi, map_a)) * cs + pm_a;
    off[5] = lds_u8(byte_addr<1>(hi, map_a)) * cs + pm_a;
    off[6] = lds_u8(byte_addr<2>(hi, map_a)) * cs + pm_a;
    off[7] = lds_u8(byte_addr<3>(hi, map_a)) * cs + pm_a;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        uint32_t P[K];
        load_pm_sh<K>(off[r], P);
        if constexpr (CHAIN) {
            RowStep<K>::chain(V, P, cin, cout);
        } else {
            RowStep<K>::plain(V, P);
        }
    }
}

// Zero bits of the lane's K words below global column `cols`; `word0` is the
// global index of the lane's first word.
template <int K>
__device__ __forceinline__ int lane_zero_count(const uint32_t* V, int64_t word0, int64_t cols) {
    int zeros = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t bits = cols - 32 * (word0 + k);
        if (bits >= 32) zeros += __popc(~V[k]);
        else if (bits > 0) zeros += __popc(~V[k] & ((1u << bits) - 1u));
    }
    return zeros;
}

// ---------------------------------------------------------------------------
// Match-mask build helpers (batch kernels): 32 column bytes -> 8 bit-planes.
// Each lane owns 32-column words of its pair's column string; per word it
// (1) realigns the 32 column bytes out of 16-byte aligned chunks (funnel
// shifts), (2) turns them into 8 bit-planes (plane b, bit j = bit b of
// column j's byte).  A code's match mask is then the AND over the planes of
// "plane == bit of the code's byte value".
//
// bit_planes8: 16 PRMT regroup the bytes by column stride 8 (word i holds
// columns i, i+8, i+16, i+24 as its bytes 0..3), then three delta swaps
// exchange the word-index bits (i2 i1 i0) with the in-byte bit index
// (b2 b1 b0): afterwards word b holds bit b of column 8k + i at position
// 8k + i.  76 ALU ops per word (the 8x8 transposes were ~110).
__device__ __forceinline__ void delta_swap(uint32_t& x, uint32_t& y, int d, uint32_t keep) {
    const uint32_t t = ((x >> d) ^ y) & keep;  // keep = positions whose bit s is 0
    y ^= t;
    x ^= t << d;
}

__device__ __forceinline__ void bit_planes8(const uint32_t* w, uint32_t* P) {
    uint32_t g[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int m = 0; m < 4; m += 2) {
            // bytes m and m+1 of w[h], w[h+2] / w[h+4], w[h+6]
            const uint32_t sel = uint32_t(m) | uint32_t(4 + m) << 4 | uint32_t(m + 1) << 8 |
                                 uint32_t(5 + m) << 12;
            const uint32_t t1 = __byte_perm(w[h], w[h + 2], sel);
            const uint32_t t2 = __byte_perm(w[h + 4], w[h + 6], sel);
            g[4 * h + m] = __byte_perm(t1, t2, 0x5410);      // columns c, c+8, c+16, c+24
            g[4 * h + m + 1] = __byte_perm(t1, t2, 0x7632);  // c = 4h + m (+1)
        }
    }
    // word index i = 4h + m; stage s pairs words i and i + 2^s
#pragma unroll
    for (int i = 0; i < 8; i += 2) delta_swap(g[i], g[i + 1], 1, 0x55555555u);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
        delta_swap(g[i], g[i + 2], 2, 0x33333333u);
        delta_swap(g[i + 1], g[i + 3], 2, 0x33333333u);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) delta_swap(g[i], g[i + 4], 4, 0x0f0f0f0fu);
#pragma unroll
    for (int b = 0; b < 8; ++b) P[b] = g[b];
}

// The 32 column bytes of the lane's word k, realigned out of the 16-byte
// aligned chunks 2k, 2k+1, 2k+2 (q = a_c / 4, fs = 8 * (a_c % 4)): word i is
// the funnel shift of W[i + q] and W[i + q + 1]; W[i + q] is picked with two
// selects (odd q, then q >= 2).
__device__ __forceinline__ void word_bytes(const uint4& c0, const uint4& c1, const uint4& c2, int q,
                                           uint32_t fs, uint32_t* w) {
    const uint32_t W[12] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x, c2.y, c2.z, c2.w};
    uint32_t a[11];
#pragma unroll
    for (int i = 0; i < 11; ++i) a[i] = (q & 1) ? W[i + 1] : W[i];
    uint32_t lo[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) lo[i] = (q & 2) ? a[i + 2] : a[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = __funnelshift_r(lo[i], lo[i + 1], fs);
}

}  // namespace wlcs
