// sweep.cuh -- the per-lane row sweep shared by the batch and single-pair
// bit-parallel kernels.
//
// A lane owns K consecutive 32-bit words of the bit vector V (32*K columns)
// and streams the row string one 16-byte chunk (16 rows) per step.  Per row:
//   code = map[byte]           (LDS.U8, per-task byte -> dense code)
//   P    = PM[code][lane][0:K] (one LDS.32/64/128 or two LDS.128)
//   V    = row update          (rowstep.cuh: AND, IADD3.X, LOP3 per word)
// Shared-memory match-mask layout, chosen so every warp-wide PM load is
// bank-conflict free:
//   K <= 4 : [code][lane][K words]             code stride 128*K bytes
//   K  > 4 : [code][K/4 slot][lane][4 words]   code stride 1024 bytes
#pragma once

#include "rowstep.cuh"
#include "wlcs_common.cuh"

namespace wlcs {

template <int K>
struct PmLayout {
    static constexpr int kWide = K > 4;
    static constexpr uint32_t code_stride = kWide ? 1024u : 128u * uint32_t(K == 3 ? 4 : K);
    static constexpr uint32_t lane_stride = kWide ? 16u : 4u * uint32_t(K == 3 ? 4 : K);
    // byte offset of word k of `lane` inside one code row
    __device__ __forceinline__ static uint32_t word_offset(uint32_t lane, int k) {
        return kWide ? uint32_t(k >> 2) * 512u + lane * 16u + uint32_t(k & 3) * 4u
                     : lane * lane_stride + uint32_t(k) * 4u;
    }
};

template <int K>
__device__ __forceinline__ void load_pm(const uint8_t* pm, uint32_t off, uint32_t* P) {
    if constexpr (K >= 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(pm + off);
        P[0] = a.x; P[1] = a.y; P[2] = a.z; P[3] = a.w;
        if constexpr (K == 8 || K == 7) {
            const uint4 b = *reinterpret_cast<const uint4*>(pm + off + 512);
            P[4] = b.x; P[5] = b.y; P[6] = b.z;
            if constexpr (K == 8) P[7] = b.w;
        } else if constexpr (K == 6) {
            const uint2 b = *reinterpret_cast<const uint2*>(pm + off + 512);
            P[4] = b.x; P[5] = b.y;
        } else if constexpr (K == 5) {
            P[4] = *reinterpret_cast<const uint32_t*>(pm + off + 512);
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

// Process the 16 rows of one chunk.  `full` = all 16 rows valid for every
// lane of the warp (warp-uniform): the fast path is fully unrolled; the
// masked path treats invalid rows as identity rows (code 0 = zero masks).
// hook(r, valid, V) runs after each row (used to store bit rows).
// MapT is uint8_t (batch: <= 255 codes) or uint16_t (single pair: up to 257).
template <bool CHAIN, int K, typename MapT, typename Hook>
__device__ __forceinline__ void sweep_chunk(bool full, uint32_t* V, const MapT* map,
                                            const uint8_t* pm, uint32_t lane_off,
                                            const uint8_t* chunk_ptr, const uint8_t* alloc_lo,
                                            const uint8_t* alloc_hi, uint32_t vm, uint32_t& cin,
                                            uint32_t& cout, const Hook& hook) {
    constexpr uint32_t cs = PmLayout<K>::code_stride;
    if (full) {
        const uint4 c = __ldg(reinterpret_cast<const uint4*>(chunk_ptr));
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t code = map[chunk_byte(c, r)];
            row_update<CHAIN, K>(V, pm, code * cs + lane_off, cin, cout);
            hook(r, true, V);
        }
    } else {
        const uint4 c = vm ? load_chunk16(chunk_ptr, alloc_lo, alloc_hi) : make_uint4(0, 0, 0, 0);
#pragma unroll 1
        for (int r = 0; r < 16; ++r) {
            const bool valid = (vm >> r) & 1u;
            const uint32_t code = valid ? uint32_t(map[chunk_byte(c, r)]) : 0u;
            row_update<CHAIN, K>(V, pm, code * cs + lane_off, cin, cout);
            hook(r, valid, V);
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

}  // namespace wlcs
