// wlcs_common.cuh -- shared device helpers for the B200 LCS kernels.
//
// Bit layout used by every bit-parallel kernel (Allison-Dix / Hyyro):
//   column j (1-based, the "child" / column string) <-> bit (j-1) of V,
//   word w = (j-1) / 32, bit (j-1) % 32; carries run toward higher columns.
//   V_0 = all ones; row i: U = V & PM[x_i]; V' = (V + U) | (V & ~PM[x_i]).
//   DP value c[i][j] = popcount(~V_i & ((1 << j) - 1)),
//   so LCS = number of zero bits of V_M below column N.
// This reproduces lcs_cell (proj/include/wavelcs/cell.hpp:30-38) value by
// value; tests/test_oracle.py checks the identity against the reference.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace wlcs {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kRowsPerStep = 16;  // one 16-byte chunk of the row string per step

// 16-byte read-only load that also asks L2 to fetch the surrounding 256-byte
// block (ld.global.nc.L2::256B): a lane streaming its own string one chunk
// per step gets the next 15 chunks staged in L2 by the first miss, so the
// one-step-ahead register prefetch then hits L2 instead of HBM.
__device__ __forceinline__ uint4 ldg_l2pf(const uint4* p) {
    uint4 v;
    asm("ld.global.nc.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p));
    return v;
}

// Byte-wise gather of a chunk that straddles the allocation end (rare; kept
// out of line so the callers' hot loops stay small).
static __device__ __noinline__ uint4 load_chunk16_slow(const uint8_t* p, const uint8_t* alloc_lo,
                                                const uint8_t* alloc_hi) {
    uint64_t lo = 0, hi = 0;
#pragma unroll 1
    for (int b = 0; b < 16; ++b) {
        const uint8_t* q = p + b;
        if (q >= alloc_lo && q < alloc_hi) {
            const uint64_t v = __ldg(q);
            if (b < 8) lo |= v << (8 * b);
            else hi |= v << (8 * (b - 8));
        }
    }
    return make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32));
}

// 16 bytes of a string starting at the 16-byte-aligned address `p`.
// Bytes outside [lo, hi) of the allocation are never touched: when the chunk
// straddles the allocation end the valid bytes are gathered one by one.
__device__ __forceinline__ uint4 load_chunk16(const uint8_t* p, const uint8_t* alloc_lo,
                                              const uint8_t* alloc_hi) {
    if (p >= alloc_lo && p + 16 <= alloc_hi) {
        return __ldg(reinterpret_cast<const uint4*>(p));
    }
    return load_chunk16_slow(p, alloc_lo, alloc_hi);
}

// Byte r (0..15) of a 16-byte chunk; r is a compile-time constant in the
// unrolled sweeps, so this is one PRMT.
__device__ __forceinline__ uint32_t chunk_byte(const uint4& c, int r) {
    const uint32_t w = (r < 4) ? c.x : (r < 8) ? c.y : (r < 12) ? c.z : c.w;
    return __byte_perm(w, 0u, 0x4440u | uint32_t(r & 3));
}

// Valid-row mask of a 16-row chunk whose first row has string index `lo`
// against a string of `len` symbols (bit r set <=> 0 <= lo + r < len).
__device__ __forceinline__ uint32_t chunk_valid_mask(int64_t lo, int64_t len) {
    int64_t b = lo < 0 ? -lo : 0;
    int64_t e = len - lo;
    if (b > 16) b = 16;
    if (e > 16) e = 16;
    if (e <= b) return 0u;
    return ((1u << e) - 1u) & ~((1u << b) - 1u);
}

// 32-bit variant for in-warp ranges (lo may be negative).
__device__ __forceinline__ uint32_t valid_mask16(int lo, int len) {
    int b = -lo;
    b = b < 0 ? 0 : (b > 16 ? 16 : b);
    int e = len - lo;
    e = e < 0 ? 0 : (e > 16 ? 16 : e);
    return e <= b ? 0u : ((1u << e) - 1u) & ~((1u << b) - 1u);
}

// One unconditional, hoistable 16-byte load for a chunk that holds valid
// bytes (vm != 0) and lies inside [alloc_lo, alloc_hi); any other chunk
// reads the 16-byte zero block `safe` instead.  `slow` flags chunks that hold
// valid bytes but straddle the allocation end: the caller re-reads those with
// load_chunk16 (rare: only the last string of a buffer).
__device__ __forceinline__ uint4 fetch_chunk_fast(const uint8_t* p, uint32_t vm,
                                                  const uint8_t* alloc_lo,
                                                  const uint8_t* alloc_hi, const uint4* safe,
                                                  bool& slow) {
    const bool inb = p >= alloc_lo && p + 16 <= alloc_hi;
    slow = vm != 0u && !inb;
    const uint4* src = (vm != 0u && inb) ? reinterpret_cast<const uint4*>(p) : safe;
    return ldg_l2pf(src);
}

__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFullMask, v, o));
    return v;
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

// gpu-scope release store / acquire load for inter-CTA flag protocols.
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace wlcs
