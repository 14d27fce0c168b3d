// probe.cu -- integer-pipe peak microbenchmark (the roofline denominator).
//
// MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks; the LCS fill is
// bound by the SM integer ALU pipe (LOP3 / IADD3), so bench.py measures that
// peak live with this kernel: every thread runs 8 independent chains of
// LOP3 (the ALU-pipe op class of the bit-parallel row step: LOP3 +
// IADD3.X + LOP3), enough ILP to keep the ALU pipe of every SM sub-partition busy.
#include <cstdint>
#include <cuda_runtime.h>

namespace wlcs {

constexpr int kProbeChains = 8;
constexpr int kProbeIters = 2048;

__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t seed, uint32_t* sink) {
    uint32_t a[kProbeChains], b[kProbeChains];
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) {
        a[c] = seed ^ (threadIdx.x * 0x9e3779b9u + c);
        b[c] = seed + c * 0x85ebca6bu + blockIdx.x;
    }
    for (int it = 0; it < kProbeIters; ++it) {
#pragma unroll
        for (int c = 0; c < kProbeChains; ++c) {
            // 2 ALU-pipe ops per chain per iteration.  Both are LOP3: a plain
            // add would be moved to the FMA pipe (IMAD.IADD) by ptxas, while
            // the fill's carry-chained IADD3.X cannot leave the ALU pipe.
            asm volatile("lop3.b32 %0, %0, %1, %2, 0xF4;" : "+r"(a[c]) : "r"(b[c]), "r"(seed));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(b[c]) : "r"(a[c]), "r"(seed));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c) acc ^= a[c] ^ b[c];
    if (acc == 0x12345678u) sink[0] = acc;  // keeps the chains alive
}

// Runs the probe `reps` times on the current device; returns the best
// sustained rate in int32 ops/s (warp lanes x instructions / second).
cudaError_t int_peak_probe(int reps, double* ops_per_s, uint32_t* scratch) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int_peak_kernel<<<blocks, threads>>>(1u, scratch);  // warm-up
    double best = 0;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        int_peak_kernel<<<blocks, threads>>>(uint32_t(r + 2), scratch);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(blocks) * threads * kProbeIters * kProbeChains * 2.0;
        const double rate = ops / (ms * 1e-3);
        if (rate > best) best = rate;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ops_per_s = best;
    return cudaGetLastError();
}

}  // namespace wlcs
