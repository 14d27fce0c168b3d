// Microbenchmark: throughput of the bit-parallel row update per 32-cell word
// on sm_100a, in three instruction mixes:
//   0 = ALU only:  AND, IADD3.X (carry chain), LOP3           (3 ALU)
//   1 = FMA adds:  AND, 2 x IMAD.WIDE.U32 (sum + carry-out in the high
//                  word, then + carry-in), LOP3                (2 ALU + 2 FMA)
//   2 = mixed:     words [0, K/2) as 1, [K/2, K) as 0
// Many warps per SM, masks from shared memory as in the real sweep.  Prints
// word-rows per clock per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int K, int MODE>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int rows, uint32_t one) {
    __shared__ uint32_t pm[4][K][256];
    for (int i = threadIdx.x; i < 4 * K * 256; i += blockDim.x) (&pm[0][0][0])[i] = i * 2654435761u;
    __syncthreads();
    uint32_t V[K];
#pragma unroll
    for (int k = 0; k < K; ++k) V[k] = 0xffffffffu;
    uint32_t code = threadIdx.x;
    for (int r = 0; r < rows; ++r) {
        code = code * 1664525u + 1013904223u;
        const uint32_t c = (code >> 30);
        uint32_t P[K];
#pragma unroll
        for (int k = 0; k < K; ++k) P[k] = pm[c][k][threadIdx.x];
        if (MODE == 0) {
            uint32_t cy = 0;
            asm volatile("add.cc.u32 %0, %0, 0;" : "+r"(cy));  // clear CC
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t u, s;
                asm("and.b32 %0, %1, %2;" : "=r"(u) : "r"(V[k]), "r"(P[k]));
                asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(s) : "r"(V[k]), "r"(u));
                asm("lop3.b32 %0, %1, %2, %3, 0xF4;" : "=r"(V[k]) : "r"(s), "r"(V[k]), "r"(P[k]));
            }
        } else {
            constexpr int KF = MODE == 1 ? K : K / 2;
            uint32_t cin = 0;
#pragma unroll
            for (int k = 0; k < KF; ++k) {
                uint32_t u;
                asm("and.b32 %0, %1, %2;" : "=r"(u) : "r"(V[k]), "r"(P[k]));
                uint64_t w = uint64_t(u);
                uint64_t r1, r2;
                asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r1) : "r"(V[k]), "r"(one), "l"(w));
                asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r2) : "r"(cin), "r"(one), "l"(r1));
                const uint32_t s = uint32_t(r2);
                cin = uint32_t(r2 >> 32);
                asm("lop3.b32 %0, %1, %2, %3, 0xF4;" : "=r"(V[k]) : "r"(s), "r"(V[k]), "r"(P[k]));
            }
            if (MODE == 2) {
                asm volatile("add.cc.u32 %0, %0, 0xffffffff;" : "+r"(cin));  // CC = cin
#pragma unroll
                for (int k = KF; k < K; ++k) {
                    uint32_t u, s;
                    asm("and.b32 %0, %1, %2;" : "=r"(u) : "r"(V[k]), "r"(P[k]));
                    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(s) : "r"(V[k]), "r"(u));
                    asm("lop3.b32 %0, %1, %2, %3, 0xF4;" : "=r"(V[k]) : "r"(s), "r"(V[k]), "r"(P[k]));
                }
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) x ^= V[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int K, int MODE>
void run(int sms, int blocks_per_sm) {
    uint32_t* out;
    cudaMalloc(&out, size_t(sms) * blocks_per_sm * 256 * 4);
    const int rows = 4096;
    bench<K, MODE><<<sms * blocks_per_sm, 256>>>(out, rows, 1u);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<K, MODE><<<sms * blocks_per_sm, 256>>>(out, rows, 1u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double wordrows = double(sms) * blocks_per_sm * 256 * rows * K;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("K=%2d mode=%d warps/SM=%2d: %.1f word-rows/clk/SM  (%.0f GCUPS at %d MHz; ALU-only roofline 21.3)\n", K, MODE,
           blocks_per_sm * 8, wordrows / cyc / sms, wordrows * 32 / (ms * 1e-3) / 1e9, clk / 1000);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {1, 2}) {
        run<8, 0>(sms, bps); run<8, 1>(sms, bps); run<8, 2>(sms, bps);
        run<12, 0>(sms, bps); run<12, 1>(sms, bps); run<12, 2>(sms, bps);
    }
    return 0;
}
