// Microbenchmark: which pipe extracts a byte of a register on sm_100a.
// The batch sweep turns each row byte into a shared-memory address once per
// row; PRMT does it on the ALU pipe, which the row update saturates.  Checks
// whether DP4A (byte_r(w) * 1 + base, one instruction) issues on another pipe:
// a 1:1 mix with LOP3 at ~2x the LOP3-only op rate means it does.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o byte_extract byte_extract.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[CH], uint32_t a, uint32_t b) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
        if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, 0x4441;" : "+r"(x[c]) : "r"(a));
        if (OP == 2) asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        if (OP == 4) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("prmt.b32 %0, %0, %1, 0x4441;" : "+r"(x[c]) : "r"(a));
        }
        if (OP == 5) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        }
        if (OP == 6) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        }
        if (OP == 7) {  // 2 LOP3 + 1 DP4A
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x69;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        }
        if (OP == 8) {  // LOP3 + DP4A + IMAD (a row's extraction + address on the FMA side)
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        }
        if (OP == 9) {  // 3 LOP3 + 1 DP4A (ratio of a K=1 row)
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x69;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int iters, uint32_t a, uint32_t b) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 7u + c;
    for (int i = 0; i < iters; ++i) step<OP>(x, a + i, b);
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one dependent chain per thread, one warp per SM sub-partition: latency
template <int OP>
__global__ void __launch_bounds__(32) lat(uint32_t* out, int iters, uint32_t a, uint32_t b) {
    uint32_t x = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, 0x4441;" : "+r"(x) : "r"(a));
        if (OP == 2) asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
        if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(a), "r"(b));
        if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(a), "r"(b));
    }
    out[threadIdx.x] = x;
}

template <int OP>
void run(const char* name, int per_step, int sms) {
    uint32_t* out;
    const int bps = 2;
    cudaMalloc(&out, size_t(sms) * bps * 256 * 4);
    const int iters = 1 << 14;
    bench<OP><<<sms * bps, 256>>>(out, iters, 3u, 5u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<OP><<<sms * bps, 256>>>(out, iters, 3u, 5u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = double(sms) * bps * 256 * iters * CH * per_step;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-34s %6.1f thread-ops/clk/SM\n", name, ops / cyc / sms);
    cudaFree(out);
}

template <int OP>
void run_lat(const char* name) {
    uint32_t* out;
    cudaMalloc(&out, 32 * 4);
    const int iters = 1 << 16;
    lat<OP><<<1, 32>>>(out, iters, 3u, 5u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    lat<OP><<<1, 32>>>(out, iters, 3u, 5u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-34s %5.2f cycles (dependent chain, incl. loop)\n", name,
           ms * 1e-3 * clk * 1e3 / iters);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("LOP3", 1, sms);
    run<1>("PRMT", 1, sms);
    run<2>("DP4A", 1, sms);
    run<3>("IMAD", 1, sms);
    run<4>("LOP3 + PRMT", 2, sms);
    run<5>("LOP3 + DP4A", 2, sms);
    run<6>("LOP3 + IMAD", 2, sms);
    run<7>("2 LOP3 + DP4A", 3, sms);
    run<8>("LOP3 + DP4A + IMAD", 3, sms);
    run<9>("3 LOP3 + DP4A", 4, sms);
    run_lat<0>("LOP3 latency");
    run_lat<1>("PRMT latency");
    run_lat<2>("DP4A latency");
    run_lat<3>("IMAD latency");
    return 0;
}
