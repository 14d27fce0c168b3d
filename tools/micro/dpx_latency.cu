// Microbenchmark: dependent-chain latency (clocks per instruction) of the
// DPX min/max instructions on sm_100a, one warp, one chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dpx_latency dpx_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(uint32_t* out, uint32_t a, uint32_t b, long long* cyc) {
    uint32_t x = threadIdx.x;
    const int N = 4096;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(a), "r"(b));
        if (OP == 1) x = __vimax3_u16x2(x, a, b);
        if (OP == 2) x = __vmaxu2(x, a);
        if (OP == 3) x = __viaddmax_u16x2(x, a, b);
        if (OP == 4) x = __vimax3_s32(x, a, b);
        if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(a));
        if (OP == 6) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 31) & 31);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}

template <int OP>
void run(const char* name) {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 128);
    cudaMalloc(&cyc, 8);
    lat<OP><<<1, 32>>>(out, 3u, 5u, cyc);
    lat<OP><<<1, 32>>>(out, 3u, 5u, cyc);
    long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-18s %5.1f clocks\n", name, double(h) / 4096);
}

int main() {
    run<0>("LOP3");
    run<1>("VIMNMX3.U16x2");
    run<2>("VIMNMX.U16x2");
    run<3>("VIADDMNMX.U16x2");
    run<4>("VIMNMX3 s32");
    run<5>("IADD");
    run<6>("SHFL.IDX");
    return 0;
}
