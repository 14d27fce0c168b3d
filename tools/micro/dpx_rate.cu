// Microbenchmark: issue rate of the DPX integer min/max instructions on
// sm_100a against plain ALU ops, and whether they co-issue with LOP3/SHF
// (i.e. run on a different pipe).  8 independent chains per thread, 16 warps
// per SM.  Prints instructions per clock per SM for each mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dpx_rate dpx_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8

template <int OP>
__device__ __forceinline__ void step(uint32_t (&x)[CH], uint32_t a, uint32_t b) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
        if (OP == 1) x[c] = __vmaxu2(x[c], a);
        if (OP == 2) x[c] = __vimax3_u16x2(x[c], a, b);
        if (OP == 3) x[c] = __viaddmax_u16x2(x[c], a, b);
        if (OP == 4) x[c] = __vimax3_s32(x[c], a, b);
        if (OP == 5) asm volatile("shf.r.wrap.b32 %0, %0, %0, %1;" : "+r"(x[c]) : "r"(a));
        if (OP == 6) {  // 1 LOP3 + 1 VIMNMX3.U16x2
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            x[c] = __vimax3_u16x2(x[c], a, b);
        }
        if (OP == 7) {  // 2 ALU + 2 DPX: the 16x2 cell pair (shift, and, add-max, max)
            uint32_t m;
            asm volatile("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(m) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, 0x00010001, 0xc0;" : "+r"(m) : "r"(m));
            x[c] = __viaddmax_u16x2(x[c], m, __vmaxu2(a, x[c ^ 1]));
        }
        if (OP == 9) {  // LOP3 + VIADDMNMX.U16x2
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            x[c] = __viaddmax_u16x2(x[c], a, b);
        }
        if (OP == 10) {  // variant A: XNOR, relu(d'+2), max(up,left), max(diag+m, .)
            uint32_t dn;
            asm volatile("lop3.b32 %0, %1, %2, 0, 0x99;" : "=r"(dn) : "r"(x[c]), "r"(b));
            const uint32_t m = __viaddmax_s16x2_relu(dn, 0x00020002u, 0u);
            x[c] = __viaddmax_u16x2(x[c ^ 1], m, __vmaxu2(a, x[c]));
        }
        if (OP == 11) {  // variant C: XOR, IADD3 diag - d + 0x10001, VIMNMX3
            uint32_t d, t;
            asm volatile("lop3.b32 %0, %1, %2, 0, 0x3c;" : "=r"(d) : "r"(x[c]), "r"(b));
            asm volatile("sub.u32 %0, %1, %2;" : "=r"(t) : "r"(x[c ^ 1]), "r"(d));
            x[c] = __vimax3_u16x2(a, x[c], t + 0x10001u);
        }
        if (OP == 8) {  // IADD3 + VIMNMX3.U16x2
            asm volatile("add.u32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
            x[c] = __vimax3_u16x2(x[c], a, b);
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int iters, uint32_t a, uint32_t b) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 7u + c;
    for (int i = 0; i < iters; ++i) {
        step<OP>(x, a + i, b);
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
    printf("%-34s %6.1f thread-ops/clk/SM  %7.2f T ops/s\n", name, ops / cyc / sms,
           ops / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("LOP3", 1, sms);
    run<5>("SHF", 1, sms);
    run<1>("VIMNMX.U16x2", 1, sms);
    run<2>("VIMNMX3.U16x2", 1, sms);
    run<3>("VIADDMNMX.U16x2", 1, sms);
    run<4>("VIMNMX3 (s32)", 1, sms);
    run<6>("LOP3 + VIMNMX3.U16x2", 2, sms);
    run<8>("IADD + VIMNMX3.U16x2", 2, sms);
    run<9>("LOP3 + VIADDMNMX.U16x2", 2, sms);
    run<10>("variant A (4 ops / 2 cells)", 4, sms);
    run<11>("variant C (3 ops / 2 cells)", 3, sms);
    run<7>("SHF+LOP3+VIMNMX+VIADDMNMX (cell x2)", 4, sms);
    return 0;
}
