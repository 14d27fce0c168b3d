// Which warps share a sub-partition?  Every warp runs the same ALU-bound loop
// and records %smid, %warpid and its duration in SM clocks; warps that share
// an SMSP take proportionally longer.  Configs: 1-warp CTAs, 2-warp CTAs
// (both busy), 2-warp CTAs with only warp 0 busy.  Shared memory forces 6
// CTAs per SM like the batch kernel.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <map>
#include <cuda_runtime.h>

__global__ void probe(unsigned long long* out, int iters, int busy_mask) {
    extern __shared__ uint32_t sm[];
    const int w = threadIdx.x >> 5;
    uint32_t smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    long long t0 = clock64();
    uint32_t a = threadIdx.x, b = a * 3, c = a * 5, e = a * 7, f = a ^ 9, g = a + 11, h = a * 13, k = a * 17;
    if ((busy_mask >> w) & 1) {
        for (int i = 0; i < iters; ++i) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(b) : "r"(c), "r"(e));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c) : "r"(e), "r"(f));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(e) : "r"(f), "r"(g));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(f) : "r"(g), "r"(h));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(g) : "r"(h), "r"(k));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(h) : "r"(k), "r"(a));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(k) : "r"(a), "r"(b));
        }
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
        const int gw = blockIdx.x * (blockDim.x >> 5) + w;
        out[gw * 4 + 0] = smid;
        out[gw * 4 + 1] = wid;
        out[gw * 4 + 2] = (unsigned long long)(t1 - t0);
        out[gw * 4 + 3] = (unsigned long long)(a ^ b ^ c ^ e ^ f ^ g ^ h ^ k) & 1 ? blockIdx.x : blockIdx.x;
    }
    if (threadIdx.x == 0) sm[0] = 1;
}

void run(const char* name, int warps_per_cta, int busy_mask, int sms) {
    const int ctas = sms * 6, nw = ctas * warps_per_cta;
    unsigned long long* d;
    cudaMalloc(&d, nw * 32);
    const int smem = 35 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<ctas, 32 * warps_per_cta, smem>>>(d, 20000, busy_mask);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(nw * 4);
    cudaMemcpy(h.data(), d, nw * 32, cudaMemcpyDeviceToHost);
    printf("== %s\n", name);
    for (int target : {0, 1, 77}) {
        printf(" SM %d:", target);
        for (int i = 0; i < nw; ++i)
            if (int(h[i * 4]) == target && ((busy_mask >> (i % warps_per_cta)) & 1))
                printf(" [cta%llu w%d wid%llu %.0fk]", h[i * 4 + 3], i % warps_per_cta, h[i * 4 + 1], h[i * 4 + 2] / 1e3);
        printf("\n");
    }
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("1-warp CTAs", 1, 1, sms);
    run("2-warp CTAs, both busy", 2, 3, sms);
    run("2-warp CTAs, warp 0 busy", 2, 1, sms);
    run("2-warp CTAs, warp 1 busy", 2, 2, sms);
    return 0;
}
