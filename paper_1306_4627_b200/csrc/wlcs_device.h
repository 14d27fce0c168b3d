// wlcs_device.h -- internal interface between the host C-ABI (capi.cu) and
// the kernel translation units.  Not installed; not part of the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace wlcs {

// Batch of packed pairs, all pointers DEVICE pointers.
struct BatchDev {
    const uint8_t* xs;
    const uint64_t* xoff;  // pairs + 1 offsets into xs
    uint64_t xs_bytes;     // extent of xs (chunk loads never read past it)
    const uint8_t* ys;
    const uint64_t* yoff;
    uint64_t ys_bytes;
    uint32_t* out;         // pairs lengths
    uint32_t pairs;
    int pm_bytes;          // shared-memory bytes for match masks per warp
    // filled by batch_launch from the workspace
    uint32_t* keys_in;
    uint32_t* vals_in;
    uint32_t* keys;
    uint32_t* vals;
    uint32_t* meta;
    uint32_t* overflow;
    const uint4* safe16;   // 16 zero bytes in device memory
};

size_t batch_workspace_bytes(uint32_t pairs, int pm_bytes);
int batch_smem_per_cta(int pm_bytes);
cudaError_t batch_launch(BatchDev d, void* workspace, int sms, cudaStream_t stream,
                         cudaEvent_t ev_main0 = nullptr, cudaEvent_t ev_main1 = nullptr);
cudaError_t int_peak_probe(int reps, double* ops_per_s, uint32_t* scratch);
uint32_t* batch_overflow_count_ptr(void* workspace, uint32_t pairs);
uint32_t* batch_overflow_list_ptr(void* workspace, uint32_t pairs);

}  // namespace wlcs

namespace wlcs {

// One pair for the strip kernel, all pointers DEVICE pointers.
struct PairDev {
    const uint8_t* rowp;    // row string (x for traceback; the shorter one for length)
    int64_t rows;
    const uint8_t* row_lo;  // allocation extent of the row string
    const uint8_t* row_hi;
    const uint8_t* colp;    // column (bit-vector) string
    int64_t cols;
    const uint16_t* map;    // 256 byte -> code map of the column alphabet
    int sigma;              // codes incl. the zero row
    const uint32_t* pmg;    // global match masks [sigma][W]
    int64_t W;              // words per row = ceil(cols / 32)
    int nstrips;            // ceil(W / (32 K))
    int nchunks;            // 16-row chunks of the row string (alignment included)
    uint32_t* carry;        // [nstrips][nchunks] carry masks between strips
    uint32_t* progress;     // [nstrips] published chunk counts
    uint32_t* ticket;       // strip ticket counter
    unsigned long long* zeros;  // LCS accumulator
    uint32_t* rows_out;     // optional: bit rows [G][Mpad][K]
    int64_t Mpad;
    const uint4* safe16;    // 16 zero bytes in device memory
};

cudaError_t pair_prepare(PairDev& d, uint32_t* present256, uint16_t* map256, uint32_t* sigma_dev,
                         cudaStream_t stream, int* sigma_host);
cudaError_t pair_build_pm(const PairDev& d, cudaStream_t stream);
int pair_smem_bytes(int K, int sigma);
cudaError_t pair_fill(const PairDev& d, int K, bool store, int sms, cudaStream_t stream);
cudaError_t pair_walk(const PairDev& d, int K, const uint8_t* x, uint8_t* out_rev,
                      unsigned long long* out_len, cudaStream_t stream);

}  // namespace wlcs
