// capi.cu -- host side of the C-ABI (include/wavelcs_capi.h).
//
// Owns the per-thread, per-device CUDA state (stream + grow-only device
// workspaces), validates arguments with the reference's semantics, and
// dispatches to the kernels.  There is deliberately no CPU compute path: if
// CUDA is unusable every compute entry point fails with WLCS_E_NO_DEVICE.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "wavelcs_capi.h"
#include "wlcs_device.h"

namespace {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
    t_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError();  // clear sticky-free errors
    int code = WLCS_E_CUDA;
    if (e == cudaErrorMemoryAllocation) code = WLCS_E_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
        e == cudaErrorInitializationError)
        code = WLCS_E_NO_DEVICE;
    return fail(code, std::string(where) + ": " + cudaGetErrorName(e) + " (" +
                          cudaGetErrorString(e) + ")");
}

#define WLCS_CUDA(call)                                   \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n + n / 4, 4096);
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            cudaGetLastError();
            want = std::max<size_t>(n, 256);
            e = cudaMalloc(&p, want);
            if (e != cudaSuccess) {
                p = nullptr;
                return e;
            }
        }
        cap = want;
        return cudaSuccess;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Ctx {
    int device = 0;
    bool timing = false;          // wlcs_set_timing: bracket the main kernel with events
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_main_ms = -1.f;
    int sms = 148;
    cudaStream_t stream = nullptr;
    // batch
    DevBuf xs, ys, xoff, yoff, out, ws;
    // single pair
    DevBuf px, py, pmg, carry, small, rows, outrev;
    ~Ctx() {
        if (stream) cudaStreamDestroy(stream);
    }
};

struct CtxTable {
    std::unordered_map<int, Ctx*> by_device;
    ~CtxTable() {
        for (auto& kv : by_device) delete kv.second;
    }
};
thread_local CtxTable t_ctx;

int get_ctx(Ctx** out) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int count = 0;
    e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return cuda_fail(e == cudaSuccess ? cudaErrorNoDevice : e, "cudaGetDeviceCount");
    auto it = t_ctx.by_device.find(dev);
    if (it != t_ctx.by_device.end()) {
        *out = it->second;
        return WLCS_OK;
    }
    Ctx* c = new Ctx();
    c->device = dev;
    e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaDeviceGetAttribute");
    }
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    t_ctx.by_device[dev] = c;
    *out = c;
    return WLCS_OK;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

// tables.cpp:9-24 verbatim semantics: (M+1)(N+1)*4 + M*N bytes in 128 bits.
int capacity_check(size_t m, size_t n, size_t budget) {
    if (budget == WLCS_NO_BUDGET) return WLCS_OK;
    const unsigned __int128 bytes = (unsigned __int128)(m + 1) * (unsigned __int128)(n + 1) * 4u +
                                    (unsigned __int128)m * (unsigned __int128)n;
    if (bytes > (unsigned __int128)budget) {
        const std::string need =
            bytes <= (unsigned __int128)~0ull
                ? std::to_string((unsigned long long)bytes)
                : std::string("more than 2^64");
        return fail(WLCS_E_CAPACITY, "tables for M=" + std::to_string(m) +
                                         ", N=" + std::to_string(n) + " need " + need +
                                         " bytes, over the " + std::to_string(budget) +
                                         "-byte budget");
    }
    return WLCS_OK;
}

// ------------------------------------------------------------ single pair
struct PairPlan {
    wlcs::PairDev d{};
    int K = 1;
};

int choose_k(const Ctx& c, int64_t W, int sigma, bool store) {
    const int forced = env_int("WLCS_PAIR_K", 0);
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
    // Largest K whose strips still give every SM sub-partition a warp and
    // whose match-mask slice fits comfortably in shared memory.
    const int64_t target = int64_t(c.sms) * 4;
    for (int K : {8, 4, 2}) {
        const int64_t strips = (W + 32 * K - 1) / (32 * K);
        if (strips >= target && wlcs::pair_smem_bytes(K, sigma) <= 96 * 1024) return K;
    }
    (void)store;
    return 1;
}

// Prepares alphabet, match masks and buffers for the pair (row, col).
int pair_setup(Ctx& c, const uint8_t* d_row, int64_t rows, const uint8_t* row_lo,
               const uint8_t* row_hi, const uint8_t* d_col, int64_t cols, bool store,
               PairPlan& plan) {
    wlcs::PairDev& d = plan.d;
    d.rowp = d_row;
    d.rows = rows;
    d.row_lo = row_lo;
    d.row_hi = row_hi;
    d.colp = d_col;
    d.cols = cols;
    d.W = (cols + 31) / 32;
    // small: present[256] u32 | map[256] u16 | sigma u32 | ticket | zeros u64 | walk len u64
    WLCS_CUDA(c.small.ensure(4096));
    uint8_t* sb = c.small.as<uint8_t>();
    uint32_t* present = reinterpret_cast<uint32_t*>(sb);
    uint16_t* map = reinterpret_cast<uint16_t*>(sb + 1024);
    uint32_t* sigma_dev = reinterpret_cast<uint32_t*>(sb + 1536);
    d.ticket = reinterpret_cast<uint32_t*>(sb + 1540);
    d.zeros = reinterpret_cast<unsigned long long*>(sb + 1544);
    d.safe16 = reinterpret_cast<const uint4*>(sb + 2048);  // zeroed below
    int sigma = 0;
    WLCS_CUDA(wlcs::pair_prepare(d, present, map, sigma_dev, c.stream, &sigma));
    plan.K = choose_k(c, d.W, sigma, store);
    if (wlcs::pair_smem_bytes(plan.K, sigma) > 220 * 1024) plan.K = 1;
    const int K = plan.K;
    d.nstrips = int((d.W + 32 * K - 1) / (32 * K));
    const int a_r = int(reinterpret_cast<uintptr_t>(d_row) & 15u);
    d.nchunks = int((rows + a_r + 15) / 16);
    WLCS_CUDA(c.pmg.ensure(size_t(sigma) * size_t(d.W) * 4));
    d.pmg = c.pmg.as<uint32_t>();
    const size_t carry_bytes = size_t(d.nstrips) * size_t(d.nchunks) * 4;
    const size_t prog_bytes = (size_t(d.nstrips) * 4 + 255) & ~size_t(255);
    WLCS_CUDA(c.carry.ensure(prog_bytes + carry_bytes));
    d.progress = c.carry.as<uint32_t>();
    d.carry = reinterpret_cast<uint32_t*>(c.carry.as<uint8_t>() + prog_bytes);
    WLCS_CUDA(cudaMemsetAsync(d.progress, 0, prog_bytes, c.stream));
    WLCS_CUDA(cudaMemsetAsync(d.ticket, 0, 4 + 4 + 8, c.stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 2048, 0, 16, c.stream));
    d.Mpad = (rows + 15) & ~int64_t(15);
    d.rows_out = nullptr;
    if (store) {
        const size_t bytes = size_t(d.nstrips) * 32 * size_t(d.Mpad) * size_t(K) * 4;
        WLCS_CUDA(c.rows.ensure(bytes));
        d.rows_out = c.rows.as<uint32_t>();
    }
    WLCS_CUDA(wlcs::pair_build_pm(d, c.stream));
    return WLCS_OK;
}

int pair_length_device(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                       const uint8_t* x_lo, const uint8_t* x_hi, const uint8_t* y_lo,
                       const uint8_t* y_hi, uint32_t* out) {
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    // Length is symmetric: sweep the shorter string as rows so the
    // sequential dimension is short and the parallel (strip) dimension wide.
    const bool x_rows = m <= n;
    PairPlan plan;
    int rc = x_rows ? pair_setup(c, dx, int64_t(m), x_lo, x_hi, dy, int64_t(n), false, plan)
                    : pair_setup(c, dy, int64_t(n), y_lo, y_hi, dx, int64_t(m), false, plan);
    if (rc) return rc;
    WLCS_CUDA(wlcs::pair_fill(plan.d, plan.K, false, c.sms, c.stream));
    unsigned long long zeros = 0;
    WLCS_CUDA(cudaMemcpyAsync(&zeros, plan.d.zeros, 8, cudaMemcpyDeviceToHost, c.stream));
    WLCS_CUDA(cudaStreamSynchronize(c.stream));
    *out = uint32_t(zeros);
    return WLCS_OK;
}

// ------------------------------------------------------------------ batch
int batch_device(Ctx& c, const uint8_t* d_xs, const uint64_t* d_xoff, const uint8_t* d_ys,
                 const uint64_t* d_yoff, size_t pairs, uint64_t xs_bytes, uint64_t ys_bytes,
                 int variant, uint32_t* d_out, cudaStream_t stream) {
    if (pairs == 0) return WLCS_OK;
    if (pairs > 0x7fffffffull) return fail(WLCS_E_INVALID_ARGUMENT, "too many pairs in one batch");
    if (variant != WLCS_VARIANT_BITPARALLEL)
        return fail(WLCS_E_CONFIG, "fill variant " + std::to_string(variant) +
                                       " is not available for batches");
    const int pm_bytes = env_int("WLCS_BATCH_PM_KB", 24) * 1024;
    const size_t ws_bytes = wlcs::batch_workspace_bytes(uint32_t(pairs), pm_bytes);
    WLCS_CUDA(c.ws.ensure(ws_bytes));
    wlcs::BatchDev d{};
    d.xs = d_xs;
    d.xoff = d_xoff;
    d.xs_bytes = xs_bytes;
    d.ys = d_ys;
    d.yoff = d_yoff;
    d.ys_bytes = ys_bytes;
    d.out = d_out;
    d.pairs = uint32_t(pairs);
    d.pm_bytes = pm_bytes;
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    WLCS_CUDA(wlcs::batch_launch(d, c.ws.p, c.sms, stream, c.timing ? c.ev0 : nullptr,
                                 c.timing ? c.ev1 : nullptr));
    uint32_t overflow = 0;
    WLCS_CUDA(cudaMemcpyAsync(&overflow,
                              wlcs::batch_overflow_count_ptr(c.ws.p, uint32_t(pairs)),
                              4, cudaMemcpyDeviceToHost, stream));
    WLCS_CUDA(cudaStreamSynchronize(stream));
    if (c.timing) WLCS_CUDA(cudaEventElapsedTime(&c.last_main_ms, c.ev0, c.ev1));
    if (overflow == 0) return WLCS_OK;
    // Pairs too long or with too large an alphabet for one warp: strip kernel.
    std::vector<uint32_t> ids(overflow);
    WLCS_CUDA(cudaMemcpy(ids.data(), wlcs::batch_overflow_list_ptr(c.ws.p, uint32_t(pairs)),
                         overflow * 4, cudaMemcpyDeviceToHost));
    for (uint32_t p : ids) {
        uint64_t xo[2], yo[2];
        WLCS_CUDA(cudaMemcpy(xo, d_xoff + p, 16, cudaMemcpyDeviceToHost));
        WLCS_CUDA(cudaMemcpy(yo, d_yoff + p, 16, cudaMemcpyDeviceToHost));
        uint32_t len = 0;
        int rc = pair_length_device(c, d_xs + xo[0], size_t(xo[1] - xo[0]), d_ys + yo[0],
                                    size_t(yo[1] - yo[0]), d_xs, d_xs + xs_bytes, d_ys,
                                    d_ys + ys_bytes, &len);
        if (rc) return rc;
        WLCS_CUDA(cudaMemcpy(d_out + p, &len, 4, cudaMemcpyHostToDevice));
    }
    return WLCS_OK;
}

int validate_offsets(const uint64_t* off, size_t pairs, const char* name) {
    for (size_t k = 0; k < pairs; ++k)
        if (off[k + 1] < off[k])
            return fail(WLCS_E_INVALID_ARGUMENT,
                        std::string(name) + " offsets decrease at pair " + std::to_string(k));
    return WLCS_OK;
}

}  // namespace

extern "C" {

int wlcs_abi_version(void) { return WLCS_ABI_VERSION; }

const char* wlcs_last_error(void) { return t_err.c_str(); }

int wlcs_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int wlcs_check_capacity(size_t m, size_t n, size_t memory_budget) {
    return capacity_check(m, n, memory_budget);
}

int wlcs_length_ex(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t memory_budget,
                   int variant, uint32_t* out) {
    if (!out) return fail(WLCS_E_INVALID_ARGUMENT, "out is NULL");
    if ((m && !x) || (n && !y)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL input");
    int rc = capacity_check(m, n, memory_budget);
    if (rc) return rc;
    Ctx* c = nullptr;
    rc = get_ctx(&c);
    if (rc) return rc;
    if (variant != WLCS_VARIANT_BITPARALLEL)
        return fail(WLCS_E_CONFIG, "fill variant " + std::to_string(variant) +
                                       " is not available for single pairs");
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    WLCS_CUDA(cudaMemcpyAsync(c->px.p, x, m, cudaMemcpyHostToDevice, c->stream));
    WLCS_CUDA(cudaMemcpyAsync(c->py.p, y, n, cudaMemcpyHostToDevice, c->stream));
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dy = c->py.as<uint8_t>();
    return pair_length_device(*c, dx, m, dy, n, dx, dx + m, dy, dy + n, out);
}

int wlcs_length(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t memory_budget,
                uint32_t* out) {
    return wlcs_length_ex(x, m, y, n, memory_budget, WLCS_VARIANT_BITPARALLEL, out);
}

int wlcs_length_device(const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n, int variant,
                       uint32_t* out, void* stream) {
    (void)stream;
    if (!out) return fail(WLCS_E_INVALID_ARGUMENT, "out is NULL");
    if ((reinterpret_cast<uintptr_t>(d_x) | reinterpret_cast<uintptr_t>(d_y)) & 15u)
        return fail(WLCS_E_INVALID_ARGUMENT, "device string buffers must be 16-byte aligned");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    if (variant != WLCS_VARIANT_BITPARALLEL)
        return fail(WLCS_E_CONFIG, "fill variant " + std::to_string(variant) +
                                       " is not available for single pairs");
    return pair_length_device(*c, d_x, m, d_y, n, d_x, d_x + m, d_y, d_y + n, out);
}

int wlcs_subsequence(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                     size_t memory_budget, uint8_t* out, size_t cap, size_t* out_len) {
    if (!out_len) return fail(WLCS_E_INVALID_ARGUMENT, "out_len is NULL");
    if ((m && !x) || (n && !y)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL input");
    int rc = capacity_check(m, n, memory_budget);
    if (rc) return rc;
    Ctx* c = nullptr;
    rc = get_ctx(&c);
    if (rc) return rc;
    *out_len = 0;
    if (m == 0 || n == 0) return WLCS_OK;
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    WLCS_CUDA(cudaMemcpyAsync(c->px.p, x, m, cudaMemcpyHostToDevice, c->stream));
    WLCS_CUDA(cudaMemcpyAsync(c->py.p, y, n, cudaMemcpyHostToDevice, c->stream));
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dy = c->py.as<uint8_t>();
    // Orientation matters for tie-breaking: rows = x (parent), columns = y.
    PairPlan plan;
    rc = pair_setup(*c, dx, int64_t(m), dx, dx + m, dy, int64_t(n), true, plan);
    if (rc) return rc;
    WLCS_CUDA(wlcs::pair_fill(plan.d, plan.K, true, c->sms, c->stream));
    const size_t maxlen = std::min(m, n);
    WLCS_CUDA(c->outrev.ensure(maxlen + 16));
    unsigned long long* dlen = plan.d.zeros + 1;
    WLCS_CUDA(wlcs::pair_walk(plan.d, plan.K, dx, c->outrev.as<uint8_t>(), dlen, c->stream));
    unsigned long long len = 0, zeros = 0;
    WLCS_CUDA(cudaMemcpyAsync(&len, dlen, 8, cudaMemcpyDeviceToHost, c->stream));
    WLCS_CUDA(cudaMemcpyAsync(&zeros, plan.d.zeros, 8, cudaMemcpyDeviceToHost, c->stream));
    WLCS_CUDA(cudaStreamSynchronize(c->stream));
    if (len != zeros)
        return fail(WLCS_E_INTERNAL, "traceback length " + std::to_string(len) +
                                         " differs from the fill length " + std::to_string(zeros));
    *out_len = size_t(len);
    if (len > cap)
        return fail(WLCS_E_INVALID_ARGUMENT, "output buffer holds " + std::to_string(cap) +
                                                 " bytes, subsequence has " + std::to_string(len));
    std::vector<uint8_t> rev(len);
    if (len) WLCS_CUDA(cudaMemcpy(rev.data(), c->outrev.p, len, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < len; ++k) out[k] = rev[len - 1 - k];
    return WLCS_OK;
}

int wlcs_length_batch_device(const uint8_t* d_xs, const uint64_t* d_x_off, const uint8_t* d_ys,
                             const uint64_t* d_y_off, size_t pairs, uint64_t xs_bytes,
                             uint64_t ys_bytes, int variant, uint32_t* d_out, void* stream) {
    if ((reinterpret_cast<uintptr_t>(d_xs) | reinterpret_cast<uintptr_t>(d_ys)) & 15u)
        return fail(WLCS_E_INVALID_ARGUMENT, "device string buffers must be 16-byte aligned");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    return batch_device(*c, d_xs, d_x_off, d_ys, d_y_off, pairs, xs_bytes, ys_bytes, variant,
                        d_out, s);
}

int wlcs_length_batch_ex(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                         const uint64_t* y_off, size_t pairs, int variant, uint32_t* out) {
    if (pairs == 0) return WLCS_OK;
    if (!x_off || !y_off || !out) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    int rc = validate_offsets(x_off, pairs, "x");
    if (rc) return rc;
    rc = validate_offsets(y_off, pairs, "y");
    if (rc) return rc;
    Ctx* c = nullptr;
    rc = get_ctx(&c);
    if (rc) return rc;
    const uint64_t xs_bytes = x_off[pairs], ys_bytes = y_off[pairs];
    if ((xs_bytes && !xs) || (ys_bytes && !ys)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL strings");
    WLCS_CUDA(c->xs.ensure(xs_bytes + 16));
    WLCS_CUDA(c->ys.ensure(ys_bytes + 16));
    WLCS_CUDA(c->xoff.ensure((pairs + 1) * 8));
    WLCS_CUDA(c->yoff.ensure((pairs + 1) * 8));
    WLCS_CUDA(c->out.ensure(pairs * 4));
    cudaStream_t s = c->stream;
    if (xs_bytes) WLCS_CUDA(cudaMemcpyAsync(c->xs.p, xs, xs_bytes, cudaMemcpyHostToDevice, s));
    if (ys_bytes) WLCS_CUDA(cudaMemcpyAsync(c->ys.p, ys, ys_bytes, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(c->xoff.p, x_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(c->yoff.p, y_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, s));
    rc = batch_device(*c, c->xs.as<uint8_t>(), c->xoff.as<uint64_t>(), c->ys.as<uint8_t>(),
                      c->yoff.as<uint64_t>(), pairs, xs_bytes, ys_bytes, variant,
                      c->out.as<uint32_t>(), s);
    if (rc) return rc;
    WLCS_CUDA(cudaMemcpyAsync(out, c->out.p, pairs * 4, cudaMemcpyDeviceToHost, s));
    WLCS_CUDA(cudaStreamSynchronize(s));
    return WLCS_OK;
}

int wlcs_length_batch(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                      const uint64_t* y_off, size_t pairs, uint32_t* out) {
    return wlcs_length_batch_ex(xs, x_off, ys, y_off, pairs, WLCS_VARIANT_BITPARALLEL, out);
}

int wlcs_set_timing(int on) {
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    c->timing = on != 0;
    c->last_main_ms = -1.f;
    return WLCS_OK;
}

int wlcs_last_kernel_ms(float* ms) {
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    *ms = c->last_main_ms;
    return WLCS_OK;
}

int wlcs_probe_int_peak(int reps, double* ops_per_s) {
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    WLCS_CUDA(c->small.ensure(4096));
    WLCS_CUDA(wlcs::int_peak_probe(reps, ops_per_s, c->small.as<uint32_t>() + 900));
    return WLCS_OK;
}

int wlcs_generate_pairs(size_t pairs, size_t lo, size_t hi, const uint8_t* alphabet,
                        size_t alphabet_len, uint64_t seed, uint8_t* xs, uint64_t* x_off,
                        uint8_t* ys, uint64_t* y_off) {
    if (alphabet_len == 0 || !alphabet || hi < lo)
        return fail(WLCS_E_INVALID_ARGUMENT, "generate_pairs: bad alphabet or length range");
    std::mt19937_64 master(seed);
    uint64_t xo = 0, yo = 0;
    x_off[0] = y_off[0] = 0;
    for (size_t k = 0; k < pairs; ++k) {
        const size_t m = lo + size_t(master() % (hi - lo + 1));
        const size_t n = lo + size_t(master() % (hi - lo + 1));
        const uint64_t sx = master(), sy = master();
        std::mt19937_64 rx(sx), ry(sy);
        for (size_t i = 0; i < m; ++i) xs[xo + i] = alphabet[rx() % alphabet_len];
        for (size_t j = 0; j < n; ++j) ys[yo + j] = alphabet[ry() % alphabet_len];
        xo += m;
        yo += n;
        x_off[k + 1] = xo;
        y_off[k + 1] = yo;
    }
    return WLCS_OK;
}

void* wlcs_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        fail(WLCS_E_OUT_OF_MEMORY, "cudaHostAlloc failed");
        return nullptr;
    }
    return p;
}

void wlcs_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int wlcs_generate_random(size_t length, const uint8_t* alphabet, size_t alphabet_len,
                         uint64_t seed, uint8_t* out) {
    if (alphabet_len == 0 || !alphabet)
        return fail(WLCS_E_INVALID_ARGUMENT, "generate_random: alphabet must not be empty");
    std::mt19937_64 rng(seed);
    for (size_t k = 0; k < length; ++k) out[k] = alphabet[rng() % alphabet_len];
    return WLCS_OK;
}

}  // extern "C"
