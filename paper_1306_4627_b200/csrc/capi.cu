// capi.cu -- host side of the C-ABI (include/wavelcs_capi.h).
//
// Owns the per-thread, per-device CUDA state (stream + grow-only device
// workspaces), validates arguments with the reference's semantics, and
// dispatches to the kernels.  There is deliberately no CPU compute path: if
// CUDA is unusable every compute entry point fails with WLCS_E_NO_DEVICE.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
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
    bool timing_pending = false;  // ev0/ev1 recorded by an asynchronous call, not yet read
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host batch pipeline: H2D of chunk k+1 || compute of k
    std::vector<cudaEvent_t> chunk_ev;
    // pinned host words for the small D2H reads (counts, lengths) that end a
    // call: a pageable destination would make each one a staged, synchronous
    // copy (~10 us) inside the caller's timed region
    uint64_t* hscratch = nullptr;
    cudaEvent_t join_ev = nullptr;       // orders c.stream after a caller's stream
    // pinned staging ring for host->device copies of pageable caller buffers
    uint8_t* hstage[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    // batch (ws: first pass per chunk; ws2 + wcarry: the device second pass)
    DevBuf xs, ys, xoff, yoff, out, ws, ws2, wcarry;
    // single pair
    DevBuf px, py, pmg, carry, small, rows, outrev, codes, ry, vbuf, wave, sink, walk, tile, sea;
    DevBuf ckpt, bandcodes;  // banded traceback
    ~Ctx() {
        if (hscratch) cudaFreeHost(hscratch);
        for (cudaEvent_t e : chunk_ev) cudaEventDestroy(e);
        if (join_ev) cudaEventDestroy(join_ev);
        for (int i = 0; i < 2; ++i) {
            if (hstage[i]) cudaFreeHost(hstage[i]);
            if (stage_ev[i]) cudaEventDestroy(stage_ev[i]);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
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
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->hscratch), 64 * sizeof(uint64_t),
                      cudaHostAllocDefault);
    if (e != cudaSuccess) {
        c->hscratch = nullptr;
        delete c;
        return cuda_fail(e, "cudaHostAlloc");
    }
    t_ctx.by_device[dev] = c;
    *out = c;
    return WLCS_OK;
}

// Waits for the end of a call's work on stream s.  A short bounded spin on
// cudaStreamQuery returns within about a microsecond of completion (a
// blocking or yielding cudaStreamSynchronize adds several to tens of
// microseconds of wake-up to every synchronous call); long waits fall back to
// the blocking synchronize.
cudaError_t stream_wait(cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e != cudaErrorNotReady) return e;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(3000))
            return cudaStreamSynchronize(s);
    }
}

// A NULL stream from the caller means the legacy default stream (torch's
// default stream, plain <<<>>> launches): never the library's own stream,
// which is non-blocking and therefore unordered with it.
cudaStream_t caller_stream(void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
}

// Orders the library's per-thread stream after the work the caller enqueued
// on `user` before this call (an event, no host wait).
int join_caller(Ctx& c, cudaStream_t user) {
    if (user == c.stream) return WLCS_OK;
    if (!c.join_ev) WLCS_CUDA(cudaEventCreateWithFlags(&c.join_ev, cudaEventDisableTiming));
    WLCS_CUDA(cudaEventRecord(c.join_ev, user));
    WLCS_CUDA(cudaStreamWaitEvent(c.stream, c.join_ev, 0));
    return WLCS_OK;
}

// Host -> device copy of a caller's buffer (the input path of the single-pair
// entry points).  Page-locked sources (wlcs_host_alloc, cudaHostAlloc) are
// copied directly; pageable ones go through a ring of two 4 MB pinned stage
// buffers, the host memcpy of chunk k+1 overlapping the DMA of chunk k (a
// stage is reused only after its previous DMA finished: its event).  Small
// copies go straight to the driver.
constexpr size_t kStageBytes = size_t(4) << 20;
int h2d_staged(Ctx& c, void* dst, const void* src, size_t n, cudaStream_t s) {
    if (n == 0) return WLCS_OK;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess &&
                        (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (pinned || n <= (size_t(64) << 10)) {
        WLCS_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s));
        return WLCS_OK;
    }
    for (int i = 0; i < 2; ++i) {
        if (!c.hstage[i]) WLCS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.hstage[i]), kStageBytes,
                                                  cudaHostAllocDefault));
        if (!c.stage_ev[i]) {
            WLCS_CUDA(cudaEventCreateWithFlags(&c.stage_ev[i], cudaEventDisableTiming));
            WLCS_CUDA(cudaEventRecord(c.stage_ev[i], s));
        }
    }
    const uint8_t* from = static_cast<const uint8_t*>(src);
    uint8_t* to = static_cast<uint8_t*>(dst);
    for (size_t off = 0, k = 0; off < n; off += kStageBytes, ++k) {
        const size_t len = std::min(kStageBytes, n - off);
        const int i = int(k & 1);
        WLCS_CUDA(cudaEventSynchronize(c.stage_ev[i]));  // its previous DMA is done
        std::memcpy(c.hstage[i], from + off, len);
        WLCS_CUDA(cudaMemcpyAsync(to + off, c.hstage[i], len, cudaMemcpyHostToDevice, s));
        WLCS_CUDA(cudaEventRecord(c.stage_ev[i], s));
    }
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

// Words per lane.  Cost model in cycles, calibrated on B200 (single-strip
// probe, tools/pair_probe.py): a 16-row step costs kStep[K] cycles when the
// strip has a sub-partition to itself; strips start ~40 steps apart (31-step
// lane pipeline + carry hand-off; tools/gpu/skew.sh); strips beyond the
// resident warps run in waves; more resident strips than sub-partitions share
// issue slots.
// Lane shapes up to K = 10 words per lane in 26.25 KB of masks per warp
// (21 codes x 1280 B: the 20-letter alphabet plus the zero row) -> 8 warps
// per SM, two per sub-partition.
// Small batches (e.g. one GPU's shard of a strong-scaling run) are bound by
// their longest task, not by throughput: narrower lane shapes (more lanes per
// pair, shorter tasks) win there.  Measured on C2-like pairs (tools/gpu/
// small_batch4.sh, fused plan): 4-8k pairs best at kmax 4, 16-32k at 8,
// 65,536 at 10.
int batch_kmax(size_t pairs = 0) {
    const int k = env_int("WLCS_BATCH_KMAX", 0);
    if (k >= 1 && k <= 12) return k;
    if (pairs && pairs <= 12288) return 4;
    if (pairs && pairs <= 40960) return 8;
    return 10;
}
int batch_pm_bytes() {  // >= flags + chunk stage; WLCS_BATCH_PM_KB overrides
    const int kb = env_int("WLCS_BATCH_PM_KB", 0);
    return kb > 0 ? std::max(kb, 14) * 1024 : 26880;
}

int choose_k(const Ctx& c, int64_t W, int64_t rows_per_prob, const wlcs::PairDev& d, int nprob) {
    const int forced = env_int("WLCS_PAIR_K", 0);
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
    const double chunks = double((rows_per_prob + 15) / 16);
    double best = 1e300;
    int best_k = 1;
    for (int K : {1, 2, 4, 8}) {
        const int smem = wlcs::pair_smem_bytes(K, d.sigma);
        if (smem > 200 * 1024) continue;
        const double step = K == 1 ? 330 : K == 2 ? 363 : K == 4 ? 535 : 987;
        const double strips = double((W + 32 * K - 1) / (32 * K));
        const double total = strips * nprob;
        const double per_sm = std::min(32, (227 * 1024) / std::max(smem, 1));
        const double active = std::min(total, per_sm * c.sms);
        const double share = std::max(1.0, active / (4.0 * c.sms));
        const double waves = std::ceil(total / active);
        const double cost = (waves * chunks + strips * 40.0) * step * share;
        if (cost < best) {
            best = cost;
            best_k = K;
        }
    }
    return best_k;
}

void set_problem(wlcs::FillProblem& P, int64_t rows, uint32_t* pmg, int64_t cols, int K) {
    P.rows = rows;
    P.pmg = pmg;
    P.cols = cols;
    P.W = (cols + 31) / 32;
    P.nstrips = int((P.W + 32 * K - 1) / (32 * K));
    P.nchunks = int((rows + 15) / 16);
    P.Mpad = int64_t(P.nchunks) * 16;
    P.Dpad = P.Mpad + 512;
    P.cwords = ((int64_t(P.nchunks) + 3) & ~int64_t(3)) + 16;
    P.walk_row0 = 0;
    P.walk_mtot = rows;
    P.ckpt_chunks = 1;
}

bool use_split(int64_t rows, bool store) {
    if (store) return false;
    const int forced = env_int("WLCS_PAIR_SPLIT", -1);
    if (forced >= 0) return forced != 0 && rows >= 2;
    return rows >= 2048;
}

// Prepares alphabet, match masks and buffers for the pair (row, col).  With
// `split` the rows are cut in half and the bottom half runs on the reversed
// strings as a second problem of the same launch (length only).
// small: present[256] u32 @0 | map[256] u16 @1024 | sigma @1536 |
//        zeros u64 @1544 | walk len u64 @1552 | walk misses u32[3] @1560 |
//        strip tickets u32[kMaxProblems] @1664 | safe16 @2048
constexpr int kTicketOff = 1664;
constexpr int kErrOff = 1596;  // strip-kernel watchdog flag (zeroed with the tickets)

// Enqueues the read of the strip kernel's watchdog flag into hscratch[7];
// after the stream wait, watchdog_failed() tells whether a carry poll timed out.
int watchdog_read(Ctx& c, cudaStream_t s) {
    WLCS_CUDA(cudaMemcpyAsync(c.hscratch + 7, c.small.as<uint8_t>() + kErrOff, 4,
                              cudaMemcpyDeviceToHost, s));
    return WLCS_OK;
}
int watchdog_failed(Ctx& c) {
    const uint32_t err = uint32_t(c.hscratch[7]);
    if (err == 0) return WLCS_OK;
    return fail(WLCS_E_INTERNAL,
                "fill kernel: a hand-off word of a neighbouring strip / band / slice never "
                "arrived (watchdog)");
}

int pair_setup(Ctx& c, const uint8_t* d_row, int64_t rows, const uint8_t* d_col, int64_t cols,
               bool store, PairPlan& plan, bool allow_split = true) {
    wlcs::PairDev& d = plan.d;
    const bool split = allow_split && use_split(rows, store);
    d.nprob = split ? 2 : 1;
    d.colp0 = d_col;
    d.prob[0].cols = cols;
    WLCS_CUDA(c.small.ensure(4096));
    uint8_t* sb = c.small.as<uint8_t>();
    uint32_t* present = reinterpret_cast<uint32_t*>(sb);
    uint16_t* map = reinterpret_cast<uint16_t*>(sb + 1024);
    uint32_t* sigma_dev = reinterpret_cast<uint32_t*>(sb + 1536);
    d.ticket = reinterpret_cast<uint32_t*>(sb + kTicketOff);
    d.error = reinterpret_cast<uint32_t*>(sb + kErrOff);
    WLCS_CUDA(c.sink.ensure(size_t(wlcs::kPairSinkWords) * 4));
    d.sink = c.sink.as<uint32_t>();
    unsigned long long* zeros = reinterpret_cast<unsigned long long*>(sb + 1544);
    d.safe16 = reinterpret_cast<const uint4*>(sb + 2048);  // zeroed below
    int sigma = 0;
    WLCS_CUDA(wlcs::pair_prepare(d, present, map, sigma_dev, c.stream, &sigma));
    const int64_t W = (cols + 31) / 32;
    const int64_t mid = split ? rows / 2 : rows;
    plan.K = choose_k(c, W, rows - mid > mid ? rows - mid : mid, d, d.nprob);
    if (wlcs::pair_smem_bytes(plan.K, sigma) > 220 * 1024)
        return fail(WLCS_E_INTERNAL, "match-mask table does not fit in shared memory");
    const int K = plan.K;
    const size_t pm_words = size_t(sigma) * size_t(W);
    WLCS_CUDA(c.pmg.ensure(pm_words * 4 * size_t(d.nprob)));
    uint32_t* pmg = c.pmg.as<uint32_t>();
    set_problem(d.prob[0], mid, pmg, cols, K);
    if (split) {
        set_problem(d.prob[1], rows - mid, pmg + pm_words, cols, K);
        WLCS_CUDA(c.ry.ensure(size_t(cols) + 16));
        WLCS_CUDA(c.vbuf.ensure(size_t(W) * 16 + 64));
        WLCS_CUDA(wlcs::pair_reverse(d_col, cols, c.ry.as<uint8_t>(), c.stream));
        d.prob[0].v_out = c.vbuf.as<uint32_t>();
        d.prob[1].v_out = c.vbuf.as<uint32_t>() + W;
    } else {
        d.prob[0].zeros = zeros;
    }
    // pre-coded rows, padded on both sides (pair_code_rows)
    size_t code_vecs = 0;
    for (int q = 0; q < d.nprob; ++q) code_vecs += 4 * size_t(wlcs::pair_code_plane(d.prob[q].nchunks));
    WLCS_CUDA(c.codes.ensure(code_vecs * 16));
    uint4* code_base = c.codes.as<uint4>();
    for (int q = 0; q < d.nprob; ++q) {
        const uint8_t* src = q == 0 ? d_row : d_row + mid;
        WLCS_CUDA(wlcs::pair_code_rows(src, d.prob[q].rows, q == 1, map, K, d.prob[q], code_base,
                                       c.stream));
        code_base += 4 * wlcs::pair_code_plane(d.prob[q].nchunks);
    }
    size_t carry_words = 0;
    for (int q = 0; q < d.nprob; ++q)
        carry_words += size_t(d.prob[q].nstrips) * size_t(d.prob[q].cwords);
    WLCS_CUDA(c.carry.ensure(carry_words * 4 + 256));
    uint32_t* carry = c.carry.as<uint32_t>();
    for (int q = 0; q < d.nprob; ++q) {
        d.prob[q].carry = carry;
        carry += size_t(d.prob[q].nstrips) * size_t(d.prob[q].cwords);
    }
    WLCS_CUDA(cudaMemsetAsync(c.carry.p, 0, carry_words * 4, c.stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 1540, 0, kTicketOff + 4 * wlcs::kMaxProblems - 1540, c.stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 2048, 0, 16, c.stream));
    if (store) {
        const size_t bytes =
            size_t(d.prob[0].nstrips) * 32 * size_t(d.prob[0].Dpad) * size_t(K) * 4;
        WLCS_CUDA(c.rows.ensure(bytes));
        d.prob[0].rows_out = c.rows.as<uint32_t>();
    }
    WLCS_CUDA(wlcs::pair_build_pm(d_col, cols, map, sigma, W, pmg, c.stream));
    if (split) WLCS_CUDA(wlcs::pair_build_pm(c.ry.as<uint8_t>(), cols, map, sigma, W,
                                             pmg + pm_words, c.stream));
    return WLCS_OK;
}

unsigned long long* pair_zeros_ptr(Ctx& c) {
    return reinterpret_cast<unsigned long long*>(c.small.as<uint8_t>() + 1544);
}

int pair_length_device(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                       uint32_t* out) {
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    // Length is symmetric: sweep the shorter string as rows so the
    // sequential dimension is short and the parallel (strip) dimension wide.
    const int orient = env_int("WLCS_PAIR_ROWS", 0);  // diagnostics: 1 = x rows, 2 = y rows
    const bool x_rows = orient == 1 ? true : orient == 2 ? false : m <= n;
    PairPlan plan;
    int rc = x_rows ? pair_setup(c, dx, int64_t(m), dy, int64_t(n), false, plan)
                    : pair_setup(c, dy, int64_t(n), dx, int64_t(m), false, plan);
    if (rc) return rc;
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev0, c.stream));
    WLCS_CUDA(wlcs::pair_fill(plan.d, plan.K, false, c.sms, c.stream));
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev1, c.stream));
    unsigned long long* zeros = pair_zeros_ptr(c);
    if (plan.d.nprob == 2) {
        const wlcs::FillProblem& P = plan.d.prob[0];
        uint32_t* scratch = c.vbuf.as<uint32_t>() + 2 * P.W;
        WLCS_CUDA(wlcs::pair_split_combine(P.v_out, plan.d.prob[1].v_out, P.W, P.cols, scratch,
                                           zeros, c.stream));
    }
    WLCS_CUDA(cudaMemcpyAsync(c.hscratch, zeros, 8, cudaMemcpyDeviceToHost, c.stream));
    if (int rc2 = watchdog_read(c, c.stream)) return rc2;
    WLCS_CUDA(stream_wait(c.stream));
    if (int rc2 = watchdog_failed(c)) return rc2;
    if (c.timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c.last_main_ms, c.ev0, c.ev1));
        c.timing_pending = false;
    }
    *out = uint32_t(c.hscratch[0]);
    return WLCS_OK;
}

// Cell-wavefront variant for one pair (wavefront.cu): rows = the longer
// string (more bands in flight), columns = the shorter one.
int pair_wave_device(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                     uint32_t* out) {
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    const bool x_rows = m >= n;
    wlcs::WavePairDev d{};
    d.rowp = x_rows ? dx : dy;
    d.m = int64_t(x_rows ? m : n);
    d.colp = x_rows ? dy : dx;
    d.n = int64_t(x_rows ? n : m);
    if (d.n >= (int64_t(1) << 24))
        return fail(WLCS_E_CONFIG, "wavefront variant: the shorter string must be < 2^24 bytes");
    d.bstride = ((d.n + 64) + 31) & ~int64_t(31);
    d.R = wlcs::wave_pair_rows(d.m, c.sms);
    if (const char* e = std::getenv("WLCS_WAVE_PAIR_R")) d.R = std::atoi(e);  // experiments
    const int64_t bands = wlcs::wave_pair_bands(d.m, d.R);
    const int64_t budget = int64_t(1) << 30;  // boundary-row ring
    int64_t nbuf = budget / (d.bstride * 4);
    if (nbuf > bands) nbuf = bands;
    if (nbuf < 2) nbuf = 2;
    d.nbuf = uint32_t(nbuf);
    const size_t bytes = size_t(nbuf) * size_t(d.bstride) * 4;
    WLCS_CUDA(c.wave.ensure(bytes));
    WLCS_CUDA(c.small.ensure(4096));
    d.bnd = c.wave.as<uint32_t>();
    d.ticket = reinterpret_cast<uint32_t*>(c.small.as<uint8_t>() + 1600);
    d.out = d.ticket + 1;
    d.error = reinterpret_cast<uint32_t*>(c.small.as<uint8_t>() + kErrOff);
    WLCS_CUDA(cudaMemsetAsync(d.bnd, 0, bytes, c.stream));
    WLCS_CUDA(cudaMemsetAsync(d.error, 0, 1608 - kErrOff, c.stream));  // error, ticket, out
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev0, c.stream));
    WLCS_CUDA(wlcs::wave_pair_launch(d, c.sms, c.stream));
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev1, c.stream));
    WLCS_CUDA(cudaMemcpyAsync(out, d.out, 4, cudaMemcpyDeviceToHost, c.stream));
    if (int rc = watchdog_read(c, c.stream)) return rc;
    WLCS_CUDA(stream_wait(c.stream));
    if (c.timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c.last_main_ms, c.ev0, c.ev1));
        c.timing_pending = false;
    }
    return watchdog_failed(c);
}

int pair_length_variant(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                        int variant, uint32_t* out) {
    if (variant == WLCS_VARIANT_WAVEFRONT) return pair_wave_device(c, dx, m, dy, n, out);
    return pair_length_device(c, dx, m, dy, n, out);
}

// ------------------------------------------------------------------ batch
// Words of the shorter string above which a pair leaves the first pass's lane
// shapes (bitpar_batch.cu: w > 32 * kmax).
bool batch_is_long(uint64_t m, uint64_t n, int kmax) {
    const uint64_t cols = m < n ? m : n;
    return (cols + 31) / 32 > uint64_t(32) * uint64_t(kmax);
}

// Enqueues one batch on `s` (device pointers, nothing waits on the host):
// the first pass (plan, scatter, main) and the second pass over the first
// pass's overflow list (bitpar_wide.cu; the list length is read on the
// device, so an empty second pass is two short launches).  With
// `long_to_host` the pairs too wide for the first pass are skipped -- the
// host entry points run them through the strip kernel instead.
int batch_enqueue(Ctx& c, const uint8_t* d_xs, const uint64_t* d_xoff, const uint8_t* d_ys,
                  const uint64_t* d_yoff, size_t pairs, uint64_t xs_bytes, uint64_t ys_bytes,
                  uint32_t* d_out, cudaStream_t s, void* ws, bool long_to_host, bool ev_start,
                  bool ev_end, int kmax) {
    if (pairs == 0) return WLCS_OK;
    wlcs::BatchDev d{};
    d.xs = d_xs;
    d.xoff = d_xoff;
    d.xs_bytes = xs_bytes;
    d.ys = d_ys;
    d.yoff = d_yoff;
    d.ys_bytes = ys_bytes;
    d.out = d_out;
    d.pairs = uint32_t(pairs);
    d.pm_bytes = batch_pm_bytes();
    d.kmax = kmax;  // the host's long-pair routing used the same value
    d.long_to_host = long_to_host ? 1 : 0;
    if ((ev_start || ev_end) && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    WLCS_CUDA(wlcs::batch_launch(d, ws, c.sms, s, ev_start ? c.ev0 : nullptr,
                                 ev_end ? c.ev1 : nullptr));
    if (ev_end) c.timing_pending = true;
    const size_t words = wlcs::wide_scratch_words(xs_bytes, ys_bytes, uint32_t(pairs));
    WLCS_CUDA(c.ws2.ensure(wlcs::wide_workspace_bytes(uint32_t(pairs))));
    WLCS_CUDA(c.wcarry.ensure(2 * words * sizeof(uint16_t)));
    wlcs::WideDev w{};
    w.xs = d_xs;
    w.xoff = d_xoff;
    w.xs_bytes = xs_bytes;
    w.ys = d_ys;
    w.yoff = d_yoff;
    w.ys_bytes = ys_bytes;
    w.out = d_out;
    w.list = wlcs::batch_overflow_list_ptr(ws, uint32_t(pairs));
    w.count = wlcs::batch_overflow_count_ptr(ws, uint32_t(pairs));
    w.cap = uint32_t(pairs);
    w.pairs_total = uint32_t(pairs);
    w.carry[0] = c.wcarry.as<uint16_t>();
    w.carry[1] = c.wcarry.as<uint16_t>() + words;
    WLCS_CUDA(wlcs::wide_launch(w, c.ws2.p, c.sms, s));
    return WLCS_OK;
}

// Cell-wavefront variant of the batch (wavefront.cu): one kernel; pairs whose
// shorter string exceeds its shared-memory row go through the single-pair
// wavefront kernel afterwards (ids and offsets read back once, lengths
// written into d_out on the caller's stream).
int batch_wave(Ctx& c, const uint8_t* d_xs, const uint64_t* d_xoff, const uint8_t* d_ys,
               const uint64_t* d_yoff, size_t pairs, uint32_t* d_out, cudaStream_t stream) {
    WLCS_CUDA(c.ws.ensure(8 + size_t(pairs) * 4));
    wlcs::WaveBatchDev d{};
    d.xs = d_xs;
    d.xoff = d_xoff;
    d.ys = d_ys;
    d.yoff = d_yoff;
    d.out = d_out;
    d.pairs = uint32_t(pairs);
    d.counter = c.ws.as<uint32_t>();
    d.overflow_count = d.counter + 1;
    d.overflow = d.counter + 2;
    WLCS_CUDA(cudaMemsetAsync(d.counter, 0, 8, stream));
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev0, stream));
    WLCS_CUDA(wlcs::wave_batch_launch(d, c.sms, stream));
    if (c.timing) {
        WLCS_CUDA(cudaEventRecord(c.ev1, stream));
        c.timing_pending = true;
    }
    uint32_t* hov = reinterpret_cast<uint32_t*>(c.hscratch);
    WLCS_CUDA(cudaMemcpyAsync(hov, d.overflow_count, 4, cudaMemcpyDeviceToHost, stream));
    WLCS_CUDA(stream_wait(stream));
    const uint32_t overflow = *hov;
    if (overflow == 0) return WLCS_OK;
    std::vector<uint32_t> ids(overflow);
    WLCS_CUDA(cudaMemcpyAsync(ids.data(), d.overflow, overflow * 4, cudaMemcpyDeviceToHost, stream));
    WLCS_CUDA(stream_wait(stream));
    std::vector<uint64_t> xo(2 * size_t(overflow)), yo(2 * size_t(overflow));
    for (uint32_t k = 0; k < overflow; ++k) {
        WLCS_CUDA(cudaMemcpyAsync(&xo[2 * k], d_xoff + ids[k], 16, cudaMemcpyDeviceToHost, stream));
        WLCS_CUDA(cudaMemcpyAsync(&yo[2 * k], d_yoff + ids[k], 16, cudaMemcpyDeviceToHost, stream));
    }
    WLCS_CUDA(stream_wait(stream));
    std::vector<uint32_t> lens(overflow);
    for (uint32_t k = 0; k < overflow; ++k) {
        int rc = pair_wave_device(c, d_xs + xo[2 * k], size_t(xo[2 * k + 1] - xo[2 * k]),
                                  d_ys + yo[2 * k], size_t(yo[2 * k + 1] - yo[2 * k]), &lens[k]);
        if (rc) return rc;
    }
    for (uint32_t k = 0; k < overflow; ++k)
        WLCS_CUDA(cudaMemcpyAsync(d_out + ids[k], &lens[k], 4, cudaMemcpyHostToDevice, stream));
    WLCS_CUDA(stream_wait(stream));  // lens is a local array
    return WLCS_OK;
}

// Host batch with the host->device copies pipelined against the compute:
// the pairs are cut into nchunks contiguous chunks; chunk k's string bytes are
// copied on copy_stream while chunk k-1 runs on the compute stream (its own
// first-pass workspace, so the chunks' plans never overlap; the second pass's
// workspace is reused in stream order).  All copies are enqueued first and the
// offsets are validated on the host while they run (copy extents are clamped
// to the buffers, so invalid offsets cannot write outside them; nothing is
// computed before the check).  Pairs wider than the first pass's lane shapes
// are finished afterwards by the strip kernel (batch_long_pairs).
struct PipePlan {
    std::vector<size_t> p0, ws_off;
};

int batch_pipe_copies(Ctx& c, const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                      const uint64_t* y_off, size_t pairs, int nchunks, PipePlan& pp) {
    const uint64_t xs_bytes = x_off[pairs], ys_bytes = y_off[pairs];
    if (!c.copy_stream) WLCS_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    while (int(c.chunk_ev.size()) < nchunks) {
        cudaEvent_t e;
        WLCS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c.chunk_ev.push_back(e);
    }
    const int pm_bytes = batch_pm_bytes();
    // tapered chunks (weights nchunks, nchunks - 1, ..., 1): the compute of
    // each chunk hides under the next chunk's copy either way, and the last
    // chunk -- whose compute is the exposed tail after the final copy -- is
    // the smallest (WLCS_BATCH_TAPER=0: equal chunks)
    pp.p0.assign(nchunks + 1, 0);
    const bool taper = env_int("WLCS_BATCH_TAPER", 1) != 0;
    const size_t wsum = taper ? size_t(nchunks) * size_t(nchunks + 1) / 2 : size_t(nchunks);
    size_t wacc = 0;
    for (int k = 0; k <= nchunks; ++k) {
        pp.p0[k] = pairs * wacc / wsum;
        if (k < nchunks) wacc += taper ? size_t(nchunks - k) : 1;
    }
    pp.ws_off.assign(nchunks + 1, 0);
    for (int k = 0; k < nchunks; ++k)
        pp.ws_off[k + 1] = pp.ws_off[k] + ((wlcs::batch_workspace_bytes(
                                                uint32_t(pp.p0[k + 1] - pp.p0[k]), pm_bytes) +
                                            255) & ~size_t(255));
    WLCS_CUDA(c.ws.ensure(pp.ws_off[nchunks]));
    cudaStream_t cs = c.copy_stream;
    uint8_t* dxs = c.xs.as<uint8_t>();
    uint8_t* dys = c.ys.as<uint8_t>();
    WLCS_CUDA(cudaMemcpyAsync(c.xoff.p, x_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, cs));
    WLCS_CUDA(cudaMemcpyAsync(c.yoff.p, y_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, cs));
    for (int k = 0; k < nchunks; ++k) {
        const uint64_t xa = std::min(x_off[pp.p0[k]], xs_bytes);
        const uint64_t xb = std::min(x_off[pp.p0[k + 1]], xs_bytes);
        const uint64_t ya = std::min(y_off[pp.p0[k]], ys_bytes);
        const uint64_t yb = std::min(y_off[pp.p0[k + 1]], ys_bytes);
        if (xb > xa) WLCS_CUDA(cudaMemcpyAsync(dxs + xa, xs + xa, xb - xa, cudaMemcpyHostToDevice, cs));
        if (yb > ya) WLCS_CUDA(cudaMemcpyAsync(dys + ya, ys + ya, yb - ya, cudaMemcpyHostToDevice, cs));
        WLCS_CUDA(cudaEventRecord(c.chunk_ev[k], cs));
    }
    return WLCS_OK;
}

int batch_pipe_compute(Ctx& c, const uint64_t* x_off, const uint64_t* y_off, size_t pairs,
                       int nchunks, int kmax, const PipePlan& pp, uint32_t* out) {
    const uint64_t xs_bytes = x_off[pairs], ys_bytes = y_off[pairs];
    cudaStream_t s = c.stream;
    for (int k = 0; k < nchunks; ++k) {
        WLCS_CUDA(cudaStreamWaitEvent(s, c.chunk_ev[k], 0));
        if (int rc = batch_enqueue(c, c.xs.as<uint8_t>(), c.xoff.as<uint64_t>() + pp.p0[k],
                                   c.ys.as<uint8_t>(), c.yoff.as<uint64_t>() + pp.p0[k],
                                   pp.p0[k + 1] - pp.p0[k], xs_bytes, ys_bytes,
                                   c.out.as<uint32_t>() + pp.p0[k], s,
                                   c.ws.as<uint8_t>() + pp.ws_off[k], true, c.timing && k == 0,
                                   c.timing && k == nchunks - 1, kmax))
            return rc;
    }
    WLCS_CUDA(cudaMemcpyAsync(out, c.out.p, pairs * 4, cudaMemcpyDeviceToHost, s));
    WLCS_CUDA(stream_wait(s));
    return WLCS_OK;
}

// One pass over both offset arrays: non-decreasing (std::invalid_argument
// otherwise) and the pairs too wide for the first pass's lane shapes.
int scan_offsets(const uint64_t* x_off, const uint64_t* y_off, size_t pairs, int kmax,
                 bool want_long, std::vector<size_t>& long_ids) {
    const uint64_t lim = uint64_t(32) * 32 * uint64_t(kmax);  // columns of 32 * kmax words
    bool bad = false, any_long = false;
    for (size_t k = 0; k < pairs; ++k) {
        const uint64_t m = x_off[k + 1] - x_off[k], n = y_off[k + 1] - y_off[k];
        bad |= (x_off[k + 1] < x_off[k]) | (y_off[k + 1] < y_off[k]);
        any_long |= (m < n ? m : n) > lim;
    }
    if (bad) {
        for (size_t k = 0; k < pairs; ++k) {
            if (x_off[k + 1] < x_off[k])
                return fail(WLCS_E_INVALID_ARGUMENT, "x offsets decrease at pair " + std::to_string(k));
            if (y_off[k + 1] < y_off[k])
                return fail(WLCS_E_INVALID_ARGUMENT, "y offsets decrease at pair " + std::to_string(k));
        }
    }
    long_ids.clear();
    if (want_long && any_long)
        for (size_t k = 0; k < pairs; ++k)
            if (batch_is_long(x_off[k + 1] - x_off[k], y_off[k + 1] - y_off[k], kmax))
                long_ids.push_back(k);
    return WLCS_OK;
}

// Pairs the first pass cannot hold (batch_is_long) through the single-pair
// strip kernel, straight from the device copy of the strings.
int batch_long_pairs(Ctx& c, const uint8_t* dxs, const uint8_t* dys, const uint64_t* x_off,
                     const uint64_t* y_off, const std::vector<size_t>& ids, uint32_t* out) {
    for (size_t p : ids) {
        uint32_t len = 0;
        int rc = pair_length_device(c, dxs + x_off[p], size_t(x_off[p + 1] - x_off[p]),
                                    dys + y_off[p], size_t(y_off[p + 1] - y_off[p]), &len);
        if (rc) return rc;
        out[p] = len;
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


// ---- column split of G slices inside ONE launch on one device ------------
// The multi-GPU column split (wlcs_colsplit_fill per rank) with every rank's
// slice played as its own pair of problems (forward + reverse) of a single
// strip-kernel launch: slice g's first strips poll inboxes that slice g-1 /
// g+1's last strips fill while running -- the same fused hand-off as between
// GPUs, but the "ranks" are co-resident CTA pools of one grid (no separate
// launches that wait on each other).  max_ctas caps the grid so that a test
// can run with fewer warps per pool than strips per problem (liveness).
// L = max_k F[k] + R[N-k] as in wlcs_length_strips.
int split_combine_host(int G, const std::vector<size_t>& lo, const std::vector<size_t>& hi,
                       const std::vector<std::vector<uint32_t>>& vf,
                       const std::vector<std::vector<uint32_t>>& vr, size_t N, uint32_t* out) {
    std::vector<int64_t> F(N + 1, 0), R(N + 1, 0);
    size_t k = 0;
    for (int g = 0; g < G; ++g)
        for (size_t c = 0; c < hi[g] - lo[g]; ++c, ++k)
            F[k + 1] = F[k] + (((vf[g][c >> 5] >> (c & 31)) & 1u) ? 0 : 1);
    k = 0;
    for (int g = G - 1; g >= 0; --g)
        for (size_t c = 0; c < hi[g] - lo[g]; ++c, ++k)
            R[k + 1] = R[k] + (((vr[g][c >> 5] >> (c & 31)) & 1u) ? 0 : 1);
    int64_t best = 0;
    for (size_t kk = 0; kk <= N; ++kk) best = std::max(best, F[kk] + R[N - kk]);
    *out = uint32_t(best);
    return WLCS_OK;
}

}  // namespace

extern "C" int wlcs_colsplit_emulate(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                                     int slices, int max_ctas, uint32_t* out) {
    if (!x || !y || !out) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    const int G = slices;
    if (G < 1 || 2 * G > wlcs::kMaxProblems)
        return fail(WLCS_E_INVALID_ARGUMENT, "slices must be 1 .. " +
                                                 std::to_string(wlcs::kMaxProblems / 2));
    if (m < 2 || n < size_t(32) * size_t(G))
        return fail(WLCS_E_INVALID_ARGUMENT, "column split needs m >= 2 and n >= 32 * slices");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    WLCS_CUDA(c->ry.ensure(n + 16));
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y, n, c->stream)) return rc_;
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dy = c->py.as<uint8_t>();
    uint8_t* dry = c->ry.as<uint8_t>();
    WLCS_CUDA(wlcs::pair_reverse(dy, int64_t(n), dry, c->stream));
    // slice bounds on word boundaries (wlcs_length_strips)
    std::vector<size_t> lo(G), hi(G);
    const size_t words = (n + 31) / 32;
    for (int g = 0; g < G; ++g) {
        lo[g] = std::min(n, words * g / G * 32);
        hi[g] = std::min(n, words * (g + 1) / G * 32);
    }
    wlcs::PairDev d{};
    d.colp0 = dy;
    d.prob[0].cols = int64_t(n);  // alphabet of the whole column string
    WLCS_CUDA(c->small.ensure(4096));
    uint8_t* sb = c->small.as<uint8_t>();
    uint16_t* map = reinterpret_cast<uint16_t*>(sb + 1024);
    d.ticket = reinterpret_cast<uint32_t*>(sb + kTicketOff);
    d.error = reinterpret_cast<uint32_t*>(sb + kErrOff);
    d.safe16 = reinterpret_cast<const uint4*>(sb + 2048);
    WLCS_CUDA(c->sink.ensure(size_t(wlcs::kPairSinkWords) * 4));
    d.sink = c->sink.as<uint32_t>();
    int sigma = 0;
    WLCS_CUDA(wlcs::pair_prepare(d, reinterpret_cast<uint32_t*>(sb), map,
                                 reinterpret_cast<uint32_t*>(sb + 1536), c->stream, &sigma));
    const int64_t mid = int64_t(m / 2);
    int64_t wmax = 0;
    for (int g = 0; g < G; ++g) wmax = std::max<int64_t>(wmax, int64_t(hi[g] - lo[g] + 31) / 32);
    const int K = choose_k(*c, wmax, int64_t(m) - mid, d, 2 * G);
    if (wlcs::pair_smem_bytes(K, sigma) > 220 * 1024)
        return fail(WLCS_E_INTERNAL, "match-mask table does not fit in shared memory");
    d.nprob = 2 * G;
    d.max_ctas = max_ctas;
    // per problem: masks [sigma][W_g]; final vectors; carries
    size_t pm_total = 0, v_total = 0;
    for (int g = 0; g < G; ++g) {
        const size_t Wg = (hi[g] - lo[g] + 31) / 32;
        pm_total += 2 * size_t(sigma) * Wg;
        v_total += 2 * Wg;
    }
    WLCS_CUDA(c->pmg.ensure(pm_total * 4));
    WLCS_CUDA(c->vbuf.ensure(v_total * 4 + 64));
    // row codes are shared by every slice of a direction
    wlcs::FillProblem fwd{}, rev{};
    fwd.rows = mid;
    fwd.nchunks = int((mid + 15) / 16);
    rev.rows = int64_t(m) - mid;
    rev.nchunks = int((rev.rows + 15) / 16);
    const size_t code_vecs =
        4 * size_t(wlcs::pair_code_plane(fwd.nchunks) + wlcs::pair_code_plane(rev.nchunks));
    WLCS_CUDA(c->codes.ensure(code_vecs * 16));
    uint4* code_base = c->codes.as<uint4>();
    WLCS_CUDA(wlcs::pair_code_rows(dx, fwd.rows, false, map, K, fwd, code_base, c->stream));
    WLCS_CUDA(wlcs::pair_code_rows(dx + mid, rev.rows, true, map, K, rev,
                                   code_base + 4 * wlcs::pair_code_plane(fwd.nchunks), c->stream));
    size_t inbox_words = 0;
    rc = wlcs_colsplit_inbox_words(m, &inbox_words);
    if (rc) return rc;
    size_t carry_words = 2 * size_t(G) * inbox_words;  // inboxes first
    uint32_t* pmg = c->pmg.as<uint32_t>();
    uint32_t* vb = c->vbuf.as<uint32_t>();
    for (int g = 0; g < G; ++g) {
        const int64_t cols = int64_t(hi[g] - lo[g]);
        const int64_t Wg = (cols + 31) / 32;
        for (int dir = 0; dir < 2; ++dir) {
            wlcs::FillProblem& P = d.prob[2 * g + dir];
            const wlcs::FillProblem& R = dir == 0 ? fwd : rev;
            set_problem(P, R.rows, pmg, cols, K);
            P.coded = R.coded;
            P.plane = R.plane;
            P.cstride = R.cstride;
            P.v_out = vb;
            WLCS_CUDA(wlcs::pair_build_pm(dir == 0 ? dy + lo[g] : dry + (n - hi[g]), cols, map,
                                          sigma, Wg, pmg, c->stream));
            pmg += size_t(sigma) * size_t(Wg);
            vb += Wg;
            carry_words += size_t(P.nstrips) * size_t(P.cwords);
        }
    }
    WLCS_CUDA(c->carry.ensure(carry_words * 4 + 256));
    uint32_t* inbox_f = c->carry.as<uint32_t>();                         // [G][inbox_words]
    uint32_t* inbox_r = inbox_f + size_t(G) * inbox_words;               // [G][inbox_words]
    uint32_t* carry = inbox_r + size_t(G) * inbox_words;
    for (int g = 0; g < G; ++g) {
        wlcs::FillProblem& F = d.prob[2 * g];
        wlcs::FillProblem& R = d.prob[2 * g + 1];
        F.ext_in = g > 0 ? inbox_f + size_t(g) * inbox_words : nullptr;
        F.ext_out = g + 1 < G ? inbox_f + size_t(g + 1) * inbox_words : nullptr;
        R.ext_in = g + 1 < G ? inbox_r + size_t(g) * inbox_words : nullptr;
        R.ext_out = g > 0 ? inbox_r + size_t(g - 1) * inbox_words : nullptr;
        for (wlcs::FillProblem* P : {&F, &R}) {
            P->carry = carry;
            carry += size_t(P->nstrips) * size_t(P->cwords);
        }
    }
    WLCS_CUDA(cudaMemsetAsync(c->carry.p, 0, carry_words * 4, c->stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 1540, 0, kTicketOff + 4 * wlcs::kMaxProblems - 1540, c->stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 2048, 0, 16, c->stream));
    if (c->timing && !c->ev0) {
        WLCS_CUDA(cudaEventCreate(&c->ev0));
        WLCS_CUDA(cudaEventCreate(&c->ev1));
    }
    if (c->timing) WLCS_CUDA(cudaEventRecord(c->ev0, c->stream));
    WLCS_CUDA(wlcs::pair_fill(d, K, false, c->sms, c->stream));
    if (c->timing) WLCS_CUDA(cudaEventRecord(c->ev1, c->stream));
    std::vector<uint32_t> vall(v_total);
    WLCS_CUDA(cudaMemcpyAsync(vall.data(), c->vbuf.p, v_total * 4, cudaMemcpyDeviceToHost, c->stream));
    rc = watchdog_read(*c, c->stream);
    if (rc) return rc;
    WLCS_CUDA(stream_wait(c->stream));
    rc = watchdog_failed(*c);
    if (rc) return rc;
    if (c->timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c->last_main_ms, c->ev0, c->ev1));
        c->timing_pending = false;
    }
    std::vector<std::vector<uint32_t>> vf(G), vr(G);
    size_t off = 0;
    for (int g = 0; g < G; ++g) {
        const size_t Wg = (hi[g] - lo[g] + 31) / 32;
        vf[g].assign(vall.begin() + off, vall.begin() + off + Wg);
        vr[g].assign(vall.begin() + off + Wg, vall.begin() + off + 2 * Wg);
        off += 2 * Wg;
    }
    return split_combine_host(G, lo, hi, vf, vr, n, out);
}

namespace {
// ---- recovered subsequence ------------------------------------------------
// Two ways to the same bytes (the reference's traceback, serial.cpp:36-61,
// with the LEFT rule of cell.hpp:30-38):
//  * full:   one fill that stores every row's bit vector (M * N / 8 bytes),
//            then the parallel walk (bitpar_pair.cu pair_walk);
//  * banded: bounded memory -- a first fill keeps only every B-th row's bit
//            vector (checkpoints, (M / B) * N / 8 bytes); then, from the
//            bottom band up, each band of B rows is filled again from its
//            checkpoint with its rows stored (B * N / 8 bytes) and walked from
//            the column where the band below was left.  Same rows, same walk
//            rule, hence the same string; memory O(N (M / B + B)) instead of
//            O(M N), for about twice the fill work.
// The band size comes from `row_cap` (bytes of stored bit rows +
// checkpoints); row_cap = 0 picks the full path while it fits an automatic
// cap (half the free device memory, at most 8 GiB) and bands beyond it.

// bytes of stored bit rows for `rows` rows of problem P at K words per lane
size_t store_bytes(const wlcs::FillProblem& P, int K, int64_t rows) {
    const int64_t mpad = (rows + 15) / 16 * 16;
    return size_t(P.nstrips) * 32 * size_t(mpad + 512) * size_t(K) * 4;
}

// band rows B (a multiple of the walk's 256-row blocks) so that the stored
// band plus the checkpoints fit `cap`; 0 when even 256 rows do not fit
int64_t band_rows_for(const wlcs::FillProblem& P, int K, int64_t M, size_t cap) {
    for (int64_t B = ((M + 255) / 256) * 256; B >= 256; B -= (B > 4096 ? B / 8 / 256 * 256 : 256)) {
        const int64_t nb = (M + B - 1) / B;
        const size_t need = store_bytes(P, K, B) + size_t(nb - 1) * size_t(P.W) * 4;
        if (need <= cap) return B;
        if (B <= 4096 && B - 256 < 256) break;
    }
    return 0;
}

int subsequence_banded(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                       size_t cap, unsigned long long* len_out) {
    PairPlan plan;
    int rc = pair_setup(c, dx, int64_t(m), dy, int64_t(n), false, plan, /*allow_split=*/false);
    if (rc) return rc;
    wlcs::PairDev& d = plan.d;
    const int K = plan.K;
    const wlcs::FillProblem full = d.prob[0];
    const int64_t M = full.rows, W = full.W;
    const int64_t B = band_rows_for(full, K, M, cap);
    if (B == 0)
        return fail(WLCS_E_OUT_OF_MEMORY,
                    "traceback memory cap of " + std::to_string(cap) +
                        " bytes is below one 256-row band (" +
                        std::to_string(store_bytes(full, K, 256)) + " bytes)");
    const int64_t nbands = (M + B - 1) / B;
    // pass 1: the whole fill, keeping V after every B rows (and the length)
    WLCS_CUDA(c.ckpt.ensure(size_t(std::max<int64_t>(nbands - 1, 1)) * size_t(W) * 4));
    d.prob[0].ckpt_out = c.ckpt.as<uint32_t>();
    d.prob[0].ckpt_chunks = int(B / 16);
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev0, c.stream));
    WLCS_CUDA(wlcs::pair_fill(d, K, false, c.sms, c.stream));
    // the walk's state between bands: entry column, {L, bytes emitted}
    uint8_t* sb = c.small.as<uint8_t>();
    unsigned long long* zeros_dev = pair_zeros_ptr(c);
    int32_t* d_entry = reinterpret_cast<int32_t*>(sb + 1704);
    unsigned long long* d_place = reinterpret_cast<unsigned long long*>(sb + 1712);
    int32_t* h_entry = reinterpret_cast<int32_t*>(c.hscratch + 8);
    *h_entry = int32_t(n);
    WLCS_CUDA(cudaMemcpyAsync(d_entry, h_entry, 4, cudaMemcpyHostToDevice, c.stream));
    WLCS_CUDA(cudaMemcpyAsync(d_place, zeros_dev, 8, cudaMemcpyDeviceToDevice, c.stream));
    WLCS_CUDA(cudaMemsetAsync(d_place + 1, 0, 8, c.stream));
    // band buffers
    WLCS_CUDA(c.rows.ensure(store_bytes(full, K, B)));
    WLCS_CUDA(c.bandcodes.ensure(4 * size_t(wlcs::pair_code_plane(int(B / 16))) * 16));
    WLCS_CUDA(c.walk.ensure(wlcs::pair_walk_scratch_bytes(B)));
    const size_t maxlen = std::min(m, n);
    WLCS_CUDA(c.outrev.ensure(maxlen + 16));
    unsigned long long* dlen = zeros_dev + 1;
    uint32_t* dmiss = reinterpret_cast<uint32_t*>(zeros_dev + 2);
    for (int64_t b = nbands - 1; b >= 0; --b) {
        const int64_t r0 = b * B, rb = std::min<int64_t>(B, M - r0);
        wlcs::FillProblem Pb = full;
        set_problem(Pb, rb, const_cast<uint32_t*>(full.pmg), full.cols, K);
        Pb.carry = c.carry.as<uint32_t>();
        Pb.v_in = b > 0 ? c.ckpt.as<uint32_t>() + (b - 1) * W : nullptr;
        Pb.ckpt_out = nullptr;
        Pb.zeros = nullptr;
        Pb.v_out = nullptr;
        Pb.rows_out = c.rows.as<uint32_t>();
        Pb.walk_row0 = r0;
        Pb.walk_mtot = M;
        Pb.walk_entry = d_entry;
        Pb.walk_place = d_place;
        WLCS_CUDA(wlcs::pair_code_rows(dx + r0, rb, false, d.map, K, Pb, c.bandcodes.as<uint4>(),
                                       c.stream));
        WLCS_CUDA(cudaMemsetAsync(Pb.carry, 0, size_t(Pb.nstrips) * size_t(Pb.cwords) * 4,
                                  c.stream));
        WLCS_CUDA(cudaMemsetAsync(d.ticket, 0, 4 * wlcs::kMaxProblems, c.stream));
        wlcs::PairDev db = d;
        db.nprob = 1;
        db.prob[0] = Pb;
        WLCS_CUDA(wlcs::pair_fill(db, K, true, c.sms, c.stream));
        WLCS_CUDA(wlcs::pair_walk(db, K, dx + r0, c.outrev.as<uint8_t>(), dlen, c.walk.p, dmiss,
                                  c.stream));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev1, c.stream));
    WLCS_CUDA(cudaMemcpyAsync(c.hscratch, d_place, 16, cudaMemcpyDeviceToHost, c.stream));
    WLCS_CUDA(stream_wait(c.stream));
    if (c.timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c.last_main_ms, c.ev0, c.ev1));
        c.timing_pending = false;
    }
    if (c.hscratch[1] != c.hscratch[0])
        return fail(WLCS_E_INTERNAL, "banded traceback emitted " + std::to_string(c.hscratch[1]) +
                                         " bytes for an LCS of length " +
                                         std::to_string(c.hscratch[0]));
    *len_out = c.hscratch[0];
    return WLCS_OK;
}

int subsequence_full(Ctx& c, const uint8_t* dx, size_t m, const uint8_t* dy, size_t n,
                     unsigned long long* len_out) {
    // Orientation matters for tie-breaking: rows = x (parent), columns = y.
    PairPlan plan;
    int rc = pair_setup(c, dx, int64_t(m), dy, int64_t(n), true, plan);
    if (rc) return rc;
    if (c.timing && !c.ev0) {
        WLCS_CUDA(cudaEventCreate(&c.ev0));
        WLCS_CUDA(cudaEventCreate(&c.ev1));
    }
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev0, c.stream));
    WLCS_CUDA(wlcs::pair_fill(plan.d, plan.K, true, c.sms, c.stream));
    if (c.timing) WLCS_CUDA(cudaEventRecord(c.ev1, c.stream));
    const size_t maxlen = std::min(m, n);
    WLCS_CUDA(c.outrev.ensure(maxlen + 16));
    unsigned long long* zeros_dev = pair_zeros_ptr(c);
    unsigned long long* dlen = zeros_dev + 1;
    WLCS_CUDA(c.walk.ensure(wlcs::pair_walk_scratch_bytes(int64_t(m))));
    uint32_t* dmiss = reinterpret_cast<uint32_t*>(zeros_dev + 2);
    WLCS_CUDA(wlcs::pair_walk(plan.d, plan.K, dx, c.outrev.as<uint8_t>(), dlen, c.walk.p, dmiss,
                              c.stream));
    WLCS_CUDA(cudaMemcpyAsync(c.hscratch, dlen, 8, cudaMemcpyDeviceToHost, c.stream));
    WLCS_CUDA(cudaMemcpyAsync(c.hscratch + 1, zeros_dev, 8, cudaMemcpyDeviceToHost, c.stream));
    WLCS_CUDA(stream_wait(c.stream));
    const unsigned long long len = c.hscratch[0], zeros = c.hscratch[1];
    if (c.timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c.last_main_ms, c.ev0, c.ev1));
        c.timing_pending = false;
    }
    if (env_int("WLCS_DEBUG_WALK", 0)) {
        uint32_t miss[3] = {0, 0, 0};
        WLCS_CUDA(cudaMemcpy(miss, dmiss, 12, cudaMemcpyDeviceToHost));
        std::fprintf(stderr,
                     "wlcs walk: %u of %lld blocks resolved by a fallback walk (resolve: %u of "
                     "%u kcycles in fallbacks)\n",
                     miss[0], (long long)((m + 255) / 256), miss[1], miss[2]);
    }
    if (len != zeros)
        return fail(WLCS_E_INTERNAL, "traceback length " + std::to_string(len) +
                                         " differs from the fill length " + std::to_string(zeros));
    *len_out = len;
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
    if (variant != WLCS_VARIANT_BITPARALLEL && variant != WLCS_VARIANT_WAVEFRONT)
        return fail(WLCS_E_CONFIG, "unknown fill variant " + std::to_string(variant));
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y, n, c->stream)) return rc_;
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dy = c->py.as<uint8_t>();
    return pair_length_variant(*c, dx, m, dy, n, variant, out);
}

int wlcs_length(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t memory_budget,
                uint32_t* out) {
    return wlcs_length_ex(x, m, y, n, memory_budget, WLCS_VARIANT_BITPARALLEL, out);
}

// Row-band decomposition (seaweed.cu): the rows of x in `bands` equal bands,
// each combed independently, composed through their DP boundaries.
int wlcs_length_rowbands(const uint8_t* x, size_t m, const uint8_t* y, size_t n, int bands,
                         uint32_t* out) {
    if (!out) return fail(WLCS_E_INVALID_ARGUMENT, "out is NULL");
    if ((m && !x) || (n && !y)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL input");
    if (bands < 1) return fail(WLCS_E_INVALID_ARGUMENT, "bands must be >= 1");
    if (m == 0 || n == 0) {
        *out = 0;
        return WLCS_OK;
    }
    if (n >= (size_t(1) << 31) || m >= (size_t(1) << 31))
        return fail(WLCS_E_CONFIG, "row-band prototype: strings must be < 2^31 bytes");
    if (size_t(bands) > m) bands = int(m);
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y, n, c->stream)) return rc_;
    // [row_lo: bands + 1 int64][out][v: bands * n][e: bands * n][t0, t1: n + 1]
    const size_t lo_bytes = (size_t(bands) + 1) * 8 + 16;
    const size_t vb = size_t(bands) * n * 4;
    WLCS_CUDA(c->sea.ensure(lo_bytes + 2 * vb + 2 * (n + 1) * 4 + 64));
    uint8_t* base = c->sea.as<uint8_t>();
    std::vector<int64_t> lo(size_t(bands) + 1);
    for (int b = 0; b <= bands; ++b) lo[size_t(b)] = int64_t(m * size_t(b) / size_t(bands));
    WLCS_CUDA(cudaMemcpyAsync(base, lo.data(), lo.size() * 8, cudaMemcpyHostToDevice, c->stream));
    uint32_t* d_out = reinterpret_cast<uint32_t*>(base + lo_bytes - 16);
    wlcs::SeaDev d{};
    d.rowp = c->px.as<uint8_t>();
    d.row_lo = reinterpret_cast<const int64_t*>(base);
    d.colp = c->py.as<uint8_t>();
    d.n = int64_t(n);
    d.v = reinterpret_cast<uint32_t*>(base + lo_bytes);
    d.e = d.v + size_t(bands) * n;
    uint32_t* t0 = d.e + size_t(bands) * n;
    uint32_t* t1 = t0 + (n + 1);
    WLCS_CUDA(wlcs::seaweed_bands(d, bands, t0, t1, d_out, c->stream));
    uint32_t* h = reinterpret_cast<uint32_t*>(c->hscratch);
    WLCS_CUDA(cudaMemcpyAsync(h, d_out, 4, cudaMemcpyDeviceToHost, c->stream));
    WLCS_CUDA(stream_wait(c->stream));
    *out = *h;
    return WLCS_OK;
}

int wlcs_length_device(const uint8_t* d_x, size_t m, const uint8_t* d_y, size_t n, int variant,
                       uint32_t* out, void* stream) {
    if (!out) return fail(WLCS_E_INVALID_ARGUMENT, "out is NULL");
    if ((reinterpret_cast<uintptr_t>(d_x) | reinterpret_cast<uintptr_t>(d_y)) & 15u)
        return fail(WLCS_E_INVALID_ARGUMENT, "device string buffers must be 16-byte aligned");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    if (variant != WLCS_VARIANT_BITPARALLEL && variant != WLCS_VARIANT_WAVEFRONT)
        return fail(WLCS_E_CONFIG, "unknown fill variant " + std::to_string(variant));
    // the strings may still be in flight on the caller's stream
    rc = join_caller(*c, caller_stream(stream));
    if (rc) return rc;
    return pair_length_variant(*c, d_x, m, d_y, n, variant, out);
}

int wlcs_subsequence_ex(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                                   size_t memory_budget, size_t row_cap, uint8_t* out, size_t cap,
                                   size_t* out_len) {
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
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y, n, c->stream)) return rc_;
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dy = c->py.as<uint8_t>();
    // stored-row bytes of the full path (the strip plan's geometry, K = the
    // cost model's choice for a store fill)
    const int64_t W = (int64_t(n) + 31) / 32;
    // full store needs about M * 32 * ceil(W / 32 / K) * K * 4 bytes >= M * N / 8
    const double full_est = double(m + 528) * double((W + 31) / 32 * 32) * 4.0;
    size_t limit = row_cap;
    if (limit == 0) {
        // automatic cap, at most 8 GiB: the full bit-row store whenever it can
        // be allocated (the buffer is reserved here, so the fill's own request
        // finds it), else half the free memory (banded).  No cudaMemGetInfo on
        // the common path: it costs ~70 us per call, and a free-memory reading
        // taken while other allocations come and go must not flip a call to
        // the ~7x slower banded traceback.
        const size_t kAutoCap = size_t(8) << 30;
        bool fits = false;
        if (full_est <= double(kAutoCap)) {
            const size_t want = size_t(full_est * 1.02) + (size_t(1) << 20);
            fits = c->rows.ensure(want) == cudaSuccess;
            if (!fits) (void)cudaGetLastError();
        }
        if (fits) {
            limit = kAutoCap;
        } else {
            size_t free_b = 0, total_b = 0;
            WLCS_CUDA(cudaMemGetInfo(&free_b, &total_b));
            limit = std::min<size_t>(free_b / 2, kAutoCap);
        }
    }
    unsigned long long len = 0;
    rc = full_est <= double(limit) ? subsequence_full(*c, dx, m, dy, n, &len)
                                   : subsequence_banded(*c, dx, m, dy, n, limit, &len);
    if (rc) return rc;
    *out_len = size_t(len);
    if (len > cap)
        return fail(WLCS_E_INVALID_ARGUMENT, "output buffer holds " + std::to_string(cap) +
                                                 " bytes, subsequence has " + std::to_string(len));
    if (len) WLCS_CUDA(cudaMemcpy(out, c->outrev.p, len, cudaMemcpyDeviceToHost));
    return WLCS_OK;
}

int wlcs_subsequence(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                     size_t memory_budget, uint8_t* out, size_t cap, size_t* out_len) {
    return wlcs_subsequence_ex(x, m, y, n, memory_budget, 0, out, cap, out_len);
}

int wlcs_length_batch_device(const uint8_t* d_xs, const uint64_t* d_x_off, const uint8_t* d_ys,
                             const uint64_t* d_y_off, size_t pairs, uint64_t xs_bytes,
                             uint64_t ys_bytes, int variant, uint32_t* d_out, void* stream) {
    if ((reinterpret_cast<uintptr_t>(d_xs) | reinterpret_cast<uintptr_t>(d_ys)) & 15u)
        return fail(WLCS_E_INVALID_ARGUMENT, "device string buffers must be 16-byte aligned");
    if (pairs > 0x7fffffffull) return fail(WLCS_E_INVALID_ARGUMENT, "too many pairs in one batch");
    if (variant != WLCS_VARIANT_BITPARALLEL && variant != WLCS_VARIANT_WAVEFRONT)
        return fail(WLCS_E_CONFIG, "unknown fill variant " + std::to_string(variant));
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    if (pairs == 0) return WLCS_OK;
    const cudaStream_t s = caller_stream(stream);
    if (variant == WLCS_VARIANT_WAVEFRONT) {
        rc = join_caller(*c, s);
        if (rc) return rc;
        return batch_wave(*c, d_xs, d_x_off, d_ys, d_y_off, pairs, d_out, s);
    }
    WLCS_CUDA(c->ws.ensure(wlcs::batch_workspace_bytes(uint32_t(pairs), batch_pm_bytes())));
    return batch_enqueue(*c, d_xs, d_x_off, d_ys, d_y_off, pairs, xs_bytes, ys_bytes, d_out, s,
                         c->ws.p, false, c->timing, c->timing, batch_kmax(pairs));
}

int wlcs_length_batch_ex(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                         const uint64_t* y_off, size_t pairs, int variant, uint32_t* out) {
    if (pairs == 0) return WLCS_OK;
    if (!x_off || !y_off || !out) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    if (pairs > 0x7fffffffull) return fail(WLCS_E_INVALID_ARGUMENT, "too many pairs in one batch");
    if (variant != WLCS_VARIANT_BITPARALLEL && variant != WLCS_VARIANT_WAVEFRONT)
        return fail(WLCS_E_CONFIG, "unknown fill variant " + std::to_string(variant));
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    const uint64_t xs_bytes = x_off[pairs], ys_bytes = y_off[pairs];
    if ((xs_bytes && !xs) || (ys_bytes && !ys)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL strings");
    WLCS_CUDA(c->xs.ensure(xs_bytes + 16));
    WLCS_CUDA(c->ys.ensure(ys_bytes + 16));
    WLCS_CUDA(c->xoff.ensure((pairs + 1) * 8));
    WLCS_CUDA(c->yoff.ensure((pairs + 1) * 8));
    WLCS_CUDA(c->out.ensure(pairs * 4));
    cudaStream_t s = c->stream;
    // pairs too wide for the first pass's lane shapes go to the strip kernel
    // (the host knows the offsets, so they never reach the device second pass)
    std::vector<size_t> long_ids;
    const int kmax = batch_kmax(pairs);
    const bool bitpar = variant == WLCS_VARIANT_BITPARALLEL;
    const int nchunks =
        bitpar ? int(std::min<size_t>(std::min<size_t>(size_t(env_int("WLCS_BATCH_CHUNKS", 3)), 64),
                                      pairs / 8192))
               : 1;
    if (nchunks >= 2 && xs_bytes + ys_bytes >= (16u << 20)) {
        PipePlan pp;
        rc = batch_pipe_copies(*c, xs, x_off, ys, y_off, pairs, nchunks, pp);
        if (rc) return rc;
        rc = scan_offsets(x_off, y_off, pairs, kmax, true, long_ids);  // while the DMA runs
        if (rc) {
            cudaStreamSynchronize(c->copy_stream);  // the copies read the caller's buffers
            return rc;
        }
        rc = batch_pipe_compute(*c, x_off, y_off, pairs, nchunks, kmax, pp, out);
        if (rc) return rc;
        return batch_long_pairs(*c, c->xs.as<uint8_t>(), c->ys.as<uint8_t>(), x_off, y_off,
                                long_ids, out);
    }
    rc = scan_offsets(x_off, y_off, pairs, kmax, bitpar, long_ids);
    if (rc) return rc;
    if (xs_bytes) WLCS_CUDA(cudaMemcpyAsync(c->xs.p, xs, xs_bytes, cudaMemcpyHostToDevice, s));
    if (ys_bytes) WLCS_CUDA(cudaMemcpyAsync(c->ys.p, ys, ys_bytes, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(c->xoff.p, x_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(c->yoff.p, y_off, (pairs + 1) * 8, cudaMemcpyHostToDevice, s));
    if (!bitpar) {
        rc = batch_wave(*c, c->xs.as<uint8_t>(), c->xoff.as<uint64_t>(), c->ys.as<uint8_t>(),
                        c->yoff.as<uint64_t>(), pairs, c->out.as<uint32_t>(), s);
    } else {
        WLCS_CUDA(c->ws.ensure(wlcs::batch_workspace_bytes(uint32_t(pairs), batch_pm_bytes())));
        rc = batch_enqueue(*c, c->xs.as<uint8_t>(), c->xoff.as<uint64_t>(), c->ys.as<uint8_t>(),
                           c->yoff.as<uint64_t>(), pairs, xs_bytes, ys_bytes,
                           c->out.as<uint32_t>(), s, c->ws.p, true, c->timing, c->timing, kmax);
    }
    if (rc) return rc;
    WLCS_CUDA(cudaMemcpyAsync(out, c->out.p, pairs * 4, cudaMemcpyDeviceToHost, s));
    WLCS_CUDA(stream_wait(s));
    return batch_long_pairs(*c, c->xs.as<uint8_t>(), c->ys.as<uint8_t>(), x_off, y_off, long_ids,
                            out);
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
    c->timing_pending = false;
    return WLCS_OK;
}

int wlcs_last_kernel_ms(float* ms) {
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    if (c->timing_pending) {  // an asynchronous batch: wait for its end event only
        WLCS_CUDA(cudaEventSynchronize(c->ev1));
        WLCS_CUDA(cudaEventElapsedTime(&c->last_main_ms, c->ev0, c->ev1));
        c->timing_pending = false;
    }
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

// ------------------------------------------------------- column split
int wlcs_colsplit_inbox_words(size_t m, size_t* words) {
    if (!words) return fail(WLCS_E_INVALID_ARGUMENT, "words is NULL");
    const size_t rows = m - m / 2;  // the larger half
    const size_t nch = (rows + 15) / 16;
    *words = ((nch + 3) & ~size_t(3)) + 16;
    return WLCS_OK;
}

int wlcs_colsplit_fill(const uint8_t* x, size_t m, const uint8_t* y, size_t n, size_t col_lo,
                       size_t col_hi, int problems, const uint32_t* d_in_fwd,
                       uint32_t* d_out_fwd, const uint32_t* d_in_rev, uint32_t* d_out_rev,
                       uint32_t* v_fwd, uint32_t* v_rev) {
    if (!x || !y) return fail(WLCS_E_INVALID_ARGUMENT, "NULL input");
    if (m < 2) return fail(WLCS_E_INVALID_ARGUMENT, "column split needs at least 2 rows");
    if (!(col_lo < col_hi && col_hi <= n))
        return fail(WLCS_E_INVALID_ARGUMENT, "column slice out of range");
    if (problems < 1 || problems > 3) return fail(WLCS_E_INVALID_ARGUMENT, "bad problems mask");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    const int64_t cols = int64_t(col_hi - col_lo);
    const int64_t W = (cols + 31) / 32;
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(size_t(cols) + 16));
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y + col_lo, size_t(cols), c->stream)) return rc_;
    const uint8_t* dx = c->px.as<uint8_t>();
    const uint8_t* dcol = c->py.as<uint8_t>();
    wlcs::PairDev d{};
    d.colp0 = dcol;
    d.prob[0].cols = cols;
    WLCS_CUDA(c->small.ensure(4096));
    uint8_t* sb = c->small.as<uint8_t>();
    uint16_t* map = reinterpret_cast<uint16_t*>(sb + 1024);
    d.ticket = reinterpret_cast<uint32_t*>(sb + kTicketOff);
    d.error = reinterpret_cast<uint32_t*>(sb + kErrOff);
    d.safe16 = reinterpret_cast<const uint4*>(sb + 2048);
    WLCS_CUDA(c->sink.ensure(size_t(wlcs::kPairSinkWords) * 4));
    d.sink = c->sink.as<uint32_t>();
    int sigma = 0;
    WLCS_CUDA(wlcs::pair_prepare(d, reinterpret_cast<uint32_t*>(sb), map,
                                 reinterpret_cast<uint32_t*>(sb + 1536), c->stream, &sigma));
    const int64_t mid = int64_t(m / 2);
    const bool want[2] = {(problems & WLCS_COLSPLIT_FORWARD) != 0,
                          (problems & WLCS_COLSPLIT_REVERSE) != 0};
    d.nprob = (want[0] ? 1 : 0) + (want[1] ? 1 : 0);
    const int K = choose_k(*c, W, int64_t(m) - mid, d, d.nprob);
    if (wlcs::pair_smem_bytes(K, sigma) > 220 * 1024)
        return fail(WLCS_E_INTERNAL, "match-mask table does not fit in shared memory");
    const size_t pm_words = size_t(sigma) * size_t(W);
    WLCS_CUDA(c->pmg.ensure(pm_words * 4 * 2));
    WLCS_CUDA(c->vbuf.ensure(size_t(W) * 8 + 64));
    WLCS_CUDA(c->ry.ensure(size_t(cols) + 16));
    uint32_t* pmg = c->pmg.as<uint32_t>();
    int q = 0;
    size_t code_vecs = 0;
    int which[2];
    for (int dir = 0; dir < 2; ++dir) {
        if (!want[dir]) continue;
        wlcs::FillProblem& P = d.prob[q];
        set_problem(P, dir == 0 ? mid : int64_t(m) - mid, pmg + pm_words * dir, cols, K);
        P.v_out = c->vbuf.as<uint32_t>() + W * dir;
        P.ext_in = dir == 0 ? d_in_fwd : d_in_rev;
        P.ext_out = dir == 0 ? d_out_fwd : d_out_rev;
        code_vecs += 4 * size_t(wlcs::pair_code_plane(P.nchunks));
        which[q++] = dir;
    }
    WLCS_CUDA(c->codes.ensure(code_vecs * 16));
    uint4* code_base = c->codes.as<uint4>();
    size_t carry_words = 0;
    for (int k = 0; k < d.nprob; ++k) {
        wlcs::FillProblem& P = d.prob[k];
        const bool rev = which[k] == 1;
        WLCS_CUDA(wlcs::pair_code_rows(rev ? dx + mid : dx, P.rows, rev, map, K, P, code_base,
                                       c->stream));
        code_base += 4 * wlcs::pair_code_plane(P.nchunks);
        carry_words += size_t(P.nstrips) * size_t(P.cwords);
    }
    WLCS_CUDA(c->carry.ensure(carry_words * 4 + 256));
    uint32_t* carry = c->carry.as<uint32_t>();
    for (int k = 0; k < d.nprob; ++k) {
        d.prob[k].carry = carry;
        carry += size_t(d.prob[k].nstrips) * size_t(d.prob[k].cwords);
    }
    WLCS_CUDA(cudaMemsetAsync(c->carry.p, 0, carry_words * 4, c->stream));
    WLCS_CUDA(cudaMemsetAsync(d.ticket, 0, 4 * wlcs::kMaxProblems, c->stream));
    WLCS_CUDA(cudaMemsetAsync(d.error, 0, 4, c->stream));
    WLCS_CUDA(cudaMemsetAsync(sb + 2048, 0, 16, c->stream));
    if (want[0]) WLCS_CUDA(wlcs::pair_build_pm(dcol, cols, map, sigma, W, pmg, c->stream));
    if (want[1]) {
        WLCS_CUDA(wlcs::pair_reverse(dcol, cols, c->ry.as<uint8_t>(), c->stream));
        WLCS_CUDA(wlcs::pair_build_pm(c->ry.as<uint8_t>(), cols, map, sigma, W, pmg + pm_words,
                                      c->stream));
    }
    // both problems have the same strip count (same columns)
    if (c->timing && !c->ev0) {
        WLCS_CUDA(cudaEventCreate(&c->ev0));
        WLCS_CUDA(cudaEventCreate(&c->ev1));
    }
    if (c->timing) WLCS_CUDA(cudaEventRecord(c->ev0, c->stream));
    WLCS_CUDA(wlcs::pair_fill(d, K, false, c->sms, c->stream));
    if (c->timing) WLCS_CUDA(cudaEventRecord(c->ev1, c->stream));
    if (want[0] && v_fwd)
        WLCS_CUDA(cudaMemcpyAsync(v_fwd, c->vbuf.as<uint32_t>(), size_t(W) * 4,
                                  cudaMemcpyDeviceToHost, c->stream));
    if (want[1] && v_rev)
        WLCS_CUDA(cudaMemcpyAsync(v_rev, c->vbuf.as<uint32_t>() + W, size_t(W) * 4,
                                  cudaMemcpyDeviceToHost, c->stream));
    rc = watchdog_read(*c, c->stream);
    if (rc) return rc;
    WLCS_CUDA(stream_wait(c->stream));
    rc = watchdog_failed(*c);
    if (rc) return rc;
    if (c->timing) {
        WLCS_CUDA(cudaEventElapsedTime(&c->last_main_ms, c->ev0, c->ev1));
        c->timing_pending = false;
    }
    return WLCS_OK;
}

int wlcs_device_alloc(size_t bytes, void** d_ptr) {
    if (!d_ptr) return fail(WLCS_E_INVALID_ARGUMENT, "d_ptr is NULL");
    Ctx* c = nullptr;
    int rc = get_ctx(&c);
    if (rc) return rc;
    WLCS_CUDA(cudaMalloc(d_ptr, bytes ? bytes : 16));
    WLCS_CUDA(cudaMemset(*d_ptr, 0, bytes ? bytes : 16));
    return WLCS_OK;
}

int wlcs_device_zero(void* d_ptr, size_t bytes) {
    if (!d_ptr) return fail(WLCS_E_INVALID_ARGUMENT, "d_ptr is NULL");
    WLCS_CUDA(cudaMemset(d_ptr, 0, bytes));
    return WLCS_OK;
}

int wlcs_device_free(void* d_ptr) {
    if (d_ptr) WLCS_CUDA(cudaFree(d_ptr));
    return WLCS_OK;
}

int wlcs_ipc_handle(void* d_ptr, uint8_t handle[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (!d_ptr || !handle) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    cudaIpcMemHandle_t h;
    WLCS_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
    std::memcpy(handle, &h, 64);
    return WLCS_OK;
}

int wlcs_ipc_open(const uint8_t handle[64], void** d_ptr) {
    if (!d_ptr || !handle) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    WLCS_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return WLCS_OK;
}

int wlcs_ipc_close(void* d_ptr) {
    if (d_ptr) WLCS_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return WLCS_OK;
}

// ------------------------------------------- single-process multi-GPU
int wlcs_length_batch_multi(const uint8_t* xs, const uint64_t* x_off, const uint8_t* ys,
                            const uint64_t* y_off, size_t pairs, int n_gpus, uint32_t* out) {
    if (n_gpus <= 1) return wlcs_length_batch(xs, x_off, ys, y_off, pairs, out);
    if (!x_off || !y_off || !out) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    if (n_gpus > wlcs_device_count())
        return fail(WLCS_E_CONFIG, "n_gpus = " + std::to_string(n_gpus) + " but only " +
                                       std::to_string(wlcs_device_count()) + " devices visible");
    int rc = validate_offsets(x_off, pairs, "x");
    if (rc) return rc;
    rc = validate_offsets(y_off, pairs, "y");
    if (rc) return rc;
    // contiguous ranges balanced by cells (paper_1306_4627_b200/multigpu.py: shard_pairs)
    std::vector<double> cum(pairs + 1, 0.0);
    for (size_t k = 0; k < pairs; ++k)
        cum[k + 1] = cum[k] + double(x_off[k + 1] - x_off[k]) * double(y_off[k + 1] - y_off[k]) + 1.0;
    std::vector<size_t> cut(n_gpus + 1, 0);
    for (int g = 1; g < n_gpus; ++g)
        cut[g] = size_t(std::lower_bound(cum.begin(), cum.end(), cum[pairs] * g / n_gpus) -
                        cum.begin());
    cut[n_gpus] = pairs;
    std::vector<int> rcs(n_gpus, WLCS_OK);
    std::vector<std::string> errs(n_gpus);
    std::vector<std::thread> th;
    for (int g = 0; g < n_gpus; ++g) {
        th.emplace_back([&, g] {
            const size_t p0 = std::min(cut[g], pairs), p1 = std::max(std::min(cut[g + 1], pairs), p0);
            if (p1 == p0) return;
            if (cudaSetDevice(g) != cudaSuccess) {
                rcs[g] = WLCS_E_CUDA;
                errs[g] = "cudaSetDevice failed";
                return;
            }
            std::vector<uint64_t> xo(p1 - p0 + 1), yo(p1 - p0 + 1);
            for (size_t k = p0; k <= p1; ++k) {
                xo[k - p0] = x_off[k] - x_off[p0];
                yo[k - p0] = y_off[k] - y_off[p0];
            }
            rcs[g] = wlcs_length_batch(xs + x_off[p0], xo.data(), ys + y_off[p0], yo.data(),
                                       p1 - p0, out + p0);
            if (rcs[g]) errs[g] = t_err;
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < n_gpus; ++g)
        if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
    return WLCS_OK;
}

int wlcs_length_strips(const uint8_t* x, size_t m, const uint8_t* y, size_t n, int n_gpus,
                       uint32_t* out) {
    if (!out) return fail(WLCS_E_INVALID_ARGUMENT, "out is NULL");
    if (n_gpus <= 1 || m < 2 || n < size_t(32 * n_gpus))
        return wlcs_length(x, m, y, n, WLCS_NO_BUDGET, out);
    if (n_gpus > wlcs_device_count())
        return fail(WLCS_E_CONFIG, "n_gpus = " + std::to_string(n_gpus) + " but only " +
                                       std::to_string(wlcs_device_count()) + " devices visible");
    // rows = the shorter string, the column string is split
    const bool x_rows = m <= n;
    const uint8_t* rows = x_rows ? x : y;
    const uint8_t* cols = x_rows ? y : x;
    const size_t M = x_rows ? m : n, N = x_rows ? n : m;
    const int G = n_gpus;
    std::vector<size_t> lo(G), hi(G);
    const size_t words = (N + 31) / 32;
    for (int g = 0; g < G; ++g) {
        lo[g] = std::min(N, words * g / G * 32);
        hi[g] = std::min(N, words * (g + 1) / G * 32);
    }
    size_t inbox_words = 0;
    int rc = wlcs_colsplit_inbox_words(M, &inbox_words);
    if (rc) return rc;
    std::vector<void*> in_f(G, nullptr), in_r(G, nullptr);
    auto cleanup = [&] {
        for (int g = 0; g < G; ++g) {
            cudaSetDevice(g);
            if (in_f[g]) cudaFree(in_f[g]);
            if (in_r[g]) cudaFree(in_r[g]);
        }
    };
    for (int g = 0; g < G; ++g) {
        WLCS_CUDA(cudaSetDevice(g));
        for (int h : {g - 1, g + 1}) {
            if (h < 0 || h >= G) continue;
            cudaError_t e = cudaDeviceEnablePeerAccess(h, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                cleanup();
                return cuda_fail(e, "cudaDeviceEnablePeerAccess");
            }
            cudaGetLastError();
        }
        rc = wlcs_device_alloc(inbox_words * 4, &in_f[g]);
        if (!rc) rc = wlcs_device_alloc(inbox_words * 4, &in_r[g]);
        if (rc) {
            cleanup();
            return rc;
        }
    }
    std::vector<std::vector<uint32_t>> vf(G), vr(G);
    std::vector<int> rcs(G, WLCS_OK);
    std::vector<std::string> errs(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) {
        vf[g].assign((hi[g] - lo[g] + 31) / 32, 0u);
        vr[g].assign((hi[g] - lo[g] + 31) / 32, 0u);
        th.emplace_back([&, g] {
            if (cudaSetDevice(g) != cudaSuccess) {
                rcs[g] = WLCS_E_CUDA;
                errs[g] = "cudaSetDevice failed";
                return;
            }
            rcs[g] = wlcs_colsplit_fill(
                rows, M, cols, N, lo[g], hi[g], WLCS_COLSPLIT_FORWARD | WLCS_COLSPLIT_REVERSE,
                g > 0 ? static_cast<const uint32_t*>(in_f[g]) : nullptr,
                g + 1 < G ? static_cast<uint32_t*>(in_f[g + 1]) : nullptr,
                g + 1 < G ? static_cast<const uint32_t*>(in_r[g]) : nullptr,
                g > 0 ? static_cast<uint32_t*>(in_r[g - 1]) : nullptr, vf[g].data(),
                vr[g].data());
            if (rcs[g]) errs[g] = t_err;
        });
    }
    for (auto& t : th) t.join();
    cleanup();
    for (int g = 0; g < G; ++g)
        if (rcs[g]) return fail(rcs[g], "device " + std::to_string(g) + ": " + errs[g]);
    // combine: L = max_k F[k] + R[N-k] (multigpu.py: colsplit_combine)
    return split_combine_host(G, lo, hi, vf, vr, N, out);
}

// ------------------------------------------------------- full tables
int wlcs_fill_tables(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                     size_t memory_budget, uint32_t* dp, uint8_t* back) {
    if (!dp || (m && n && !back)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL output");
    if ((m && !x) || (n && !y)) return fail(WLCS_E_INVALID_ARGUMENT, "NULL input");
    int rc = capacity_check(m, n, memory_budget);
    if (rc) return rc;
    Ctx* c = nullptr;
    rc = get_ctx(&c);
    if (rc) return rc;
    if (m == 0 || n == 0) {  // all-zero DpTable, empty BacktrackTable (serial.cpp:13-16)
        std::memset(dp, 0, (m + 1) * (n + 1) * sizeof(uint32_t));
        return WLCS_OK;
    }
    WLCS_CUDA(c->px.ensure(m + 16));
    WLCS_CUDA(c->py.ensure(n + 16));
    if (int rc_ = h2d_staged(*c, c->px.p, x, m, c->stream)) return rc_;
    if (int rc_ = h2d_staged(*c, c->py.p, y, n, c->stream)) return rc_;
    PairPlan plan;
    rc = pair_setup(*c, c->px.as<uint8_t>(), int64_t(m), c->py.as<uint8_t>(), int64_t(n), true,
                    plan);
    if (rc) return rc;
    WLCS_CUDA(wlcs::pair_fill(plan.d, plan.K, true, c->sms, c->stream));
    const size_t dp_bytes = (m + 1) * (n + 1) * sizeof(uint32_t), back_bytes = m * n;
    DevBuf tdp, tback;
    WLCS_CUDA(tdp.ensure(dp_bytes));
    WLCS_CUDA(tback.ensure(back_bytes));
    WLCS_CUDA(wlcs::pair_tables(plan.d, plan.K, tdp.as<uint32_t>(), tback.as<uint8_t>(),
                                c->stream));
    WLCS_CUDA(cudaMemcpyAsync(dp, tdp.p, dp_bytes, cudaMemcpyDeviceToHost, c->stream));
    WLCS_CUDA(cudaMemcpyAsync(back, tback.p, back_bytes, cudaMemcpyDeviceToHost, c->stream));
    WLCS_CUDA(stream_wait(c->stream));
    return WLCS_OK;
}

// ------------------------------------------------- block-kernel contract
int wlcs_fill_block(const uint8_t* x, const uint8_t* y, uint32_t* c, size_t c_stride, uint8_t* b,
                    size_t b_stride, size_t i_first, size_t i_last, size_t j_first, size_t j_last) {
    if (i_last < i_first || j_last < j_first) return WLCS_OK;  // empty tile
    if (!x || !y || !c || !b) return fail(WLCS_E_INVALID_ARGUMENT, "NULL argument");
    if (i_first == 0 || j_first == 0)
        return fail(WLCS_E_OUT_OF_RANGE, "block cell ranges are 1-based");
    if (j_last >= c_stride || j_last > b_stride)
        return fail(WLCS_E_OUT_OF_RANGE, "block columns exceed the table stride");
    const size_t h = i_last - i_first + 1, w = j_last - j_first + 1;
    if (h > size_t(INT32_MAX) || w > size_t(INT32_MAX))
        return fail(WLCS_E_INVALID_ARGUMENT, "block too large");
    Ctx* ctx = nullptr;
    int rc = get_ctx(&ctx);
    if (rc) return rc;
    // borders: north row (corner first) and west column, packed after the symbols
    std::vector<uint32_t> border(w + 1 + h);
    for (size_t k = 0; k <= w; ++k) border[k] = c[(i_first - 1) * c_stride + (j_first - 1) + k];
    for (size_t r = 0; r < h; ++r) border[w + 1 + r] = c[(i_first + r) * c_stride + (j_first - 1)];
    const size_t sym = ((h + w) + 15) & ~size_t(15);
    const size_t cells = h * w;
    WLCS_CUDA(ctx->tile.ensure(sym + border.size() * 4 + cells * 5 + 64));
    uint8_t* base = ctx->tile.as<uint8_t>();
    uint32_t* d_border = reinterpret_cast<uint32_t*>(base + sym);
    uint32_t* d_cv = d_border + border.size();
    uint8_t* d_bv = reinterpret_cast<uint8_t*>(d_cv + cells);
    cudaStream_t s = ctx->stream;
    WLCS_CUDA(cudaMemcpyAsync(base, x + (i_first - 1), h, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(base + h, y + (j_first - 1), w, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(cudaMemcpyAsync(d_border, border.data(), border.size() * 4, cudaMemcpyHostToDevice, s));
    WLCS_CUDA(wlcs::tile_fill(base, base + h, d_border, d_border + w + 1, d_cv, d_bv, int(h),
                              int(w), s));
    std::vector<uint32_t> cv(cells);
    std::vector<uint8_t> bv(cells);
    WLCS_CUDA(cudaMemcpyAsync(cv.data(), d_cv, cells * 4, cudaMemcpyDeviceToHost, s));
    WLCS_CUDA(cudaMemcpyAsync(bv.data(), d_bv, cells, cudaMemcpyDeviceToHost, s));
    WLCS_CUDA(stream_wait(s));
    for (size_t r = 0; r < h; ++r) {
        std::memcpy(c + (i_first + r) * c_stride + j_first, cv.data() + r * w, w * 4);
        std::memcpy(b + (i_first + r - 1) * b_stride + (j_first - 1), bv.data() + r * w, w);
    }
    return WLCS_OK;
}

}  // extern "C"
