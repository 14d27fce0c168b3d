// facade_core.cpp -- the reference's C++ API (include/wavelcs/*.hpp) over
// the C-ABI of the B200 library.  Status codes come back as the reference's
// exception types; every fill runs on the device (there is no host kernel).
//
// Reference semantics followed here (paths under /root/reference/proj):
//   check_capacity        src/tables.cpp:9-24 (formula and message in capi.cu)
//   lcs_fill_serial       src/serial.cpp:11-30   capacity check, then tables
//   lcs_length            src/serial.cpp:32-34
//   traceback             src/serial.cpp:36-61
//   brute_force_lcs       src/serial.cpp:63-89
//   BlockGrid et al.      src/parallel.cpp:38-83
//   compute_block         src/parallel.cpp:230-249
//   lcs_fill_parallel     src/parallel.cpp:251-274   error order:
//                         workers -> kernel -> capacity -> block size
//                         (the last only when both inputs are non-empty)
//   kernel selection      src/kernels.cpp:32-91
#include <algorithm>
#include <chrono>
#include <string>
#include <thread>

#include "wavelcs_b200.hpp"
#include "wavelcs_capi.h"

namespace wavelcs {
namespace {

[[noreturn]] void raise_status(int rc) {
    const std::string msg = wlcs_last_error();
    switch (rc) {
        case WLCS_E_CAPACITY: throw CapacityError(msg);
        case WLCS_E_CONFIG: throw ConfigError(msg);
        case WLCS_E_OUT_OF_RANGE: throw std::out_of_range(msg);
        case WLCS_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case WLCS_E_INPUT: throw InputError(msg);
        default: throw DeviceError(msg);
    }
}

inline void check(int rc) {
    if (rc != WLCS_OK) raise_status(rc);
}

inline const std::uint8_t* u8(const Sequence& s) {
    return reinterpret_cast<const std::uint8_t*>(s.data());
}

std::size_t blocks_along(std::size_t cells, std::size_t side) {
    return (cells + side - 1) / side;
}

}  // namespace

// ---------------------------------------------------------------- sequence
bool is_subsequence(const Sequence& candidate, const Sequence& text) noexcept {
    auto want = candidate.begin();
    for (auto it = text.begin(); it != text.end() && want != candidate.end(); ++it)
        want += (*it == *want) ? 1 : 0;
    return want == candidate.end();
}

double similarity_percent(std::size_t lcs_len, std::size_t parent_len, std::size_t child_len) {
    if (lcs_len > std::min(parent_len, child_len))
        throw std::invalid_argument("similarity_percent: LCS length exceeds min(M, N)");
    return child_len == 0 ? 100.0 : 100.0 * double(lcs_len) / double(child_len);
}

// ------------------------------------------------------------------ serial
void check_capacity(std::size_t m, std::size_t n, std::size_t budget) {
    check(wlcs_check_capacity(m, n, budget));
}

Length lcs_length(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    std::uint32_t out = 0;
    check(wlcs_length(u8(x), x.size(), u8(y), y.size(), memory_budget, &out));
    return out;
}

Sequence lcs_subsequence(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    std::string buf(std::min(x.size(), y.size()), '\0');
    std::size_t len = 0;
    check(wlcs_subsequence(u8(x), x.size(), u8(y), y.size(), memory_budget,
                           reinterpret_cast<std::uint8_t*>(buf.data()), buf.size(), &len));
    buf.resize(len);
    return Sequence(std::move(buf));
}

FillResult lcs_fill_serial(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    check(wlcs_check_capacity(x.size(), y.size(), memory_budget));  // before any allocation
    FillResult out{DpTable(x.size(), y.size()), BacktrackTable(x.size(), y.size())};
    if (!x.empty() && !y.empty())
        check(wlcs_fill_tables(u8(x), x.size(), u8(y), y.size(), kNoMemoryBudget, out.dp.data(),
                               reinterpret_cast<std::uint8_t*>(out.back.data())));
    return out;
}

Sequence traceback(const BacktrackTable& back, const Sequence& x, std::size_t i, std::size_t j) {
    if (i > back.rows() || j > back.cols())
        throw std::out_of_range("traceback: (" + std::to_string(i) + ", " + std::to_string(j) +
                                ") lies outside the " + std::to_string(back.rows()) + " x " +
                                std::to_string(back.cols()) + " arrow table");
    std::string out;
    out.reserve(std::min(i, j));
    while (i != 0 && j != 0) {
        const Arrow a = back.at(i, j);
        if (a == Arrow::Diag) out.push_back(x[i - 1]);
        i -= (a != Arrow::Left) ? 1 : 0;
        j -= (a != Arrow::Up) ? 1 : 0;
    }
    std::reverse(out.begin(), out.end());
    return Sequence(std::move(out));
}

Length brute_force_lcs(const Sequence& x, const Sequence& y) {
    const bool x_short = x.size() <= y.size();
    const Sequence& s = x_short ? x : y;
    const Sequence& l = x_short ? y : x;
    if (s.size() > 20)
        throw std::invalid_argument("brute_force_lcs: min(M, N) = " + std::to_string(s.size()) +
                                    " > 20 is too long to enumerate");
    Length best = 0;
    std::string pick;
    for (std::uint64_t mask = 1; mask < (std::uint64_t{1} << s.size()); ++mask) {
        const Length bits = Length(__builtin_popcountll(mask));
        if (bits <= best) continue;
        pick.clear();
        for (std::uint64_t m = mask; m != 0; m &= m - 1) pick.push_back(s[std::size_t(__builtin_ctzll(m))]);
        if (is_subsequence(Sequence(pick), l)) best = bits;
    }
    return best;
}

std::vector<Length> lcs_length_batch(const std::vector<Sequence>& xs,
                                     const std::vector<Sequence>& ys) {
    if (xs.size() != ys.size()) throw std::invalid_argument("lcs_length_batch: size mismatch");
    std::vector<std::uint64_t> xo(1, 0), yo(1, 0);
    std::size_t xt = 0, yt = 0;
    for (std::size_t k = 0; k < xs.size(); ++k) {
        xo.push_back(xt += xs[k].size());
        yo.push_back(yt += ys[k].size());
    }
    std::string xcat, ycat;
    xcat.reserve(xt);
    ycat.reserve(yt);
    for (std::size_t k = 0; k < xs.size(); ++k) {
        xcat += xs[k].view();
        ycat += ys[k].view();
    }
    std::vector<Length> out(xs.size(), 0);
    check(wlcs_length_batch(reinterpret_cast<const std::uint8_t*>(xcat.data()), xo.data(),
                            reinterpret_cast<const std::uint8_t*>(ycat.data()), yo.data(),
                            xs.size(), out.data()));
    return out;
}

// ----------------------------------------------------------------- kernels
void fill_block_device(const BlockArgs& a) {
    check(wlcs_fill_block(reinterpret_cast<const std::uint8_t*>(a.x),
                          reinterpret_cast<const std::uint8_t*>(a.y), a.c, a.c_stride,
                          reinterpret_cast<std::uint8_t*>(a.b), a.b_stride, a.i_first, a.i_last,
                          a.j_first, a.j_last));
}

void fill_block_scalar(const BlockArgs& a) { fill_block_device(a); }

bool kernel_available(KernelKind kind) noexcept {
    return kind == KernelKind::Auto || kind == KernelKind::Scalar || kind == KernelKind::B200;
}

KernelKind detect_kernel() noexcept { return KernelKind::B200; }

const char* kernel_name(KernelKind kind) noexcept {
    switch (kind) {
        case KernelKind::Auto: return "auto";
        case KernelKind::Scalar: return "scalar";
        case KernelKind::Avx2: return "avx2";
        case KernelKind::Neon: return "neon";
        case KernelKind::B200: return "b200";
    }
    return "unknown";
}

BlockKernelFn resolve_kernel(KernelKind kind) {
    const KernelKind k = kind == KernelKind::Auto ? detect_kernel() : kind;
    if (!kernel_available(k))
        throw ConfigError(std::string("kernel '") + kernel_name(k) +
                          "' is not available on this host (the B200 build has no host "
                          "SIMD kernels)");
    return k == KernelKind::Scalar ? &fill_block_scalar : &fill_block_device;
}

// ---------------------------------------------------------------- parallel
BlockGrid::BlockGrid(std::size_t m, std::size_t n, std::size_t block_size)
    : m_(m), n_(n), block_size_(block_size),
      block_rows_(blocks_along(m, block_size)), block_cols_(blocks_along(n, block_size)) {}

CellRect BlockGrid::cells(BlockCoord block) const {
    const std::size_t i0 = block.row * block_size_, j0 = block.col * block_size_;
    return CellRect{i0 + 1, std::min(i0 + block_size_, m_), j0 + 1,
                    std::min(j0 + block_size_, n_)};
}

BlockGrid partition_blocks(std::size_t m, std::size_t n, std::size_t block_size) {
    if (block_size == 0) throw ConfigError("block size must be at least 1");
    return BlockGrid(m, n, block_size);
}

std::size_t WaveSchedule::block_count() const noexcept {
    std::size_t total = 0;
    for (const auto& w : waves) total += w.size();
    return total;
}

WaveSchedule wavefront_schedule(const BlockGrid& grid) {
    WaveSchedule out;
    if (grid.empty()) return out;
    const std::size_t R = grid.block_rows(), C = grid.block_cols();
    out.waves.resize(R + C - 1);
    // wave d holds (r, d - r); rows listed from the bottom of the wave up
    for (std::size_t d = 0; d + 1 < R + C; ++d) {
        const std::size_t r_top = d + 1 > C ? d + 1 - C : 0;
        for (std::size_t r = std::min(d, R - 1) + 1; r-- > r_top;) out.waves[d].push_back({r, d - r});
    }
    return out;
}

unsigned default_worker_count() noexcept {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1u;
}

void compute_block(const BlockGrid& grid, BlockCoord block, const Sequence& x, const Sequence& y,
                   DpTable& dp, BacktrackTable& back) {
    if (block.row >= grid.block_rows() || block.col >= grid.block_cols())
        throw std::out_of_range("compute_block: block (" + std::to_string(block.row) + ", " +
                                std::to_string(block.col) + ") is outside the " +
                                std::to_string(grid.block_rows()) + " x " +
                                std::to_string(grid.block_cols()) + " grid");
    const CellRect r = grid.cells(block);
    BlockArgs a;
    a.x = x.data();
    a.y = y.data();
    a.c = dp.data();
    a.c_stride = dp.stride();
    a.b = back.data();
    a.b_stride = back.stride();
    a.i_first = r.i_first;
    a.i_last = r.i_last;
    a.j_first = r.j_first;
    a.j_last = r.j_last;
    fill_block_device(a);
}

TimedFill lcs_fill_parallel(const Sequence& x, const Sequence& y, const ParallelConfig& config) {
    if (config.workers == 0) throw ConfigError("worker count must be at least 1");
    (void)resolve_kernel(config.kernel);  // ConfigError for a kind this build lacks
    check(wlcs_check_capacity(x.size(), y.size(), config.memory_budget));
    const auto t0 = std::chrono::steady_clock::now();
    TimedFill out{DpTable(x.size(), y.size()), BacktrackTable(x.size(), y.size()), 0.0};
    if (!x.empty() && !y.empty()) {
        (void)partition_blocks(x.size(), y.size(), config.block_size);  // ConfigError for B = 0
        check(wlcs_fill_tables(u8(x), x.size(), u8(y), y.size(), kNoMemoryBudget, out.dp.data(),
                               reinterpret_cast<std::uint8_t*>(out.back.data())));
    }
    out.elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

}  // namespace wavelcs
