// oracle/ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference sources where they lie under
// /root/reference/proj/src into oracle/_ref/libwavelcs_ref.so.  It is used
//   * by tests/ as the parity oracle (golden fixtures, small-size checks), and
//   * by bench.py --impl reference / cpu_baseline to time the reference's own
//     CPU fill on the GPU box's host cores.
// The product library never loads it.
//
// Everything here calls the reference's public API (include/wavelcs/*.hpp):
//   lcs_fill_parallel  parallel.hpp:92-93 / parallel.cpp:251-274
//   lcs_fill_serial    serial.hpp:20-21
//   lcs_length         serial.hpp:24-25
//   traceback          serial.hpp:30
//   brute_force_lcs    serial.hpp:36
//   generate_random    io.hpp:34
//   check_capacity     tables.hpp:16
// The batch driver (ref_batch_lengths) is harness code: the reference has no
// batch API, so each pair runs lcs_fill_parallel(workers=1) on a std::thread
// pool, exactly as SURVEY.md section 8(d) prescribes for the CPU baseline.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "wavelcs/errors.hpp"
#include "wavelcs/io.hpp"
#include "wavelcs/parallel.hpp"
#include "wavelcs/serial.hpp"
#include "wavelcs/tables.hpp"

namespace {

thread_local std::string g_err;

// 0 ok, 1 CapacityError, 2 ConfigError, 3 out_of_range, 4 invalid_argument,
// 5 InputError, 9 other.
template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const wavelcs::CapacityError& e) {
        g_err = e.what();
        return 1;
    } catch (const wavelcs::ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 4;
    } catch (const wavelcs::InputError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

wavelcs::Sequence seq_of(const char* p, std::size_t n) {
    return wavelcs::Sequence(std::string(p, n));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_default_workers() { return wavelcs::default_worker_count(); }

int ref_check_capacity(std::size_t m, std::size_t n, std::size_t budget) {
    return guarded([&] { wavelcs::check_capacity(m, n, budget); });
}

// wavelcs::lcs_length(x, y, budget)  (serial path, serial.cpp:32-34)
int ref_lcs_length_serial(const char* x, std::size_t m, const char* y, std::size_t n,
                          std::size_t budget, std::uint32_t* out) {
    return guarded([&] { *out = wavelcs::lcs_length(seq_of(x, m), seq_of(y, n), budget); });
}

// lcs_fill_parallel(x, y, cfg).dp.final_length(); seconds = the reference's
// own fill timer (TimedFill::elapsed_seconds, parallel.cpp:258-272).
int ref_lcs_length_parallel(const char* x, std::size_t m, const char* y, std::size_t n,
                            unsigned workers, std::size_t block, std::size_t budget,
                            std::uint32_t* out, double* seconds) {
    return guarded([&] {
        wavelcs::ParallelConfig cfg;
        cfg.workers = workers;
        cfg.block_size = block;
        cfg.memory_budget = budget;
        const auto fill = wavelcs::lcs_fill_parallel(seq_of(x, m), seq_of(y, n), cfg);
        *out = fill.dp.final_length();
        if (seconds) *seconds = fill.elapsed_seconds;
    });
}

// The CLI's compute path (tools/wavelcs_main.cpp:78-86): lcs_fill_parallel
// then traceback(fill.back, parent, M, N).
int ref_lcs_subsequence(const char* x, std::size_t m, const char* y, std::size_t n,
                        unsigned workers, std::size_t budget, char* out, std::size_t cap,
                        std::size_t* out_len, double* seconds) {
    return guarded([&] {
        wavelcs::ParallelConfig cfg;
        cfg.workers = workers;
        cfg.memory_budget = budget;
        const wavelcs::Sequence xs = seq_of(x, m), ys = seq_of(y, n);
        const auto t0 = std::chrono::steady_clock::now();
        const auto fill = wavelcs::lcs_fill_parallel(xs, ys, cfg);
        const wavelcs::Sequence lcs = wavelcs::traceback(fill.back, xs, m, n);
        if (seconds)
            *seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out_len = lcs.size();
        if (lcs.size() > cap) throw std::out_of_range("output buffer too small");
        std::memcpy(out, lcs.data(), lcs.size());
    });
}

// Full DpTable / BacktrackTable through the parallel fill.
int ref_fill_tables(const char* x, std::size_t m, const char* y, std::size_t n, unsigned workers,
                    std::size_t block, std::uint32_t* dp, std::uint8_t* back) {
    return guarded([&] {
        wavelcs::ParallelConfig cfg;
        cfg.workers = workers;
        cfg.block_size = block;
        cfg.memory_budget = ~std::size_t{0};
        const auto fill = wavelcs::lcs_fill_parallel(seq_of(x, m), seq_of(y, n), cfg);
        std::memcpy(dp, fill.dp.data(), (m + 1) * (n + 1) * sizeof(std::uint32_t));
        if (m * n != 0) std::memcpy(back, fill.back.data(), m * n);
    });
}

// traceback(back, x, i, j) over a caller-provided arrow table (serial.cpp:36-61).
int ref_traceback(const std::uint8_t* back, std::size_t rows, std::size_t cols, const char* x,
                  std::size_t m, std::size_t i, std::size_t j, char* out, std::size_t* out_len) {
    return guarded([&] {
        wavelcs::BacktrackTable table(rows, cols);
        if (rows * cols != 0) std::memcpy(table.data(), back, rows * cols);
        const wavelcs::Sequence lcs = wavelcs::traceback(table, seq_of(x, m), i, j);
        *out_len = lcs.size();
        std::memcpy(out, lcs.data(), lcs.size());
    });
}

int ref_brute_force(const char* x, std::size_t m, const char* y, std::size_t n,
                    std::uint32_t* out) {
    return guarded([&] { *out = wavelcs::brute_force_lcs(seq_of(x, m), seq_of(y, n)); });
}

int ref_generate_random(std::size_t length, const char* alphabet, std::size_t alen,
                        std::uint64_t seed, char* out) {
    return guarded([&] {
        const auto s = wavelcs::generate_random(length, seq_of(alphabet, alen), seed);
        std::memcpy(out, s.data(), length);
    });
}

// Harness batch driver: `threads` std::threads pull pairs from an atomic
// counter and run lcs_fill_parallel(workers=1) per pair.  Returns wall
// seconds through *seconds.
int ref_batch_lengths(const char* xs, const std::uint64_t* xoff, const char* ys,
                      const std::uint64_t* yoff, std::size_t pairs, unsigned threads,
                      std::uint32_t* out, double* seconds) {
    return guarded([&] {
        if (threads == 0) threads = 1;
        std::atomic<std::size_t> next{0};
        std::atomic<int> failed{0};
        auto worker = [&] {
            wavelcs::ParallelConfig cfg;
            cfg.workers = 1;
            cfg.memory_budget = ~std::size_t{0};
            for (;;) {
                const std::size_t p = next.fetch_add(1);
                if (p >= pairs) break;
                try {
                    const auto fill = wavelcs::lcs_fill_parallel(
                        seq_of(xs + xoff[p], xoff[p + 1] - xoff[p]),
                        seq_of(ys + yoff[p], yoff[p + 1] - yoff[p]), cfg);
                    out[p] = fill.dp.final_length();
                } catch (...) {
                    failed.store(1);
                }
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < threads; ++t) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
        if (seconds)
            *seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (failed.load()) throw std::runtime_error("a batch pair failed");
    });
}

}  // extern "C"
