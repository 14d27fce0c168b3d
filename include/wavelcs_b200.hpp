// wavelcs_b200.hpp -- C++ drop-in facade for the reference "wavelcs" LCS
// entry points, backed by the B200 library through the C-ABI
// (include/wavelcs_capi.h).  Same namespace, names, argument meaning and
// exception types as the reference headers (paths under /root/reference/proj):
//
//   Length lcs_length(x, y, memory_budget)     include/wavelcs/serial.hpp:24-25
//   check_capacity(m, n, budget)               include/wavelcs/tables.hpp:16
//   class Sequence, is_subsequence             include/wavelcs/sequence.hpp:13-38
//   CapacityError / ConfigError / InputError /
//   EquivalenceError                           include/wavelcs/errors.hpp:8-30
//   generate_random(length, alphabet, seed)    include/wavelcs/io.hpp:34
//
// plus the single-call subsequence that replaces the composition
//   traceback(lcs_fill_parallel(x, y, cfg).back, x, M, N)
// (tools/wavelcs_main.cpp:78-86; serial.hpp:30; parallel.hpp:92-93) and a
// batch entry point.  Link against paper_1306_4627_b200/_lib/libwavelcs_b200.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace wavelcs {

using Length = std::uint32_t;

inline constexpr std::size_t kDefaultMemoryBudget = std::size_t{2} * 1024 * 1024 * 1024;
inline constexpr std::size_t kNoMemoryBudget = ~std::size_t{0};

class CapacityError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ConfigError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class InputError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class EquivalenceError : public std::logic_error {
public:
    using std::logic_error::logic_error;
};
/// CUDA failure inside the library (no reference counterpart: the reference
/// never leaves the CPU).  There is no CPU fallback.
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class Sequence {
public:
    Sequence() = default;
    explicit Sequence(std::string symbols) : symbols_(std::move(symbols)) {}
    std::size_t size() const noexcept { return symbols_.size(); }
    bool empty() const noexcept { return symbols_.empty(); }
    char operator[](std::size_t pos) const { return symbols_[pos]; }
    const char* data() const noexcept { return symbols_.data(); }
    std::string_view view() const noexcept { return symbols_; }
    const std::string& str() const noexcept { return symbols_; }
    void push_back(char symbol) { symbols_.push_back(symbol); }
    auto begin() const noexcept { return symbols_.begin(); }
    auto end() const noexcept { return symbols_.end(); }
    friend bool operator==(const Sequence&, const Sequence&) = default;

private:
    std::string symbols_;
};

bool is_subsequence(const Sequence& candidate, const Sequence& text) noexcept;

void check_capacity(std::size_t m, std::size_t n, std::size_t budget = kDefaultMemoryBudget);

/// LCS length on the GPU.  Throws CapacityError exactly when the reference's
/// tables would exceed memory_budget (the device path itself is O(M+N)).
Length lcs_length(const Sequence& x, const Sequence& y,
                  std::size_t memory_budget = kDefaultMemoryBudget);

/// The reference's recovered subsequence (LEFT tie-break), in one call.
Sequence lcs_subsequence(const Sequence& x, const Sequence& y,
                         std::size_t memory_budget = kDefaultMemoryBudget);

/// Which recurrence case produced a cell (cell.hpp:13-25).
enum class Arrow : std::uint8_t { Diag = 0, Up = 1, Left = 2 };

/// (M+1) x (N+1) prefix LCS lengths, row-major; same layout and accessors as
/// the reference's DpTable (tables.hpp:20-45).
class DpTable {
public:
    DpTable() = default;
    DpTable(std::size_t m, std::size_t n) : rows_(m + 1), cols_(n + 1), cells_(rows_ * cols_, 0) {}
    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    Length at(std::size_t i, std::size_t j) const { return cells_[i * cols_ + j]; }
    Length& at(std::size_t i, std::size_t j) { return cells_[i * cols_ + j]; }
    Length* data() noexcept { return cells_.data(); }
    const Length* data() const noexcept { return cells_.data(); }
    std::size_t stride() const noexcept { return cols_; }
    Length final_length() const { return cells_.empty() ? 0 : cells_.back(); }
    friend bool operator==(const DpTable&, const DpTable&) = default;

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<Length> cells_;
};

/// M x N arrows, 1-based accessors; the reference's BacktrackTable
/// (tables.hpp:49-71).
class BacktrackTable {
public:
    BacktrackTable() = default;
    BacktrackTable(std::size_t m, std::size_t n) : rows_(m), cols_(n), cells_(m * n, Arrow::Left) {}
    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    Arrow at(std::size_t i, std::size_t j) const { return cells_[(i - 1) * cols_ + (j - 1)]; }
    Arrow& at(std::size_t i, std::size_t j) { return cells_[(i - 1) * cols_ + (j - 1)]; }
    Arrow* data() noexcept { return cells_.data(); }
    const Arrow* data() const noexcept { return cells_.data(); }
    std::size_t stride() const noexcept { return cols_; }
    friend bool operator==(const BacktrackTable&, const BacktrackTable&) = default;

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<Arrow> cells_;
};

struct FillResult {
    DpTable dp;
    BacktrackTable back;
};

/// lcs_fill_serial (serial.hpp:21-22) with the tables filled on the device:
/// identical DpTable / BacktrackTable contents, same CapacityError.
FillResult lcs_fill_serial(const Sequence& x, const Sequence& y,
                           std::size_t memory_budget = kDefaultMemoryBudget);

/// traceback (serial.hpp:30): walks the arrow table from (i, j); forward
/// order; std::out_of_range when (i, j) is outside the table.  Host code (it
/// reads a host table, exactly like the reference).
Sequence traceback(const BacktrackTable& back, const Sequence& x, std::size_t i, std::size_t j);

/// Lengths of many independent pairs (xs[k], ys[k]).
std::vector<Length> lcs_length_batch(const std::vector<Sequence>& xs,
                                     const std::vector<Sequence>& ys);

Sequence generate_random(std::size_t length, const Sequence& alphabet, std::uint64_t seed);

/// similarity_percent (sequence.cpp:18-26): 100 * L / |child| (100 when the
/// child is empty); std::invalid_argument when L > min(M, N).
double similarity_percent(std::size_t lcs_len, std::size_t parent_len, std::size_t child_len);

// ---- input path (io.hpp / io.cpp semantics) --------
enum class InputFormat { Plain, Fasta };
/// ".fa" / ".fasta" -> Fasta, anything else Plain (io.cpp:38-44).
InputFormat format_from_path(const std::filesystem::path& path) noexcept;
/// Whole file; Plain strips ASCII whitespace, Fasta keeps the first record
/// upper-cased; InputError on unreadable files / malformed FASTA; with
/// validate_dna, InputError on a symbol outside {A,C,G,T} (io.cpp:46-101).
Sequence load_sequence(const std::filesystem::path& path, InputFormat format,
                       bool validate_dna = false);
Sequence parse_fasta(std::string_view bytes);
void validate_dna_alphabet(const Sequence& seq);
void write_plain(const Sequence& seq, const std::filesystem::path& path);

}  // namespace wavelcs
