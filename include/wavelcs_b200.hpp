// wavelcs_b200.hpp -- the C++ drop-in for the reference "wavelcs" library,
// backed by the B200 library (libwavelcs_b200.so) through the C-ABI
// (include/wavelcs_capi.h).
//
// The reference's own headers are mirrored one for one under
// include/wavelcs/ (cell, errors, sequence, tables, kernels, serial, parallel,
// io, bench: same names, signatures, layouts, error types and error order), so
// the reference's callers and tests compile unchanged against -Iinclude and
// link -lwavelcs_b200 (tests/cpp/Makefile builds the reference's own test
// sources that way).  This header adds the entry points the reference lacks:
//
//   lcs_subsequence(x, y, budget)   traceback(lcs_fill_parallel(x, y).back, x, M, N)
//                                   in one call, without the tables
//   lcs_length_batch(xs, ys)        many independent pairs at once
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "wavelcs/bench.hpp"
#include "wavelcs/cell.hpp"
#include "wavelcs/errors.hpp"
#include "wavelcs/io.hpp"
#include "wavelcs/kernels.hpp"
#include "wavelcs/parallel.hpp"
#include "wavelcs/sequence.hpp"
#include "wavelcs/serial.hpp"
#include "wavelcs/tables.hpp"

namespace wavelcs {

/// Budget sentinel: skip the reference's table-capacity check.
inline constexpr std::size_t kNoMemoryBudget = ~std::size_t{0};

/// The reference's recovered subsequence (LEFT tie-break), in one call, with
/// O(M N / 8) device memory instead of 5 M N bytes of tables.
Sequence lcs_subsequence(const Sequence& x, const Sequence& y,
                         std::size_t memory_budget = kDefaultMemoryBudget);

/// Lengths of many independent pairs (xs[k], ys[k]).
std::vector<Length> lcs_length_batch(const std::vector<Sequence>& xs,
                                     const std::vector<Sequence>& ys);

}  // namespace wavelcs
