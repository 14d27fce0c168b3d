// wavelcs/cell.hpp -- drop-in for the reference header of the same name
// (/root/reference/proj/include/wavelcs/cell.hpp:13-38): the DP cell type,
// the arrow codes and the one-cell recurrence.  Header-only; the device
// kernels (paper_1306_4627_b200/csrc) compute the same integers 32 cells at a
// time (Hyyro identity) and the same arrows.
#pragma once

#include <cstddef>
#include <cstdint>

namespace wavelcs {

/// A DP value: LCS length of two prefixes (32-bit, as in the reference).
using Length = std::uint32_t;

/// Which case of the recurrence produced a cell; the traceback follows it.
enum class Arrow : std::uint8_t {
    Diag = 0,  // x_i == y_j: continue at (i-1, j-1)
    Up = 1,    // continue at (i-1, j)
    Left = 2,  // continue at (i, j-1)
};

struct CellStep {
    Length value;
    Arrow arrow;
};

/// One cell: a match extends the diagonal; otherwise the larger of the upper
/// and left neighbours, with equality resolved to LEFT (strict `>` for Up).
constexpr CellStep lcs_cell(char x_i, char y_j, Length diag, Length up, Length left) noexcept {
    return x_i == y_j ? CellStep{diag + 1, Arrow::Diag}
                      : (up > left ? CellStep{up, Arrow::Up} : CellStep{left, Arrow::Left});
}

}  // namespace wavelcs
