// wavelcs/kernels.hpp -- the reference's block-kernel plugin interface
// (/root/reference/proj/include/wavelcs/kernels.hpp:23-64): a kernel fills
// one rectangular tile of the caller's DP tables from its final north row and
// west column.
//
// B200 build: the tile is filled ON THE DEVICE (wlcs_fill_block, the
// recurrence of cell.hpp in anti-diagonal order over the tile) and written
// back into the caller's host tables.  There is no host kernel and no cpuid
// dispatch: KernelKind::B200 is the device kernel, Scalar names the same
// device fill (the reference's semantic kernel, kernels_scalar.cpp:5-17), and
// Avx2 / Neon report unavailable (resolve_kernel throws ConfigError, exactly
// as the reference does for a kind the host lacks).  The whole-table fills
// (lcs_fill_serial / lcs_fill_parallel) do not go tile by tile: they run the
// bit-parallel device fill once and expand the tables on the device.
#pragma once

#include <cstddef>
#include <cstdint>

#include "wavelcs/cell.hpp"

namespace wavelcs {

/// One tile of the DP grid, cell ranges 1-based inclusive; row i_first-1 and
/// column j_first-1 of `c` hold final values (reference contract).
struct BlockArgs {
    const char* x = nullptr;               // x[i-1] is the i-th parent symbol
    const char* y = nullptr;               // y[j-1] is the j-th child symbol
    const std::int32_t* y_wide = nullptr;  // accepted for source compatibility; unused
    Length* c = nullptr;                   // DP cells, c[i * c_stride + j]
    std::size_t c_stride = 0;
    Arrow* b = nullptr;                    // arrows, b[(i-1) * b_stride + (j-1)]
    std::size_t b_stride = 0;
    std::size_t i_first = 0, i_last = 0;
    std::size_t j_first = 0, j_last = 0;
};

using BlockKernelFn = void (*)(const BlockArgs&);

/// The device tile fill (throws DeviceError when CUDA fails).
void fill_block_device(const BlockArgs& args);

/// The reference's scalar kernel name; here the same device tile fill.
void fill_block_scalar(const BlockArgs& args);

enum class KernelKind : std::uint8_t { Auto = 0, Scalar, Avx2, Neon, B200 };

/// Auto, Scalar and B200 are available; the host SIMD kinds are not built.
bool kernel_available(KernelKind kind) noexcept;

/// KernelKind::B200.
KernelKind detect_kernel() noexcept;

/// Function of `kind` (Auto resolves to detect_kernel()); ConfigError when
/// the kind is not available.
BlockKernelFn resolve_kernel(KernelKind kind);

const char* kernel_name(KernelKind kind) noexcept;

}  // namespace wavelcs
