// facade.cpp -- the wavelcs:: C++ facade (include/wavelcs_b200.hpp) over the
// C-ABI.  Maps wlcs_status codes back onto the reference's exception types.
#include "wavelcs_b200.hpp"

#include <string>

#include "wavelcs_capi.h"

namespace wavelcs {
namespace {

void raise(int rc) {
    if (rc == WLCS_OK) return;
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

const std::uint8_t* bytes(const Sequence& s) {
    return reinterpret_cast<const std::uint8_t*>(s.data());
}

}  // namespace

// sequence.cpp:8-16 semantics (single left-to-right scan).
bool is_subsequence(const Sequence& candidate, const Sequence& text) noexcept {
    std::size_t matched = 0;
    for (std::size_t pos = 0; pos < text.size() && matched < candidate.size(); ++pos)
        if (text[pos] == candidate[matched]) ++matched;
    return matched == candidate.size();
}

void check_capacity(std::size_t m, std::size_t n, std::size_t budget) {
    raise(wlcs_check_capacity(m, n, budget));
}

Length lcs_length(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    std::uint32_t out = 0;
    raise(wlcs_length(bytes(x), x.size(), bytes(y), y.size(), memory_budget, &out));
    return out;
}

Sequence lcs_subsequence(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    std::string buf(std::min(x.size(), y.size()), '\0');
    std::size_t len = 0;
    raise(wlcs_subsequence(bytes(x), x.size(), bytes(y), y.size(), memory_budget,
                           reinterpret_cast<std::uint8_t*>(buf.data()), buf.size(), &len));
    buf.resize(len);
    return Sequence(std::move(buf));
}

FillResult lcs_fill_serial(const Sequence& x, const Sequence& y, std::size_t memory_budget) {
    // capacity first, before any allocation (serial.cpp:12)
    raise(wlcs_check_capacity(x.size(), y.size(), memory_budget));
    FillResult out{DpTable(x.size(), y.size()), BacktrackTable(x.size(), y.size())};
    if (x.empty() || y.empty()) return out;
    raise(wlcs_fill_tables(bytes(x), x.size(), bytes(y), y.size(), memory_budget,
                           out.dp.data(), reinterpret_cast<std::uint8_t*>(out.back.data())));
    return out;
}

// serial.cpp:36-61 semantics.
Sequence traceback(const BacktrackTable& back, const Sequence& x, std::size_t i, std::size_t j) {
    if (i > back.rows() || j > back.cols())
        throw std::out_of_range("traceback: position (" + std::to_string(i) + ", " +
                                std::to_string(j) + ") outside " + std::to_string(back.rows()) +
                                " x " + std::to_string(back.cols()) + " table");
    std::string reversed;
    while (i > 0 && j > 0) {
        switch (back.at(i, j)) {
            case Arrow::Diag:
                reversed.push_back(x[i - 1]);
                --i;
                --j;
                break;
            case Arrow::Up:
                --i;
                break;
            case Arrow::Left:
                --j;
                break;
        }
    }
    return Sequence(std::string(reversed.rbegin(), reversed.rend()));
}

std::vector<Length> lcs_length_batch(const std::vector<Sequence>& xs,
                                     const std::vector<Sequence>& ys) {
    if (xs.size() != ys.size()) throw std::invalid_argument("lcs_length_batch: size mismatch");
    std::string xcat, ycat;
    std::vector<std::uint64_t> xo(xs.size() + 1, 0), yo(ys.size() + 1, 0);
    for (std::size_t k = 0; k < xs.size(); ++k) {
        xcat += xs[k].str();
        ycat += ys[k].str();
        xo[k + 1] = xcat.size();
        yo[k + 1] = ycat.size();
    }
    std::vector<Length> out(xs.size(), 0);
    raise(wlcs_length_batch(reinterpret_cast<const std::uint8_t*>(xcat.data()), xo.data(),
                            reinterpret_cast<const std::uint8_t*>(ycat.data()), yo.data(),
                            xs.size(), out.data()));
    return out;
}

Sequence generate_random(std::size_t length, const Sequence& alphabet, std::uint64_t seed) {
    std::string s(length, '\0');
    raise(wlcs_generate_random(length, bytes(alphabet), alphabet.size(), seed,
                               reinterpret_cast<std::uint8_t*>(s.data())));
    return Sequence(std::move(s));
}

}  // namespace wavelcs
