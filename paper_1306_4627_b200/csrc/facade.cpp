// facade.cpp -- the wavelcs:: C++ facade (include/wavelcs_b200.hpp) over the
// C-ABI.  Maps wlcs_status codes back onto the reference's exception types.
#include "wavelcs_b200.hpp"

#include <algorithm>
#include <cctype>
#include <fstream>
#include <sstream>
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

double similarity_percent(std::size_t lcs_len, std::size_t parent_len, std::size_t child_len) {
    if (lcs_len > std::min(parent_len, child_len))
        throw std::invalid_argument("similarity_percent: LCS length exceeds min(M, N)");
    if (child_len == 0) return 100.0;  // empty child fully matches
    return 100.0 * static_cast<double>(lcs_len) / static_cast<double>(child_len);
}

namespace {
bool is_ascii_space(char b) noexcept {
    return b == ' ' || b == '\t' || b == '\n' || b == '\v' || b == '\f' || b == '\r';
}
std::string read_file(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw InputError("cannot open '" + path.string() + "' for reading");
    std::ostringstream buffer;
    buffer << in.rdbuf();
    if (in.bad()) throw InputError("read failure on '" + path.string() + "'");
    return std::move(buffer).str();
}
}  // namespace

InputFormat format_from_path(const std::filesystem::path& path) noexcept {
    const auto ext = path.extension().string();
    return (ext == ".fa" || ext == ".fasta") ? InputFormat::Fasta : InputFormat::Plain;
}

Sequence parse_fasta(std::string_view bytes) {
    std::string symbols;
    bool in_record = false;
    std::size_t pos = 0;
    while (pos < bytes.size()) {
        std::size_t eol = bytes.find('\n', pos);
        if (eol == std::string_view::npos) eol = bytes.size();
        const std::string_view line = bytes.substr(pos, eol - pos);
        pos = eol + 1;
        if (!line.empty() && line.front() == '>') {
            if (in_record) break;  // first record only
            in_record = true;
            continue;
        }
        for (const char b : line) {
            if (is_ascii_space(b)) continue;
            if (!in_record) throw InputError("malformed FASTA: sequence data before the '>' header");
            symbols.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(b))));
        }
    }
    if (!in_record) throw InputError("malformed FASTA: no '>' header found");
    return Sequence(std::move(symbols));
}

void validate_dna_alphabet(const Sequence& seq) {
    for (std::size_t off = 0; off < seq.size(); ++off) {
        const char b = seq[off];
        if (!(b == 'A' || b == 'C' || b == 'G' || b == 'T'))
            throw InputError("symbol '" + std::string(1, b) + "' at offset " + std::to_string(off) +
                             " is outside the {A, C, G, T} alphabet");
    }
}

Sequence load_sequence(const std::filesystem::path& path, InputFormat format, bool validate_dna) {
    const std::string bytes = read_file(path);
    Sequence seq;
    if (format == InputFormat::Fasta) {
        seq = parse_fasta(bytes);
    } else {
        std::string stripped;
        stripped.reserve(bytes.size());
        for (const char b : bytes)
            if (!is_ascii_space(b)) stripped.push_back(b);
        seq = Sequence(std::move(stripped));
    }
    if (validate_dna) validate_dna_alphabet(seq);
    return seq;
}

void write_plain(const Sequence& seq, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw InputError("cannot open '" + path.string() + "' for writing");
    out.write(seq.data(), static_cast<std::streamsize>(seq.size()));
    if (!out) throw InputError("write failure on '" + path.string() + "'");
}

}  // namespace wavelcs
