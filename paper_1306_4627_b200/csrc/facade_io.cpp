// facade_io.cpp -- sequence I/O of the reference API (include/wavelcs/io.hpp)
// with the reference's formats, bytes and error behaviour
// (/root/reference/proj/src/io.cpp:38-135; error texts kept byte for byte,
// since callers and tests match on them).  Host code: the bytes then go to
// the device through the C-ABI's pinned staging.
#include <array>
#include <cctype>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#include "wavelcs_b200.hpp"
#include "wavelcs_capi.h"

namespace wavelcs {
namespace {

// ASCII whitespace as the reference strips it: ' ' \t \n \v \f \r.
constexpr std::array<bool, 256> kSpace = [] {
    std::array<bool, 256> t{};
    for (unsigned char c : {' ', '\t', '\n', '\v', '\f', '\r'}) t[c] = true;
    return t;
}();

inline bool space(char c) noexcept { return kSpace[static_cast<unsigned char>(c)]; }

std::string slurp(const std::filesystem::path& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw InputError("cannot open '" + path.string() + "' for reading");
    std::string data;
    std::array<char, 1 << 16> chunk;
    std::size_t got;
    while ((got = std::fread(chunk.data(), 1, chunk.size(), f)) > 0) data.append(chunk.data(), got);
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) throw InputError("read failure on '" + path.string() + "'");
    return data;
}

}  // namespace

InputFormat format_from_path(const std::filesystem::path& path) noexcept {
    const std::string ext = path.extension().string();
    return ext == ".fa" || ext == ".fasta" ? InputFormat::Fasta : InputFormat::Plain;
}

Sequence parse_fasta(std::string_view bytes) {
    // states: before the first header, inside the first record; a second
    // header ends the scan
    enum { Before, Inside } state = Before;
    std::string out;
    std::size_t line_start = 0;
    while (line_start < bytes.size()) {
        std::size_t line_end = bytes.find('\n', line_start);
        if (line_end == std::string_view::npos) line_end = bytes.size();
        const std::string_view line = bytes.substr(line_start, line_end - line_start);
        line_start = line_end + 1;
        if (!line.empty() && line[0] == '>') {
            if (state == Inside) break;
            state = Inside;
            continue;
        }
        for (char c : line) {
            if (space(c)) continue;
            if (state == Before) throw InputError("malformed FASTA: sequence data before the '>' header");
            out += static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
        }
    }
    if (state == Before) throw InputError("malformed FASTA: no '>' header found");
    return Sequence(std::move(out));
}

void validate_dna_alphabet(const Sequence& seq) {
    const std::string& s = seq.str();
    const std::size_t bad = s.find_first_not_of("ACGT");
    if (bad != std::string::npos)
        throw InputError("symbol '" + std::string(1, s[bad]) + "' at offset " + std::to_string(bad) +
                         " is outside the {A, C, G, T} alphabet");
}

Sequence load_sequence(const std::filesystem::path& path, InputFormat format, bool validate_dna) {
    std::string raw = slurp(path);
    Sequence seq;
    if (format == InputFormat::Fasta) {
        seq = parse_fasta(raw);
    } else {
        std::erase_if(raw, space);
        seq = Sequence(std::move(raw));
    }
    if (validate_dna) validate_dna_alphabet(seq);
    return seq;
}

Sequence generate_random(std::size_t length, const Sequence& alphabet, std::uint64_t seed) {
    if (alphabet.empty()) throw std::invalid_argument("generate_random: alphabet must not be empty");
    std::string s(length, '\0');
    if (wlcs_generate_random(length, reinterpret_cast<const std::uint8_t*>(alphabet.data()),
                             alphabet.size(), seed, reinterpret_cast<std::uint8_t*>(s.data())))
        throw std::invalid_argument(wlcs_last_error());
    return Sequence(std::move(s));
}

void write_plain(const Sequence& seq, const std::filesystem::path& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw InputError("cannot open '" + path.string() + "' for writing");
    out.write(seq.data(), static_cast<std::streamsize>(seq.size()));
    if (!out) throw InputError("write failure on '" + path.string() + "'");
}

}  // namespace wavelcs
