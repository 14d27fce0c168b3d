// wavelcs_b200 -- command-line front end on the GPU path (SURVEY.md 8(f)
// rank 2), mirroring the reference's tools/wavelcs_main.cpp subcommands and
// output lines (compute: "LCS length:", "Similarity:", "Fill time:", "LCS:";
// bench: the reference CSV header extended with device GCUPS; gen).  The
// reference's CLI11 is not vendored, so arguments are parsed here.  Every
// computation goes through the C++ facade (include/wavelcs_b200.hpp) and thus
// the device; --workers / --block-size / --kernel are accepted for command-
// line compatibility and have no effect on the device path.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "wavelcs_b200.hpp"
#include "wavelcs_capi.h"

namespace {

using namespace wavelcs;

struct Args {
    std::vector<std::string> v;
    size_t i = 0;
    bool more() const { return i < v.size(); }
    std::string next(const std::string& opt) {
        if (i >= v.size()) throw ConfigError("option " + opt + " needs a value");
        return v[i++];
    }
};

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    size_t p = 0;
    while (p <= s.size()) {
        const size_t q = s.find(sep, p);
        out.push_back(s.substr(p, q == std::string::npos ? std::string::npos : q - p));
        if (q == std::string::npos) break;
        p = q + 1;
    }
    return out;
}

InputFormat pick_format(const std::string& flag, const std::string& path) {
    if (flag == "plain") return InputFormat::Plain;
    if (flag == "fasta") return InputFormat::Fasta;
    return format_from_path(path);
}

int run_compute(Args& a) {
    std::string parent, child, format;
    bool with_tb = false, validate = false;
    while (a.more()) {
        const std::string o = a.next("");
        if (o == "--parent") parent = a.next(o);
        else if (o == "--child") child = a.next(o);
        else if (o == "--traceback") with_tb = true;
        else if (o == "--format") {
            format = a.next(o);
            if (format != "plain" && format != "fasta")
                throw ConfigError("--format must be plain or fasta");
        } else if (o == "--validate-dna") validate = true;
        else if (o == "--workers" || o == "--block-size" || o == "--kernel") (void)a.next(o);
        else throw ConfigError("unknown option " + o);
    }
    if (parent.empty() || child.empty()) throw ConfigError("compute needs --parent and --child");
    const Sequence x = load_sequence(parent, pick_format(format, parent), validate);
    const Sequence y = load_sequence(child, pick_format(format, child), validate);
    const auto t0 = std::chrono::steady_clock::now();
    Sequence lcs;
    Length len;
    if (with_tb) {
        lcs = lcs_subsequence(x, y, kNoMemoryBudget);
        len = Length(lcs.size());
    } else {
        len = lcs_length(x, y, kNoMemoryBudget);
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("LCS length:  %u\n", len);
    std::printf("Similarity:  %.2f%% of the child sequence\n",
                similarity_percent(len, x.size(), y.size()));
    std::printf("Fill time:   %.6f s (device=B200, variant=bitparallel)\n", secs);
    if (with_tb) std::printf("LCS:         %s\n", lcs.str().c_str());
    return 0;
}

int run_bench(Args& a) {
    std::vector<std::string> sizes;
    std::string out_path;
    std::uint64_t seed = 1;
    unsigned reps = 3;
    while (a.more()) {
        const std::string o = a.next("");
        if (o == "--sizes") {
            for (const auto& s : split(a.next(o), ',')) sizes.push_back(s);
        } else if (o == "--seed") seed = std::stoull(a.next(o));
        else if (o == "--repetitions") {
            reps = unsigned(std::stoul(a.next(o)));
            if (reps == 0) throw ConfigError("--repetitions must be positive");
        } else if (o == "--out") out_path = a.next(o);
        else if (o == "--workers" || o == "--block-size" || o == "--kernel") (void)a.next(o);
        else throw ConfigError("unknown option " + o);
    }
    if (sizes.empty()) throw ConfigError("bench needs --sizes");
    if (out_path.empty()) throw ConfigError("bench needs --out");
    std::ofstream out(out_path, std::ios::trunc);
    if (!out) throw InputError("cannot open '" + out_path + "' for writing");
    out << "# wavelcs_b200 benchmark (device: B200, bit-parallel fill)\n";
    out << "# generator: mt19937_64, symbol = alphabet[next() % |alphabet|], alphabet=ACGT\n";
    out << "# seeds: parent = seed, child = seed + 0x9e3779b97f4a7c15\n";
    // roofline denominator: the device's measured int32 ALU peak, 3 ops per
    // 32-cell word-row
    double peak_ops = 0.0;
    if (wlcs_probe_int_peak(3, &peak_ops) != WLCS_OK) throw DeviceError(wlcs_last_error());
    const double gcups_peak = peak_ops * 32.0 / 3.0 / 1e9;
    out << "# int roofline: " << gcups_peak << " GCUPS (measured int32 ALU peak x 32/3)\n";
    out << "M,N,repetitions,device_s,gcups,roofline_frac,lcs_length\n";
    size_t n_rec = 0;
    for (const auto& st : sizes) {
        const size_t xpos = st.find_first_of("xX");
        if (xpos == std::string::npos || xpos == 0 || xpos + 1 >= st.size())
            throw ConfigError("--sizes entries must look like MxN, got '" + st + "'");
        const size_t m = std::stoull(st.substr(0, xpos)), n = std::stoull(st.substr(xpos + 1));
        const Sequence x = generate_random(m, Sequence("ACGT"), seed);
        const Sequence y = generate_random(n, Sequence("ACGT"), seed + 0x9e3779b97f4a7c15ull);
        Length len = lcs_length(x, y, kNoMemoryBudget);  // warm-up
        // equivalence gate (bench.cpp:100-106 semantics): the two device
        // fill variants must agree
        std::uint32_t wave = 0;
        if (wlcs_length_ex(reinterpret_cast<const std::uint8_t*>(x.data()), m,
                           reinterpret_cast<const std::uint8_t*>(y.data()), n, WLCS_NO_BUDGET,
                           WLCS_VARIANT_WAVEFRONT, &wave) != WLCS_OK)
            throw DeviceError(wlcs_last_error());
        if (wave != len)
            throw EquivalenceError("M=" + std::to_string(m) + " N=" + std::to_string(n) +
                                   ": bit-parallel " + std::to_string(len) + " vs wavefront " +
                                   std::to_string(wave));
        double best = 1e300;
        for (unsigned r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            len = lcs_length(x, y, kNoMemoryBudget);
            best = std::min(best, std::chrono::duration<double>(
                                      std::chrono::steady_clock::now() - t0).count());
        }
        char line[256];
        const double gcups = double(m) * double(n) / best / 1e9;
        std::snprintf(line, sizeof line, "%zu,%zu,%u,%.6f,%.1f,%.4f,%u\n", m, n, reps, best,
                      gcups, gcups / gcups_peak, len);
        out << line;
        std::cout << line;
        ++n_rec;
    }
    std::cout << "wrote " << n_rec << " records to " << out_path << '\n';
    return 0;
}

int run_gen(Args& a) {
    size_t length = 0;
    bool have_len = false, have_seed = false;
    std::string alphabet = "ACGT", out_path;
    std::uint64_t seed = 0;
    while (a.more()) {
        const std::string o = a.next("");
        if (o == "--length") {
            length = std::stoull(a.next(o));
            have_len = true;
        } else if (o == "--alphabet") alphabet = a.next(o);
        else if (o == "--seed") {
            seed = std::stoull(a.next(o));
            have_seed = true;
        } else if (o == "--out") out_path = a.next(o);
        else throw ConfigError("unknown option " + o);
    }
    if (!have_len || !have_seed || out_path.empty())
        throw ConfigError("gen needs --length, --seed and --out");
    write_plain(generate_random(length, Sequence(alphabet), seed), out_path);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args a;
    for (int k = 1; k < argc; ++k) a.v.emplace_back(argv[k]);
    if (a.v.empty()) {
        std::cerr << "usage: wavelcs_b200 {compute|bench|gen} [options]\n";
        return 1;
    }
    try {
        const std::string cmd = a.next("");
        if (cmd == "compute") return run_compute(a);
        if (cmd == "bench") return run_bench(a);
        if (cmd == "gen") return run_gen(a);
        throw ConfigError("unknown subcommand " + cmd);
    } catch (const std::exception& err) {
        std::cerr << "error: " << err.what() << '\n';
        return 1;
    }
}
