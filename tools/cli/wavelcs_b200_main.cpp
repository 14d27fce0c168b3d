// wavelcs_b200 -- command-line front end on the GPU path (SURVEY.md 8(f)
// rank 2), mirroring the reference's tools/wavelcs_main.cpp subcommands and
// output lines (compute: "LCS length:", "Similarity:", "Fill time:", "LCS:";
// bench: the reference's cases, equivalence gate and 8-column CSV, or with
// --gcups the device throughput / roofline schema; gen).  The
// reference's CLI11 is not vendored, so arguments are parsed here.  Every
// computation goes through the C++ facade (include/wavelcs_b200.hpp) and thus
// the device; --workers / --block-size / --kernel are validated as the
// reference validates them and otherwise do not change the device path.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <iostream>
#include <string>
#include <utility>
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

KernelKind parse_kernel(const std::string& name) {
    for (KernelKind k : {KernelKind::Auto, KernelKind::Scalar, KernelKind::Avx2, KernelKind::Neon,
                         KernelKind::B200})
        if (name == kernel_name(k)) return k;
    throw ConfigError("--kernel must be one of auto, scalar, avx2, neon, b200; got '" + name + "'");
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
        else if (o == "--workers") {
            if (std::stoul(a.next(o)) == 0) throw ConfigError("worker count must be at least 1");
        } else if (o == "--block-size") {
            if (std::stoull(a.next(o)) == 0) throw ConfigError("block size must be at least 1");
        } else if (o == "--kernel") (void)resolve_kernel(parse_kernel(a.next(o)));
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

std::pair<size_t, size_t> parse_size(const std::string& st) {
    const size_t xpos = st.find_first_of("xX");
    if (xpos == std::string::npos || xpos == 0 || xpos + 1 >= st.size())
        throw ConfigError("--sizes entries must look like MxN, got '" + st + "'");
    try {
        return {std::stoull(st.substr(0, xpos)), std::stoull(st.substr(xpos + 1))};
    } catch (const std::exception&) {
        throw ConfigError("--sizes entries must look like MxN, got '" + st + "'");
    }
}

// --gcups: device throughput per size (bit-parallel length fill, best of R),
// the GPU variants' equivalence gate, and the fraction of the measured int
// roofline -- the B200 measurement; the default mode is the reference's.
int run_bench_gcups(const std::vector<std::pair<size_t, size_t>>& sizes, std::uint64_t seed,
                    unsigned reps, const std::string& out_path) {
    std::ofstream out(out_path, std::ios::trunc);
    if (!out) throw InputError("cannot open '" + out_path + "' for writing");
    out << "# wavelcs_b200 benchmark (device: B200, bit-parallel fill)\n";
    out << "# generator: mt19937_64, symbol = alphabet[next() % |alphabet|], alphabet=ACGT\n";
    out << "# seeds: parent = seed, child = seed + 0x9e3779b97f4a7c15\n";
    double peak_ops = 0.0;
    if (wlcs_probe_int_peak(3, &peak_ops) != WLCS_OK) throw DeviceError(wlcs_last_error());
    const double gcups_peak = peak_ops * 32.0 / 3.0 / 1e9;
    out << "# int roofline: " << gcups_peak << " GCUPS (measured int32 ALU peak x 32/3)\n";
    out << "M,N,repetitions,device_s,gcups,roofline_frac,lcs_length\n";
    for (const auto& [m, n] : sizes) {
        const Sequence x = generate_random(m, Sequence("ACGT"), seed);
        const Sequence y = generate_random(n, Sequence("ACGT"), seed + kChildSeedOffset);
        Length len = lcs_length(x, y, kNoMemoryBudget);  // warm-up
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
        for (unsigned r = 0; r < reps; ++r)
            best = std::min(best, time_fill([&] { len = lcs_length(x, y, kNoMemoryBudget); }));
        char line[256];
        const double gcups = double(m) * double(n) / best / 1e9;
        std::snprintf(line, sizeof line, "%zu,%zu,%u,%.6f,%.1f,%.4f,%u\n", m, n, reps, best, gcups,
                      gcups / gcups_peak, len);
        out << line;
        std::cout << line;
    }
    std::cout << "wrote " << sizes.size() << " records to " << out_path << '\n';
    return 0;
}

// The reference's bench subcommand (tools/wavelcs_main.cpp:110-139): the
// cases (--sizes or --table1, crossed with --workers), run_benchmark with its
// serial / parallel equivalence gate, and write_csv's 8-column schema.
int run_bench(Args& a) {
    std::vector<std::pair<size_t, size_t>> sizes;
    std::vector<unsigned> workers;
    std::string out_path;
    std::uint64_t seed = 1;
    unsigned reps = 3;
    size_t block = kDefaultBlockSize;
    bool table1 = false, gcups = false;
    KernelKind kernel = KernelKind::Auto;
    while (a.more()) {
        const std::string o = a.next("");
        if (o == "--sizes") {
            for (const auto& st : split(a.next(o), ',')) sizes.push_back(parse_size(st));
        } else if (o == "--table1") table1 = true;
        else if (o == "--gcups") gcups = true;
        else if (o == "--seed") seed = std::stoull(a.next(o));
        else if (o == "--repetitions") {
            reps = unsigned(std::stoul(a.next(o)));
            if (reps == 0) throw ConfigError("--repetitions must be positive");
        } else if (o == "--workers") {
            for (const auto& w : split(a.next(o), ',')) workers.push_back(unsigned(std::stoul(w)));
        } else if (o == "--block-size") block = std::stoull(a.next(o));
        else if (o == "--kernel") kernel = parse_kernel(a.next(o));
        else if (o == "--out") out_path = a.next(o);
        else throw ConfigError("unknown option " + o);
    }
    if (out_path.empty()) throw ConfigError("bench needs --out");
    if (sizes.empty() && !table1) throw ConfigError("bench needs --sizes or --table1");
    if (gcups) {
        if (table1)
            for (const BenchCase& c : table1_cases(1, block, seed))
                sizes.emplace_back(c.parent_len, c.child_len);
        return run_bench_gcups(sizes, seed, reps, out_path);
    }
    if (workers.empty()) workers.push_back(default_worker_count());
    std::vector<BenchCase> cases;
    for (const unsigned w : workers) {
        if (table1) {
            for (const BenchCase& c : table1_cases(w, block, seed, reps)) cases.push_back(c);
        } else {
            for (const auto& [m, n] : sizes) cases.push_back({m, n, w, block, seed, reps});
        }
    }
    BenchOptions options;
    options.kernel = kernel;
    options.progress = &std::cout;
    const std::vector<BenchRecord> records = run_benchmark(cases, options);
    write_csv(records, out_path);
    std::cout << "wrote " << records.size() << " records to " << out_path << '\n';
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
