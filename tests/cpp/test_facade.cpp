// test_facade.cpp -- the reference's own unit cases (proj/tests/test_core.cpp,
// test_parallel.cpp) re-expressed against the C++ facade, run on the GPU.
// Plain asserts (doctest is not available); exit status = failures.
#include <cstdio>
#include <random>
#include <string>

#include "wavelcs_b200.hpp"

using namespace wavelcs;

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

template <typename E, typename Fn>
static bool throws(Fn&& fn) {
    try {
        fn();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Sequence seq(const char* t) { return Sequence(t); }

static Sequence random_dna(std::mt19937_64& rng, std::size_t n) {
    static const char a[] = "ACGT";
    std::string s(n, 'A');
    for (auto& c : s) c = a[rng() % 4];
    return Sequence(s);
}

int main() {
    // test_core.cpp:58-62 lcs_length examples
    CHECK(lcs_length(seq(""), seq("")) == 0);
    CHECK(lcs_length(seq("ATGC"), seq("ATGC")) == 4);
    CHECK(lcs_length(seq("ABCBDAB"), seq("BDCABA")) == 4);
    // test_core.cpp:74-85 traceback on the classic pair follows the LEFT tie-break
    CHECK(lcs_subsequence(seq("ABCBDAB"), seq("BDCABA")) == seq("BDAB"));
    CHECK(lcs_subsequence(seq("ATGC"), seq("ATGC")) == seq("ATGC"));
    // test_core.cpp:122-126 capacity budget yields a clean error
    CHECK(throws<CapacityError>([] { lcs_length(seq("ATGC"), seq("ATGC"), 16); }));
    CHECK(!throws<CapacityError>([] { lcs_length(seq("ATGC"), seq("ATGC"), 1024); }));
    CHECK(throws<CapacityError>([] { lcs_length(seq(""), seq(""), 1); }));
    // test_core.cpp:128-138 symmetry and bounds
    std::mt19937_64 rng(2024);
    for (int round = 0; round < 50; ++round) {
        const Sequence x = random_dna(rng, rng() % 40), y = random_dna(rng, rng() % 40);
        const Length f = lcs_length(x, y);
        CHECK(f == lcs_length(y, x));
        CHECK(f <= std::min(x.size(), y.size()));
        CHECK(lcs_length(x, x) == x.size());
    }
    // test_core.cpp:140-151 appending a shared symbol extends the LCS by one
    std::mt19937_64 rng2(7);
    for (int round = 0; round < 50; ++round) {
        const Sequence x = random_dna(rng2, rng2() % 60), y = random_dna(rng2, rng2() % 60);
        const char shared = "ACGT"[rng2() % 4];
        CHECK(lcs_length(Sequence(x.str() + shared), Sequence(y.str() + shared)) ==
              lcs_length(x, y) + 1);
    }
    // test_core.cpp:182-193 traceback validity
    std::mt19937_64 rng3(31337);
    for (int round = 0; round < 40; ++round) {
        const Sequence x = random_dna(rng3, rng3() % 64), y = random_dna(rng3, rng3() % 64);
        const Sequence s = lcs_subsequence(x, y);
        CHECK(s.size() == lcs_length(x, y));
        CHECK(is_subsequence(s, x));
        CHECK(is_subsequence(s, y));
    }
    // test_parallel.cpp:191-199 lopsided 5000x200 (generate_random seeds 320/321)
    const Sequence dna("ACGT");
    const Sequence lx = generate_random(5000, dna, 320), ly = generate_random(200, dna, 321);
    CHECK(lcs_length(lx, ly) == lcs_length(ly, lx));
    // batch agrees with single calls
    std::vector<Sequence> xs, ys;
    for (int k = 0; k < 64; ++k) {
        xs.push_back(random_dna(rng3, rng3() % 300));
        ys.push_back(random_dna(rng3, rng3() % 300));
    }
    const auto lens = lcs_length_batch(xs, ys);
    for (int k = 0; k < 64; ++k) CHECK(lens[k] == lcs_length(xs[k], ys[k]));
    // full tables + traceback, as the reference's callers compose them
    // (test_core.cpp:50-56,74-85: BDAB; serial.hpp:21-30)
    {
        const FillResult f = lcs_fill_serial(seq("ABCBDAB"), seq("BDCABA"));
        CHECK(f.dp.final_length() == 4);
        CHECK(f.dp.rows() == 8 && f.dp.cols() == 7);
        CHECK(traceback(f.back, seq("ABCBDAB"), 7, 6) == seq("BDAB"));
        CHECK(f.back.at(1, 4) == Arrow::Diag);  // x_1 = A == y_4 = A
        CHECK(throws<std::out_of_range>([&] { traceback(f.back, seq("ABCBDAB"), 8, 6); }));
        CHECK(throws<CapacityError>([] { lcs_fill_serial(seq("ATGC"), seq("ATGC"), 16); }));
        const FillResult e = lcs_fill_serial(seq(""), seq("ATGC"));
        CHECK(e.dp.final_length() == 0 && e.dp.rows() == 1 && e.dp.cols() == 5);
        std::mt19937_64 rng4(5);
        for (int k = 0; k < 20; ++k) {
            const Sequence x = random_dna(rng4, 1 + rng4() % 120), y = random_dna(rng4, 1 + rng4() % 120);
            const FillResult t = lcs_fill_serial(x, y);
            CHECK(t.dp.final_length() == lcs_length(x, y));
            CHECK(traceback(t.back, x, x.size(), y.size()) == lcs_subsequence(x, y));
        }
    }
    std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
    return failures;
}
