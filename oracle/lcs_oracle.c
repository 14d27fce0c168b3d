/*
 * oracle/lcs_oracle.c -- CPU restatement of the reference LCS table fill.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_1306_4627_b200/) links, loads or calls this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it, and only
 * as the checker.
 *
 * Pinning: every function below is cross-checked in tests/test_oracle.py
 * against (a) the reference's own golden vectors (proj/tests/test_core.cpp,
 * test_kernels.cpp, acceptance.cpp) and (b) the reference library itself,
 * compiled from /root/reference/proj/src into oracle/_ref/ by oracle/Makefile
 * (fixtures generated from it are committed under tests/golden/).
 *
 * Reference semantics restated here (paths relative to /root/reference/proj):
 *   lcs_cell            include/wavelcs/cell.hpp:30-38
 *   fill_block_scalar   src/kernels_scalar.cpp:5-17 (row-major, 1-based)
 *   DpTable layout      include/wavelcs/tables.hpp:20-45  ((M+1)x(N+1) uint32)
 *   BacktrackTable      include/wavelcs/tables.hpp:49-71  (MxN uint8, init Left)
 *   check_capacity      src/tables.cpp:9-24
 *   traceback           src/serial.cpp:36-61
 *   brute_force_lcs     src/serial.cpp:63-89
 *   is_subsequence      src/sequence.cpp:8-16
 *   generate_random     src/io.cpp:103-115 (std::mt19937_64, alphabet[r % |A|])
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ARROW_DIAG 0u
#define ARROW_UP 1u
#define ARROW_LEFT 2u

/* lcs_cell, cell.hpp:30-38: match -> diag+1/Diag; up > left -> up/Up;
 * else left/Left (strict '>' makes ties go LEFT). */
static inline uint32_t cell_value(uint8_t xi, uint8_t yj, uint32_t diag, uint32_t up,
                                  uint32_t left, uint8_t* arrow) {
    if (xi == yj) {
        *arrow = ARROW_DIAG;
        return diag + 1u;
    }
    if (up > left) {
        *arrow = ARROW_UP;
        return up;
    }
    *arrow = ARROW_LEFT;
    return left;
}

/* check_capacity, tables.cpp:9-24: 4(M+1)(N+1) + MN bytes in 128-bit.
 * Returns 1 when the request exceeds the budget (the reference throws). */
int orc_capacity_exceeded(uint64_t m, uint64_t n, uint64_t budget) {
    unsigned __int128 bytes = (unsigned __int128)(m + 1) * (unsigned __int128)(n + 1) * 4u +
                              (unsigned __int128)m * (unsigned __int128)n;
    return bytes > (unsigned __int128)budget;
}

/* Two-row restatement of fill_block_scalar over the whole grid
 * (kernels_scalar.cpp:6-16, serial.cpp:11-30) keeping only values. */
uint32_t orc_length_cells(const uint8_t* x, size_t m, const uint8_t* y, size_t n) {
    if (m == 0 || n == 0) return 0;
    uint32_t* prev = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    uint32_t* cur = (uint32_t*)calloc(n + 1, sizeof(uint32_t));
    if (!prev || !cur) {
        free(prev);
        free(cur);
        return UINT32_MAX;
    }
    for (size_t i = 1; i <= m; ++i) {
        const uint8_t xi = x[i - 1];
        cur[0] = 0;
        for (size_t j = 1; j <= n; ++j) {
            uint8_t a;
            cur[j] = cell_value(xi, y[j - 1], prev[j - 1], prev[j], cur[j - 1], &a);
        }
        uint32_t* t = prev;
        prev = cur;
        cur = t;
    }
    uint32_t r = prev[n];
    free(prev);
    free(cur);
    return r;
}

/* Full reference tables: dp is (m+1)*(n+1) uint32 row-major, back is m*n
 * arrows (Diag=0, Up=1, Left=2), exactly tables.hpp:20-71 layouts. */
void orc_fill_tables(const uint8_t* x, size_t m, const uint8_t* y, size_t n, uint32_t* dp,
                     uint8_t* back) {
    const size_t cs = n + 1;
    memset(dp, 0, (m + 1) * cs * sizeof(uint32_t));
    if (m * n != 0) memset(back, ARROW_LEFT, m * n);
    for (size_t i = 1; i <= m; ++i) {
        uint32_t* cur = dp + i * cs;
        const uint32_t* prv = cur - cs;
        uint8_t* arr = back + (i - 1) * n;
        for (size_t j = 1; j <= n; ++j) {
            cur[j] = cell_value(x[i - 1], y[j - 1], prv[j - 1], prv[j], cur[j - 1], &arr[j - 1]);
        }
    }
}

/* traceback, serial.cpp:36-61.  Returns the subsequence length written to
 * out (forward order); returns (size_t)-1 when (i, j) is outside the table. */
size_t orc_traceback(const uint8_t* back, size_t rows, size_t cols, const uint8_t* x, size_t i,
                     size_t j, uint8_t* out) {
    if (i > rows || j > cols) return (size_t)-1;
    size_t len = 0;
    while (i > 0 && j > 0) {
        const uint8_t a = back[(i - 1) * cols + (j - 1)];
        if (a == ARROW_DIAG) {
            out[len++] = x[i - 1];
            --i;
            --j;
        } else if (a == ARROW_UP) {
            --i;
        } else {
            --j;
        }
    }
    for (size_t k = 0; k < len / 2; ++k) {
        uint8_t t = out[k];
        out[k] = out[len - 1 - k];
        out[len - 1 - k] = t;
    }
    return len;
}

/* ---------------------------------------------------------------------
 * Bit-parallel restatement (Allison-Dix / Hyyro, 64-bit words).
 * Column j (1-based) of row i is bit (j-1) of V_i.  V_0 = all ones,
 * U = V & PM[x_i], V' = (V + U) | (V & ~PM[x_i]).  Then
 * c[i][j] = popcount(~V_i & ((1 << j) - 1)), so LCS = N - popcount(V_M).
 * The identity with lcs_cell values is checked exhaustively in
 * tests/test_oracle.py (and was verified in SURVEY.md section 8(a)).
 * ------------------------------------------------------------------- */
static void build_pm64(const uint8_t* y, size_t n, size_t words, uint64_t* pm /* 256*words */) {
    memset(pm, 0, 256 * words * sizeof(uint64_t));
    for (size_t j = 0; j < n; ++j) pm[(size_t)y[j] * words + (j >> 6)] |= 1ull << (j & 63);
}

static inline void bitpar_row(uint64_t* V, const uint64_t* P, size_t words) {
    unsigned carry = 0;
    for (size_t w = 0; w < words; ++w) {
        const uint64_t v = V[w];
        const uint64_t u = v & P[w];
        const uint64_t s1 = v + u;
        const unsigned c1 = s1 < v;
        const uint64_t s = s1 + carry;
        const unsigned c2 = s < s1;
        carry = c1 | c2;
        V[w] = s | (v & ~P[w]);
    }
}

static size_t zeros_in_prefix(const uint64_t* V, size_t nbits) {
    size_t full = nbits >> 6, z = 0;
    for (size_t w = 0; w < full; ++w) z += (size_t)__builtin_popcountll(~V[w]);
    if (nbits & 63) z += (size_t)__builtin_popcountll(~V[full] & ((1ull << (nbits & 63)) - 1));
    return z;
}

uint32_t orc_length_bitpar(const uint8_t* x, size_t m, const uint8_t* y, size_t n) {
    if (m == 0 || n == 0) return 0;
    const size_t words = (n + 63) >> 6;
    uint64_t* pm = (uint64_t*)malloc(256 * words * sizeof(uint64_t));
    uint64_t* V = (uint64_t*)malloc(words * sizeof(uint64_t));
    if (!pm || !V) {
        free(pm);
        free(V);
        return UINT32_MAX;
    }
    build_pm64(y, n, words, pm);
    for (size_t w = 0; w < words; ++w) V[w] = ~0ull;
    for (size_t i = 0; i < m; ++i) bitpar_row(V, pm + (size_t)x[i] * words, words);
    uint32_t r = (uint32_t)zeros_in_prefix(V, n);
    free(pm);
    free(V);
    return r;
}

/* Batch convenience for the tests: lengths of many packed pairs. */
void orc_length_batch(const uint8_t* xs, const uint64_t* xoff, const uint8_t* ys,
                      const uint64_t* yoff, size_t pairs, uint32_t* out) {
    for (size_t p = 0; p < pairs; ++p)
        out[p] = orc_length_bitpar(xs + xoff[p], (size_t)(xoff[p + 1] - xoff[p]), ys + yoff[p],
                                   (size_t)(yoff[p + 1] - yoff[p]));
}

/* Exact reference traceback computed from stored bit rows instead of the
 * arrow table (memory M*N/8 bytes instead of 5*M*N).  Walk rule
 * (serial.cpp:44-58 with the arrows of cell.hpp:30-38):
 *   x_i == y_j             -> Diag (emit x_i)
 *   c[i-1][j] > c[i][j-1]  -> Up
 *   otherwise              -> Left
 * c values come from prefix zero counts of the rows, accelerated by a
 * per-row cumulative count every 512 bits.
 * Returns the length, or -1 on allocation failure. */
int64_t orc_subsequence_bitrows(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                                uint8_t* out) {
    if (m == 0 || n == 0) return 0;
    const size_t words = (n + 63) >> 6;
    const size_t blocks = (words + 7) >> 3; /* 512-bit blocks */
    uint64_t* pm = (uint64_t*)malloc(256 * words * sizeof(uint64_t));
    uint64_t* rows = (uint64_t*)malloc((m + 1) * words * sizeof(uint64_t));
    uint32_t* cum = (uint32_t*)malloc((m + 1) * blocks * sizeof(uint32_t));
    if (!pm || !rows || !cum) {
        free(pm);
        free(rows);
        free(cum);
        return -1;
    }
    build_pm64(y, n, words, pm);
    for (size_t w = 0; w < words; ++w) rows[w] = ~0ull;
    for (size_t i = 1; i <= m; ++i) {
        memcpy(rows + i * words, rows + (i - 1) * words, words * sizeof(uint64_t));
        bitpar_row(rows + i * words, pm + (size_t)x[i - 1] * words, words);
    }
    for (size_t i = 0; i <= m; ++i) {
        const uint64_t* R = rows + i * words;
        uint32_t acc = 0;
        for (size_t b = 0; b < blocks; ++b) {
            cum[i * blocks + b] = acc;
            for (size_t w = b * 8; w < words && w < b * 8 + 8; ++w)
                acc += (uint32_t)__builtin_popcountll(~R[w]);
        }
    }
#define C_AT(ii, jj)                                                                        \
    (cum[(ii) * blocks + ((jj) >> 9)] +                                                     \
     (uint32_t)zeros_in_prefix(rows + (ii) * words + (((jj) >> 9) << 3), (jj) & 511))
    size_t i = m, j = n, len = 0;
    while (i > 0 && j > 0) {
        if (x[i - 1] == y[j - 1]) {
            out[len++] = x[i - 1];
            --i;
            --j;
        } else if (C_AT(i - 1, j) > C_AT(i, j - 1)) {
            --i;
        } else {
            --j;
        }
    }
#undef C_AT
    for (size_t k = 0; k < len / 2; ++k) {
        uint8_t t = out[k];
        out[k] = out[len - 1 - k];
        out[len - 1 - k] = t;
    }
    free(pm);
    free(rows);
    free(cum);
    return (int64_t)len;
}

/* brute_force_lcs, serial.cpp:63-89 (enumerate subsets of the shorter). */
int orc_is_subsequence(const uint8_t* cand, size_t cn, const uint8_t* text, size_t tn) {
    size_t matched = 0;
    for (size_t pos = 0; pos < tn && matched < cn; ++pos)
        if (text[pos] == cand[matched]) ++matched;
    return matched == cn;
}

int64_t orc_brute_force(const uint8_t* x, size_t m, const uint8_t* y, size_t n) {
    const uint8_t* s = m <= n ? x : y;
    const uint8_t* l = m <= n ? y : x;
    const size_t sn = m <= n ? m : n, ln = m <= n ? n : m;
    if (sn > 20) return -1;
    uint32_t best = 0;
    uint8_t cand[20];
    for (uint64_t mask = 0; mask < (1ull << sn); ++mask) {
        uint32_t picked = (uint32_t)__builtin_popcountll(mask);
        if (picked <= best) continue;
        size_t c = 0;
        for (size_t p = 0; p < sn; ++p)
            if (mask & (1ull << p)) cand[c++] = s[p];
        if (orc_is_subsequence(cand, c, l, ln)) best = picked;
    }
    return best;
}

/* ---------------------------------------------------------------------
 * generate_random, io.cpp:103-115: std::mt19937_64 (published MT19937-64
 * parameters, pinned by the C++ standard) and symbol = alphabet[r % |A|].
 * ------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t xv = (s->mt[i] & 0xFFFFFFFF80000000ull) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = xv >> 1;
            if (xv & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

void orc_generate_random(size_t length, const uint8_t* alphabet, size_t alen, uint64_t seed,
                         uint8_t* out) {
    mt64_t s;
    mt64_seed(&s, seed);
    for (size_t k = 0; k < length; ++k) out[k] = alphabet[mt64_next(&s) % alen];
}

/* ---------------------------------------------------------------------
 * Column-strip decomposition (the multi-GPU / multi-warp interface):
 * rows [0, rows) of the bit-parallel fill restricted to columns
 * [c0, c0 + ns) of y, with the strip's bit vector V (ceil(ns/64) words)
 * carried across calls, carry_in[i] (0/1) injected into the strip's lowest
 * column for row i and carry_out[i] = the carry leaving column c0+ns-1.
 * ns must be a multiple of 64 except for the rightmost strip, so that the
 * carry out of the last word is the carry out of the strip.  Chaining the
 * strips left to right reproduces the whole-row fill (SURVEY.md section 7,
 * "decompositions verified exact").
 * ------------------------------------------------------------------- */
void orc_strip_rows(const uint8_t* x, size_t rows, const uint8_t* ystrip, size_t ns,
                    uint64_t* V, const uint8_t* carry_in, uint8_t* carry_out) {
    const size_t words = (ns + 63) >> 6;
    uint64_t* pm = (uint64_t*)malloc(256 * (words ? words : 1) * sizeof(uint64_t));
    if (!pm) return;
    build_pm64(ystrip, ns, words, pm);
    for (size_t i = 0; i < rows; ++i) {
        const uint64_t* P = pm + (size_t)x[i] * words;
        unsigned carry = carry_in ? carry_in[i] : 0u;
        for (size_t w = 0; w < words; ++w) {
            const uint64_t v = V[w];
            const uint64_t u = v & P[w];
            const uint64_t s1 = v + u;
            const unsigned c1 = s1 < v;
            const uint64_t s = s1 + carry;
            const unsigned c2 = s < s1;
            carry = c1 | c2;
            V[w] = s | (v & ~P[w]);
        }
        if (carry_out) carry_out[i] = (uint8_t)carry;
    }
    free(pm);
}

/* zero bits of V below ns (the strip's contribution to the LCS length) */
uint64_t orc_strip_zeros(const uint64_t* V, size_t ns) { return zeros_in_prefix(V, ns); }

/* ---------------------------------------------------------------------
 * Full-size check (i) of SURVEY.md 8(c): the two-row lcs_cell loop of
 * orc_length_cells (kernels_scalar.cpp:6-16 + cell.hpp:30-38, values only)
 * spread over `threads` column strips so that 1e12-cell configurations (C4,
 * C5) finish in minutes.  Strip t keeps its own row segment; for every row it
 * needs the left neighbour's value in column lo_t - 1 of this row (left) and
 * of the previous row (diag), which strip t-1 publishes in edge[t-1][i]
 * followed by a release store of its row counter.  Same arithmetic as the
 * one-thread loop; only the order in which independent cells are visited
 * changes.  Returns UINT32_MAX on allocation failure.
 * ------------------------------------------------------------------- */
#include <pthread.h>
#include <stdatomic.h>
#include <sched.h>

typedef struct {
    const uint8_t* x;
    size_t m;
    const uint8_t* y;
    size_t lo, hi;            /* columns [lo, hi), 1-based j = lo+1 .. hi */
    uint32_t* edge_in;        /* left strip's last column per row, NULL for t = 0 */
    _Atomic size_t* ready_in; /* rows published by the left strip */
    uint32_t* edge_out;       /* this strip's last column per row (m + 1) */
    _Atomic size_t* ready_out;
    uint32_t last;
} cells_strip_t;

#define CELLS_PUBLISH_ROWS 256

static void* cells_strip_main(void* arg) {
    cells_strip_t* s = (cells_strip_t*)arg;
    const size_t w = s->hi - s->lo;
    uint32_t* row = (uint32_t*)calloc(w + 1, sizeof(uint32_t)); /* row[0] = column lo */
    if (!row) {
        s->last = UINT32_MAX;
        return NULL;
    }
    const uint8_t* ys = s->y + s->lo;
    size_t avail = 0;
    for (size_t i = 1; i <= s->m; ++i) {
        if (s->edge_in) {
            while (avail < i) {
                avail = atomic_load_explicit(s->ready_in, memory_order_acquire);
                if (avail < i) sched_yield();
            }
        }
        const uint8_t xi = s->x[i - 1];
        uint32_t diag = row[0];                          /* c[i-1][lo] */
        uint32_t left = s->edge_in ? s->edge_in[i] : 0u; /* c[i][lo]   */
        row[0] = left;
        for (size_t k = 1; k <= w; ++k) {
            const uint32_t up = row[k];
            uint8_t a;
            left = cell_value(xi, ys[k - 1], diag, up, left, &a);
            diag = up;
            row[k] = left;
        }
        s->edge_out[i] = row[w];
        if ((i % CELLS_PUBLISH_ROWS) == 0 || i == s->m)
            atomic_store_explicit(s->ready_out, i, memory_order_release);
    }
    s->last = row[w];
    free(row);
    return NULL;
}

uint32_t orc_length_cells_mt(const uint8_t* x, size_t m, const uint8_t* y, size_t n,
                             int threads) {
    if (m == 0 || n == 0) return 0;
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = (int)n;
    cells_strip_t* st = (cells_strip_t*)calloc((size_t)threads, sizeof(cells_strip_t));
    uint32_t* edges = (uint32_t*)calloc((size_t)threads * (m + 1), sizeof(uint32_t));
    _Atomic size_t* ready = (_Atomic size_t*)calloc((size_t)threads, sizeof(_Atomic size_t));
    pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!st || !edges || !ready || !tid) {
        free(st);
        free(edges);
        free((void*)ready);
        free(tid);
        return UINT32_MAX;
    }
    for (int t = 0; t < threads; ++t) {
        st[t].x = x;
        st[t].m = m;
        st[t].y = y;
        st[t].lo = n * (size_t)t / (size_t)threads;
        st[t].hi = n * (size_t)(t + 1) / (size_t)threads;
        st[t].edge_in = t ? edges + (size_t)(t - 1) * (m + 1) : NULL;
        st[t].ready_in = t ? &ready[t - 1] : NULL;
        st[t].edge_out = edges + (size_t)t * (m + 1);
        st[t].ready_out = &ready[t];
        atomic_init(&ready[t], 0);
    }
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, cells_strip_main, &st[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    uint32_t r = st[threads - 1].last;
    for (int t = 0; t < threads; ++t)
        if (st[t].last == UINT32_MAX) r = UINT32_MAX;
    free(st);
    free(edges);
    free((void*)ready);
    free(tid);
    return r;
}

/* The C2 batch generator of bench.py / tests, restated on the oracle side so
 * that the reference arm never loads the product library: master =
 * std::mt19937_64(seed); per pair m = lo + master() % (hi - lo + 1), n
 * likewise, then seed_x = master(), seed_y = master() and the strings are
 * generate_random(m, alphabet, seed_x) / generate_random(n, alphabet, seed_y)
 * (io.cpp:103-115).  Same procedure as wlcs_generate_pairs
 * (include/wavelcs_capi.h); tests/test_oracle.py checks they agree byte for
 * byte.  xs / ys must hold pairs * hi bytes, offsets pairs + 1 entries. */
void orc_generate_pairs(size_t pairs, size_t lo, size_t hi, const uint8_t* alphabet, size_t alen,
                        uint64_t seed, uint8_t* xs, uint64_t* x_off, uint8_t* ys,
                        uint64_t* y_off) {
    mt64_t master;
    mt64_seed(&master, seed);
    uint64_t xo = 0, yo = 0;
    x_off[0] = y_off[0] = 0;
    for (size_t k = 0; k < pairs; ++k) {
        const size_t m = lo + (size_t)(mt64_next(&master) % (uint64_t)(hi - lo + 1));
        const size_t n = lo + (size_t)(mt64_next(&master) % (uint64_t)(hi - lo + 1));
        const uint64_t sx = mt64_next(&master), sy = mt64_next(&master);
        orc_generate_random(m, alphabet, alen, sx, xs + xo);
        orc_generate_random(n, alphabet, alen, sy, ys + yo);
        xo += m;
        yo += n;
        x_off[k + 1] = xo;
        y_off[k + 1] = yo;
    }
}
