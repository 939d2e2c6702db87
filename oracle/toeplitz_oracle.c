/*
 * oracle/toeplitz_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for Toeplitz-hashing randomness
 * extraction (arXiv 2011.04130, Zhao / Ma / Zhou, Sec. III.B).  It exists to
 * check the CUDA path bit for bit.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load it.  It shares
 * no code, header, table or helper with paper_2011_04130_b200/csrc and it
 * never calls into it.
 *
 * What it computes (Sec. III.B, the displayed m x n
 * Toeplitz matrix; "preserving k_n to k_{n+m-1}"):
 *
 *     k = T r  (mod 2),   T[i][j] = a_{n+i-j}   (1-based i, j, a)
 *
 * Row 1 of the displayed matrix is (a_n, a_{n-1}, ..., a_1); the last row is
 * (a_{n+m-1}, ..., a_m); every diagonal is constant.  With the
 * 0-based seed s[k] = a_{k+1} and 0-based i < m, j < n this is
 *
 *     y_i = XOR_{j=0}^{n-1} ( s[i - j + n - 1] AND x_j ).          (C1)
 *
 * Conventions fixed by BASELINE.json / SURVEY.md Sec. 0:
 *   C2  every bit stream is MSB-first: bit k of a byte buffer is
 *       (buf[k>>3] >> (7-(k&7))) & 1 -- raw bits, seed and output alike.
 *   C3  block b is raw bits [b*n, (b+1)*n).
 *   C4  output: block b's y_i is global output bit b*m + i; pad bits of the
 *       last byte are 0; ceil(n_blocks*m/8) bytes.
 *
 * Two modes, same formula:
 *   (i)  oracle_extract_scalar : the literal bit loop of (C1).
 *   (ii) oracle_extract_words  : (C1) with 64 values of j per AND/XOR.  Row i
 *        of T, read along j, is s[i+n-1], s[i+n-2], ..., s[i] -- i.e. the
 *        window rs[m-1-i .. m-1-i+n) of the reversed seed rs[k] = s[L-1-k].
 *        The accumulator XORs (window AND x) 64 bits at a time; y_i is the
 *        parity of the accumulator.  Nothing is blocked, fused or reordered
 *        beyond taking 64 consecutive j at once.
 *
 * Both parallelise over blocks with OpenMP (blocks are independent,
 * PAPER.md:273, Fig. 5).  Return value: 0 ok, -1 bad arguments.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline int get_bit(const uint8_t *buf, uint64_t k) {
    return (buf[k >> 3] >> (7 - (k & 7))) & 1;
}

static inline void or_bit(uint8_t *buf, uint64_t k, int v) {
    if (v) buf[k >> 3] |= (uint8_t)(1u << (7 - (k & 7)));
}

static int check_args(uint64_t n_blocks, uint64_t n, uint64_t m) {
    if (n == 0 || m == 0 || m >= n || n_blocks == 0) return -1;
    return 0;
}

static void set_threads(int n_threads) {
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- mode (i): literal bit loop of (C1) -------------------------------- */

/* y for ONE block, written to out_block (m bits MSB-first from bit 0; the
 * buffer must be zeroed, ceil(m/8) bytes). */
static void block_scalar(const uint8_t *raw, uint64_t b, uint64_t n, uint64_t m,
                         const uint8_t *seed, uint8_t *out, uint64_t out_bit0) {
    for (uint64_t i = 0; i < m; ++i) {
        int acc = 0;
        for (uint64_t j = 0; j < n; ++j) {
            /* s[i - j + n - 1] AND x_j ; the index is in [0, n+m-1). */
            acc ^= get_bit(seed, i + n - 1 - j) & get_bit(raw, b * n + j);
        }
        or_bit(out, out_bit0 + i, acc);
    }
}

int oracle_extract_scalar(const uint8_t *raw, uint64_t n_blocks, uint64_t n,
                          uint64_t m, const uint8_t *seed, uint8_t *out,
                          int n_threads) {
    if (check_args(n_blocks, n, m)) return -1;
    set_threads(n_threads);
    uint64_t out_bytes = (n_blocks * m + 7) / 8;
    memset(out, 0, out_bytes);
    /* Blocks whose outputs share a byte must not race on |=: give each block
     * its own scratch and merge serially. */
    uint64_t blk_bytes = (m + 7) / 8;
    uint8_t *scratch = (uint8_t *)calloc(n_blocks, blk_bytes);
    if (!scratch) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < (int64_t)n_blocks; ++b)
        block_scalar(raw, (uint64_t)b, n, m, seed, scratch + (uint64_t)b * blk_bytes, 0);
    for (uint64_t b = 0; b < n_blocks; ++b)
        for (uint64_t i = 0; i < m; ++i)
            or_bit(out, b * m + i, get_bit(scratch + b * blk_bytes, i));
    free(scratch);
    return 0;
}

/* ---- mode (ii): same formula, 64 j per AND/XOR ---------------------------- */

/* Pack bits [off, off+len) of an MSB-first stream into LSB-first uint64 words:
 * value with stream index off+q goes to bit (q & 63) of word q >> 6. */
static void pack_lsb64(const uint8_t *buf, uint64_t off, uint64_t len, uint64_t *w,
                       uint64_t n_words) {
    memset(w, 0, n_words * sizeof(uint64_t));
    for (uint64_t q = 0; q < len; ++q)
        if (get_bit(buf, off + q)) w[q >> 6] |= (uint64_t)1 << (q & 63);
}

/* 64 consecutive values starting at index o of an LSB-first word array. */
static inline uint64_t window64(const uint64_t *w, uint64_t o) {
    uint64_t q = o >> 6, r = o & 63;
    if (r == 0) return w[q];
    return (w[q] >> r) | (w[q + 1] << (64 - r));
}

typedef struct {
    uint64_t L, nw, rw_words;
    uint64_t *rs;     /* reversed seed rs[k] = s[L-1-k], LSB-first words, zero padded */
} seed_ctx;

static int seed_ctx_init(seed_ctx *c, const uint8_t *seed, uint64_t n, uint64_t m) {
    c->L = n + m - 1;
    c->nw = (n + 63) / 64;
    /* windows start at o <= m-1 and read nw words + 1 spill word */
    c->rw_words = (m - 1) / 64 + c->nw + 2;
    c->rs = (uint64_t *)calloc(c->rw_words, sizeof(uint64_t));
    if (!c->rs) return -1;
    for (uint64_t k = 0; k < c->L; ++k)
        if (get_bit(seed, c->L - 1 - k)) c->rs[k >> 6] |= (uint64_t)1 << (k & 63);
    return 0;
}

static void block_words(const uint8_t *raw, uint64_t b, uint64_t n, uint64_t m,
                        const seed_ctx *c, uint64_t *xw, uint8_t *out,
                        uint64_t out_bit0) {
    pack_lsb64(raw, b * n, n, xw, c->nw);   /* x_j at bit j; j >= n are 0 */
    for (uint64_t i = 0; i < m; ++i) {
        /* T[i][j] = s[i-j+n-1] = rs[m-1-i+j]: window of rs starting at m-1-i */
        uint64_t o = m - 1 - i, acc = 0;
        for (uint64_t w = 0; w < c->nw; ++w)
            acc ^= window64(c->rs, o + 64 * w) & xw[w];
        or_bit(out, out_bit0 + i, __builtin_popcountll(acc) & 1);
    }
}

int oracle_extract_words(const uint8_t *raw, uint64_t n_blocks, uint64_t n,
                         uint64_t m, const uint8_t *seed, uint8_t *out,
                         int n_threads) {
    if (check_args(n_blocks, n, m)) return -1;
    set_threads(n_threads);
    seed_ctx c;
    if (seed_ctx_init(&c, seed, n, m)) return -1;
    uint64_t out_bytes = (n_blocks * m + 7) / 8;
    memset(out, 0, out_bytes);
    uint64_t blk_bytes = (m + 7) / 8;
    uint8_t *scratch = (uint8_t *)calloc(n_blocks, blk_bytes);
    if (!scratch) { free(c.rs); return -1; }
    int err = 0;
#pragma omp parallel
    {
        uint64_t *xw = (uint64_t *)malloc(c.nw * sizeof(uint64_t));
        if (!xw) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t b = 0; b < (int64_t)n_blocks; ++b)
                block_words(raw, (uint64_t)b, n, m, &c, xw,
                            scratch + (uint64_t)b * blk_bytes, 0);
            free(xw);
        }
    }
    if (!err)
        for (uint64_t b = 0; b < n_blocks; ++b)
            for (uint64_t i = 0; i < m; ++i)
                or_bit(out, b * m + i, get_bit(scratch + b * blk_bytes, i));
    free(scratch);
    free(c.rs);
    return err ? -1 : 0;
}

/* Selected blocks only (for sampled checks at full size): block ids[q] of the
 * n_blocks-block stream `raw`; its m output bits are written MSB-first from
 * bit 0 of out + q*ceil(m/8).  mode 0 = scalar, 1 = words. */
int oracle_extract_blocks(const uint8_t *raw, const uint64_t *ids, uint64_t count,
                          uint64_t n, uint64_t m, const uint8_t *seed,
                          uint8_t *out, int mode, int n_threads) {
    if (check_args(count, n, m)) return -1;
    set_threads(n_threads);
    uint64_t blk_bytes = (m + 7) / 8;
    memset(out, 0, count * blk_bytes);
    seed_ctx c;
    if (seed_ctx_init(&c, seed, n, m)) return -1;
    int err = 0;
#pragma omp parallel
    {
        uint64_t *xw = (uint64_t *)malloc(c.nw * sizeof(uint64_t));
        if (!xw) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t q = 0; q < (int64_t)count; ++q) {
                if (mode == 0)
                    block_scalar(raw, ids[q], n, m, seed, out + (uint64_t)q * blk_bytes, 0);
                else
                    block_words(raw, ids[q], n, m, &c, xw, out + (uint64_t)q * blk_bytes, 0);
            }
            free(xw);
        }
    }
    free(c.rs);
    return err ? -1 : 0;
}

/* 256-bin histogram of 8-bit ADC samples (P'(x) is the
 * empirical distribution).  Plain counting loop. */
void oracle_hist256(const uint8_t *samples, uint64_t count, uint64_t *counts) {
    memset(counts, 0, 256 * sizeof(uint64_t));
    for (uint64_t q = 0; q < count; ++q) counts[samples[q]]++;
}

/* Sampled outputs (for full-size checks where a whole block is too slow):
 * y_i of block b for the `count` pairs (blocks[q], rows[q]); out[q] = 0/1.
 * Same formula (C1), 64 values of j per AND/XOR. */
int oracle_extract_rows(const uint8_t *raw, const uint64_t *blocks, const uint64_t *rows,
                        uint64_t count, uint64_t n, uint64_t m, const uint8_t *seed,
                        uint8_t *out, int n_threads) {
    if (check_args(1, n, m)) return -1;
    for (uint64_t q = 0; q < count; ++q)
        if (rows[q] >= m) return -1;
    set_threads(n_threads);
    seed_ctx c;
    if (seed_ctx_init(&c, seed, n, m)) return -1;
    int err = 0;
#pragma omp parallel
    {
        uint64_t *xw = (uint64_t *)malloc(c.nw * sizeof(uint64_t));
        uint64_t cur = UINT64_MAX;
        if (!xw) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t q = 0; q < (int64_t)count; ++q) {
                if (blocks[q] != cur) {
                    pack_lsb64(raw, blocks[q] * n, n, xw, c.nw);
                    cur = blocks[q];
                }
                uint64_t o = m - 1 - rows[q], acc = 0;
                for (uint64_t w = 0; w < c.nw; ++w) acc ^= window64(c.rs, o + 64 * w) & xw[w];
                out[q] = (uint8_t)(__builtin_popcountll(acc) & 1);
            }
            free(xw);
        }
    }
    free(c.rs);
    return err ? -1 : 0;
}

/* ---- modified Toeplitz (Sec. III.D; Listing 3 at 415-429) ----
 * k = [T_{m x (n-m)} || I_m] r with an n-bit seed a' = (a_1..a_n).  Reading
 * A24: T is "the last m rows and the first (n-m) columns" of the
 * n x n circulant A_c with first column a', A_c[i][j] =
 * a'[(i - j) mod n] (0-based), and "k_i = k'_i + r_{i+1} (n-m <= i <= n-1)"
 * adds the last m raw bits.  With t = i - (n-m) in [0, m):
 *
 *     y_t = XOR_{j < n-m} ( a'[(n-m+t-j) mod n] AND r_j )  XOR  r_{n-m+t}.
 *
 * Literal bit loop; seed buffer holds n bits MSB-first (C2), block b is raw
 * bits [b n, (b+1) n) (C3), output as C4. */
int oracle_modified_extract(const uint8_t *raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                            const uint8_t *seed, uint8_t *out, int n_threads) {
    if (check_args(n_blocks, n, m)) return -1;
    set_threads(n_threads);
    memset(out, 0, (n_blocks * m + 7) / 8);
    uint64_t blk_bytes = (m + 7) / 8;
    uint8_t *scratch = (uint8_t *)calloc(n_blocks, blk_bytes);
    if (!scratch) return -1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < (int64_t)n_blocks; ++b) {
        for (uint64_t t = 0; t < m; ++t) {
            uint64_t i = n - m + t;  /* row of A_c */
            int acc = get_bit(raw, (uint64_t)b * n + i);  /* I_m part: r_{i+1} (1-based) */
            for (uint64_t j = 0; j < n - m; ++j)
                acc ^= get_bit(seed, (i + n - j) % n) & get_bit(raw, (uint64_t)b * n + j);
            or_bit(scratch + (uint64_t)b * blk_bytes, t, acc);
        }
    }
    for (uint64_t b = 0; b < n_blocks; ++b)
        for (uint64_t t = 0; t < m; ++t)
            or_bit(out, b * m + t, get_bit(scratch + b * blk_bytes, t));
    free(scratch);
    return 0;
}

/* Modified Toeplitz, sampled outputs, 64 values of j per AND/XOR: the same
 * formula as oracle_modified_extract, y_t = XOR_{j<n-m} a'[n-m+t-j] r_j XOR
 * r_{n-m+t} (no wrap occurs for t < m, j < n-m).  Row t of T, read along j, is
 * a window of the reversed sequence of a'[1..n-1]. */
int oracle_modified_rows(const uint8_t *raw, const uint64_t *blocks, const uint64_t *rows,
                         uint64_t count, uint64_t n, uint64_t m, const uint8_t *seed,
                         uint8_t *out, int n_threads) {
    if (check_args(1, n, m)) return -1;
    for (uint64_t q = 0; q < count; ++q)
        if (rows[q] >= m) return -1;
    set_threads(n_threads);
    const uint64_t np = n - m;  /* columns of T */
    /* s[k] = a'[k+1], k < n-1 (packed MSB-first) */
    uint8_t *s = (uint8_t *)calloc((n + 7) / 8 + 1, 1);
    if (!s) return -1;
    for (uint64_t k = 0; k + 1 < n; ++k) or_bit(s, k, get_bit(seed, k + 1));
    seed_ctx c;
    if (seed_ctx_init(&c, s, np, m)) { free(s); return -1; }  /* L = np + m - 1 = n - 1 */
    int err = 0;
#pragma omp parallel
    {
        uint64_t *xw = (uint64_t *)malloc(c.nw * sizeof(uint64_t));
        uint64_t cur = UINT64_MAX;
        if (!xw) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t q = 0; q < (int64_t)count; ++q) {
                if (blocks[q] != cur) {
                    pack_lsb64(raw, blocks[q] * n, np, xw, c.nw);
                    cur = blocks[q];
                }
                /* T[t][j] = s[t - j + np - 1] = rs[m-1-t+j] */
                uint64_t o = m - 1 - rows[q], acc = 0;
                for (uint64_t w = 0; w < c.nw; ++w) acc ^= window64(c.rs, o + 64 * w) & xw[w];
                out[q] = (uint8_t)((__builtin_popcountll(acc) & 1) ^ get_bit(raw, blocks[q] * n + np + rows[q]));
            }
            free(xw);
        }
    }
    free(c.rs);
    free(s);
    return err ? -1 : 0;
}
