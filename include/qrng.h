/*
 * qrng.h -- C ABI of libqrng.so: B200 (sm_100a) Toeplitz-hashing randomness
 * extraction and min-entropy sizing, after arXiv 2011.04130 (Zhao, Ma, Zhou,
 * "Performance Optimization on Practical Quantum Random Number Generators").
 *
 * Citations: PAPER.md:<line> is the paper text, SPEC.md:<line> the derived CPU
 * spec (interfaces / error split only).  Conventions C1-C4 are fixed in
 * DESIGN.md "Readings of the paper" (from BASELINE.json and SURVEY.md Sec. 0).
 *
 *  C1  y = T x mod 2 with T[i][j] = s[i - j + n - 1], 0 <= i < m, 0 <= j < n:
 *      the m x n Toeplitz matrix displayed at PAPER.md:193 (row 1 = a_n..a_1,
 *      last row = a_{n+m-1}..a_m, a_k = s[k-1]), equivalently outputs
 *      k_n..k_{n+m-1} of the circulant product.
 *  C2  Every bit buffer is MSB-first: bit k is (buf[k >> 3] >> (7 - (k & 7))) & 1.
 *      An array of 8-bit ADC samples therefore IS the packed raw bit stream.
 *  C3  Block b is raw bits [b*n, (b+1)*n)  (block segmentation, Fig. 5).
 *  C4  Output: block b's y_i is output bit b*m + i; ceil(n_blocks*m/8) bytes;
 *      pad bits of the last byte are written as 0.
 *
 * Pointers named d_* are CUDA device pointers, h_* host pointers.  The caller
 * owns every buffer it passes; the library owns only plans and their
 * workspace.  Results never depend on the path taken, the stream or the
 * number of GPUs the caller shards blocks over (blocks are independent).
 * There is no CPU fallback: without a usable sm_100 device every entry point
 * that touches data returns QRNG_E_CUDA.
 */
#ifndef QRNG_H_
#define QRNG_H_

#include <stdint.h>
#include <cuda_runtime_api.h>

#if defined(__GNUC__)
#define QRNG_API __attribute__((visibility("default")))
#else
#define QRNG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    QRNG_OK            = 0,
    QRNG_E_INVALID     = 1, /* argument violates a precondition ("validation error") */
    QRNG_E_UNSUPPORTED = 2, /* valid for the method, outside this build's limits */
    QRNG_E_NO_OUTPUT   = 3, /* derived m <= 0: block too short for the security parameter */
    QRNG_E_CUDA        = 4, /* a CUDA call failed or no sm_100 device ("runtime error") */
    QRNG_E_NOMEM       = 5  /* device or host allocation failed */
} qrng_status;

/* Extraction path.  AUTO picks by n (crossover measured on B200). */
/* QRNG_PATH_BITS: the product on the CUDA cores, one lane per output bit
 * (parity of popcount(seed window AND reversed block), bits.cu) -- what AUTO
 * runs for small batches of a dense-GEMM shape (n m n_blocks up to 6e8 bit-MACs
 * at n <= 1024, 6e8 + 2.7e8 log2(n/1024) above: where the tensor-core kernel
 * is latency-bound); n % 32 == 0. */
typedef enum { QRNG_PATH_AUTO = 0, QRNG_PATH_GEMM = 1, QRNG_PATH_NTT = 2, QRNG_PATH_BITS = 3 } qrng_path;

/* Ideal ADC model: Gaussian N(mu, sigma^2) discretised on bins [k-1/2, k+1/2),
 * edge bins absorbing the tails (reading A10).  sigma > 0. */
typedef struct { double mu, sigma; } qrng_gauss;

typedef struct {
    uint64_t counts[256];   /* histogram of the samples (bins >= 2^bit_depth are 0)   */
    uint64_t n_samples;
    uint32_t bit_depth;     /* N */
    uint32_t reserved;
    double   mu, sigma;     /* model used: fitted (population sigma) or supplied       */
    double   h_min_hist;    /* -log2(max_x counts[x] / n_samples)   PAPER.md:59 on P'  */
    double   h_min_ideal;   /* -log2 max P(x) of the model          PAPER.md:59 on P   */
    double   stat_dist;     /* d_U(P', P) = 1/2 sum |P' - P|, U = all 2^N bins */
    double   delta_h_m;     /* log2(d_U / 2^(-N-1) + 1)       */
    double   h_min_mod;     /* max(0, h_min_ideal - delta_h_m)       */
    int64_t  m;             /* floor(n * h_min_mod / N) - s       */
} qrng_entropy_report;

typedef struct qrng_plan qrng_plan;

/* ---------------------------------------------------------------------------
 * Min-entropy and output length.
 *
 * qrng_minentropy: histogram of n_samples uint8 ADC samples on the device,
 * then the host finalises in double precision: H_min of the histogram, the
 * model P (supplied, or N(mu, sigma^2) fitted from the histogram when model is
 * NULL), d_U(P', P), Delta H_m, H_min^modify and m = floor(n*H_mod/N) - s, where
 * s = 2 log2(1/eps) is passed as an integer (reading A7).  Synchronous on
 * `stream` (one 2 KiB device-to-host copy).  rep is a host pointer and is
 * filled even when QRNG_E_NO_OUTPUT is returned.
 * Errors: E_INVALID if d_samples or rep is NULL, n_samples == 0, bit_depth
 * outside [1, 8], a sample >= 2^bit_depth, or model->sigma <= 0;
 * E_NO_OUTPUT if the derived m <= 0.
 */
QRNG_API qrng_status qrng_minentropy(const uint8_t *d_samples, uint64_t n_samples, uint32_t bit_depth,
                            const qrng_gauss *model, uint64_t n, uint32_t s,
                            qrng_entropy_report *rep, cudaStream_t stream);

/* Building blocks of qrng_minentropy for sharded samples (one process per
 * GPU): each rank ACCUMULATES its shard's counts into d_counts (uint64[256],
 * device, caller-zeroed) asynchronously, the caller all-reduces the 256
 * counts, then any rank finalises on the host.  h_counts is a host pointer.
 * d_samples may have any alignment (e.g. a shard slice samples[lo:hi]); the
 * same holds for qrng_minentropy. */
QRNG_API qrng_status qrng_hist256_async(const uint8_t *d_samples, uint64_t n_samples,
                               uint64_t *d_counts, cudaStream_t stream);
QRNG_API qrng_status qrng_entropy_from_counts(const uint64_t *h_counts, uint32_t bit_depth,
                                     const qrng_gauss *model, uint64_t n, uint32_t s,
                                     qrng_entropy_report *rep);

/* ---------------------------------------------------------------------------
 * Toeplitz extraction y = T x mod 2 of every block (C1-C4).
 *
 * d_raw_bits : n_blocks*n bits (C2, C3), ceil(n_blocks*n/8) bytes, 16-byte aligned.
 * d_seed     : L = n+m-1 seed bits a_1..a_L (C2), ceil(L/8) bytes, 16-byte aligned;
 *              bits past L are ignored.  One seed serves every block.
 * d_out      : ceil(n_blocks*m/8) bytes, 4-byte aligned, written completely (C4); no
 *              byte past ceil(n_blocks*m/8) is touched.
 * Errors: E_INVALID if a pointer is NULL or misaligned (d_raw_bits / d_seed 16 bytes,
 *         d_out 4 bytes), n == 0, m == 0,
 *         m >= n, n_blocks == 0, or d_out overlaps d_raw_bits or d_seed;
 *         E_UNSUPPORTED if n % 32 != 0 or L > 2^26;  E_CUDA / E_NOMEM on device failures.
 *         L <= 2^23 runs the tensor-core path or the NTT modulo p = 119*2^23 + 1;
 *         2^23 < L <= 2^26 (n around 2^24..2^25, past the 2-adic limit of that
 *         prime) runs the same multi-pass NTT modulo p = 7*2^26 + 1 (the prime
 *         of qrng_dist_* below).
 * The one-shot calls build a temporary plan (seed preparation included) and
 * release it stream-ordered; _async returns once the work is enqueued.
 */
QRNG_API qrng_status qrng_toeplitz_extract(const uint8_t *d_raw_bits, uint64_t n_blocks, uint64_t n,
                                  uint64_t m, const uint8_t *d_seed, uint8_t *d_out);
QRNG_API qrng_status qrng_toeplitz_extract_async(const uint8_t *d_raw_bits, uint64_t n_blocks, uint64_t n,
                                        uint64_t m, const uint8_t *d_seed, uint8_t *d_out,
                                        cudaStream_t stream);

/* End-to-end form with HOST buffers (h_raw_bits / h_seed / h_out, pinned
 * memory recommended): copies in, extracts and copies the key back on
 * `stream`, then synchronises it.  Same layouts and errors as above except
 * that host pointers need no particular alignment. */
QRNG_API qrng_status qrng_toeplitz_extract_host(const uint8_t *h_raw_bits, uint64_t n_blocks, uint64_t n,
                                       uint64_t m, const uint8_t *h_seed, uint8_t *h_out,
                                       cudaStream_t stream);

/* Streaming ingest (the paper's continuous 10 Gbit
 * stream): batches of raw bits arriving in HOST memory are
 * extracted with a reused plan in a three-stage pipeline (host->device copy,
 * extraction, device->host copy, each on its own CUDA stream) with `depth`
 * device buffer pairs, so the copy of one batch, the extraction of the
 * previous one and the key copy of the one before overlap.
 *   qrng_stream_create: plan (not owned; must outlive the stream), max_blocks
 *     per batch (device buffers are sized for it), depth >= 2 (<= 8), flags:
 *     QRNG_STREAM_HIST also accumulates the 256-bin histogram of every
 *     submitted batch's bytes (the ADC samples, C2) for on-line min-entropy
 *     monitoring (qrng_stream_counts -> qrng_entropy_from_counts).
 *   qrng_stream_submit: enqueue one batch (h_raw_bits: n_blocks * n bits,
 *     h_out: ceil(n_blocks * m / 8) bytes; pinned host memory for overlap);
 *     returns once enqueued; blocks only while all `depth` slots are busy.
 *     Both host buffers must stay valid until the batch completes
 *     (qrng_stream_synchronize, or `depth` further submits).
 *   qrng_stream_synchronize: wait for every submitted batch; returns the first
 *     error of any batch since the last call.
 *   qrng_stream_counts: synchronise and copy the accumulated counts (256 x u64).
 * Errors: E_INVALID for NULL arguments, n_blocks == 0 or > max_blocks, depth
 * outside [2, 8]; E_NOMEM / E_CUDA on device failures. */
typedef struct qrng_stream qrng_stream;
#define QRNG_STREAM_HIST 1u
QRNG_API qrng_status qrng_stream_create(const qrng_plan *plan, uint64_t max_blocks, uint32_t depth, uint32_t flags,
                                        qrng_stream **out);
QRNG_API qrng_status qrng_stream_submit(qrng_stream *stream, const uint8_t *h_raw_bits, uint64_t n_blocks,
                                        uint8_t *h_out);
QRNG_API qrng_status qrng_stream_synchronize(qrng_stream *stream);
QRNG_API qrng_status qrng_stream_counts(qrng_stream *stream, uint64_t *h_counts256);
QRNG_API void        qrng_stream_destroy(qrng_stream *stream);

/* ---------------------------------------------------------------------------
 * NEXT-4: ONE block across `world` GPUs -- a distributed
 * four-step NTT modulo p = 7*2^26 + 1 (2-adicity 26; P = 2^ceil(log2 L) <= 2^26,
 * window sums <= n < p, so the result is exact as in C1; PAPER.md:213-241 for
 * the circulant embedding, PAPER.md:273 for cutting the work of a long stream).
 * With t = N2 n1 + n2 (N2 = P / world) and k = k1 + world k2, rank r owns the
 * spectrum slice k1 = r: it forms it from the (replicated) block bits with no
 * communication, multiplies by the seed spectrum slice of its plan, transforms
 * back and twists; ONE all-to-all of N2 words per rank then gives each rank
 * all slices of its columns, and qrng_dist_finish completes the radix-world
 * inverse and ORs the window parities into the key.  One process per GPU; the
 * all-to-all (equal chunks of N2/world words) and the final OR of the ranks'
 * keys (their bits are disjoint, so a byte-wise SUM all-reduce is an OR) are
 * the caller's collectives (torch.distributed / NCCL in the Python binding).
 *
 * qrng_dist_plan_create: world in {1, 2, 4, 8}, rank < world; d_seed as for
 *   qrng_plan_create (read on `stream`, may be freed afterwards).
 * qrng_dist_exchange_words: N2, the words of every rank's exchange buffer.
 * qrng_dist_local: d_block_bits = the block's n bits (C2, ceil(n/8) bytes, any
 *   alignment); d_buf = N2 uint32 words, 16-byte aligned, written completely;
 *   words [r' N2/world, (r'+1) N2/world) go to rank r'.
 * qrng_dist_finish: d_recv = N2 words, chunk k1 received from rank k1;
 *   d_key = ceil(m/8) bytes, 4-byte aligned, ZEROED by the caller; this rank's
 *   key bits are ORed in (bit i = y_i, C4); other bits stay 0.
 * Errors: E_INVALID for NULL/misaligned pointers, bad world/rank, 0 < m < n
 *   violated; E_UNSUPPORTED for n % 32 != 0 or L > 2^26; E_CUDA / E_NOMEM. */
typedef struct qrng_dist_plan qrng_dist_plan;
QRNG_API qrng_status qrng_dist_plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t world,
                                           uint32_t rank, cudaStream_t stream, qrng_dist_plan **plan);
QRNG_API uint64_t    qrng_dist_exchange_words(const qrng_dist_plan *plan);
QRNG_API qrng_status qrng_dist_local(const qrng_dist_plan *plan, const uint8_t *d_block_bits, uint32_t *d_buf,
                                     cudaStream_t stream);
QRNG_API qrng_status qrng_dist_finish(const qrng_dist_plan *plan, const uint32_t *d_recv, uint8_t *d_key,
                                      cudaStream_t stream);
QRNG_API void        qrng_dist_plan_destroy(qrng_dist_plan *plan);

/* Plans: seed preparation (a3) once per (seed, n, m), reused over many batches.
 * qrng_plan_create reads d_seed on `stream` (the seed may be freed once that
 * stream has passed the call).  qrng_plan_extract has the layouts of
 * qrng_toeplitz_extract for n_blocks blocks of the plan's n.  A plan may be
 * used from several streams at once; destroy it only after its work is done. */
QRNG_API qrng_status qrng_plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed,
                             cudaStream_t stream, qrng_plan **plan);
QRNG_API qrng_status qrng_plan_extract(const qrng_plan *plan, const uint8_t *d_raw_bits,
                              uint64_t n_blocks, uint8_t *d_out, cudaStream_t stream);
QRNG_API void        qrng_plan_destroy(qrng_plan *plan);

/* Modified Toeplitz extraction (Sec. III.D; Listing 3 at
 * PAPER.md:415-429): k = [T_{m x (n-m)} | I_m] r with an n-bit seed a' =
 * (a_1..a_n) instead of n+m-1 bits.  Reading A24: T = the last m
 * rows and first n-m columns of the n x n circulant A_c with first column a'
 * (PAPER.md:257), plus the last m raw bits (k_i = k'_i + r_{i+1}):
 *     y_t = XOR_{j<n-m} a'[(n-m+t-j) mod n] AND r_j  XOR  r_{n-m+t},  0 <= t < m.
 * d_seed holds the n seed bits (C2); raw/out layouts, alignment and errors as
 * qrng_toeplitz_extract (n % 32 == 0, n - 1 <= 2^23).  Path: the tensor-core
 * path when n - m <= 2^16 (each block's first n - m bits repacked, zero
 * prefixed, to a multiple of 128 bits; C1 product with seed bits a_2..a_n;
 * then XOR of the last m raw bits), else the NTT path (transform length
 * 2^ceil(log2(n-1)) instead of 2^ceil(log2(n+m-1))); qrng_debug_set_path
 * forces either (GEMM with n - m > 2^16: QRNG_E_UNSUPPORTED).  The GEMM path
 * allocates an n_blocks x (n-m rounded up to 128)/8-byte workspace per call
 * (stream-ordered).  The plan works with qrng_plan_extract / qrng_plan_destroy. */
QRNG_API qrng_status qrng_plan_create_modified(uint64_t n, uint64_t m, const uint8_t *d_seed,
                                               cudaStream_t stream, qrng_plan **plan);
QRNG_API qrng_status qrng_modified_toeplitz_extract_async(const uint8_t *d_raw_bits, uint64_t n_blocks,
                                                          uint64_t n, uint64_t m, const uint8_t *d_seed,
                                                          uint8_t *d_out, cudaStream_t stream);
/* Path the plan runs (QRNG_PATH_GEMM, QRNG_PATH_NTT or a forced
 * QRNG_PATH_BITS); -1 for NULL.  An AUTO plan with QRNG_PATH_GEMM and no
 * Karatsuba tree runs small batches (see QRNG_PATH_BITS) on the CUDA cores;
 * qrng_debug_last_path tells which ran. */
QRNG_API int         qrng_plan_path(const qrng_plan *plan);
/* BENCH / TEST ONLY: product path of the most recent extraction in this
 * process (QRNG_PATH_*), -1 before the first. */
QRNG_API int         qrng_debug_last_path(void);

/* How a plan computes its product (for benchmarks and tests).
 *   path                 QRNG_PATH_GEMM, QRNG_PATH_NTT or QRNG_PATH_BITS
 *   karatsuba_depth      GEMM path: depth of the GF(2) Karatsuba decomposition
 *                        (0 = one dense product); see qrng_debug_set_karatsuba
 *   leaves               GEMM path: Toeplitz products the tensor cores run
 *   macs_per_block       GEMM path: int8 multiply-accumulates per block over all
 *                        leaves (n*m for the dense product)
 *   log2_transform       NTT path: log2 of the cyclic length P
 *   blocks_per_transform NTT path: blocks that share one transform (2: two
 *                        blocks as x1 + 2^k x2, P <= 2^15; G = 4: the packed
 *                        three-prime form, multi-pass sizes with n < 2^21)
 *   primes               NTT path: transforms per direction for each group of
 *                        blocks_per_transform blocks (3 in the packed form)
 *   x_words, y_words     Karatsuba: 32-bit workspace words per block of the
 *                        combined inputs (Q buffers) and of the leaf parities
 * Errors: E_INVALID for NULL arguments. */
typedef struct {
    int32_t path, karatsuba_depth, leaves, log2_transform;
    int32_t blocks_per_transform, primes;
    uint64_t macs_per_block;
    uint32_t x_words, y_words;
} qrng_plan_info_t;
QRNG_API qrng_status qrng_plan_info(const qrng_plan *plan, qrng_plan_info_t *info);

/* Thread-local message for the last non-OK status returned on this thread. */
QRNG_API const char *qrng_last_error(void);
/* Library version string, e.g. "qrng-b200 0.1 sm_100a". */
QRNG_API const char *qrng_version(void);

/* TEST ONLY: force the path of plans created afterwards on this process
 * (QRNG_PATH_AUTO restores the measured crossover; QRNG_PATH_BITS needs
 * n % 32 == 0 and a seed of at most ~1.6e6 bits, else E_UNSUPPORTED).  Used to
 * cross-check the independent GPU paths and to measure the crossovers; not a
 * backend switch. */
QRNG_API void        qrng_debug_set_path(int path);

/* TEST / BENCH ONLY: depth of the GF(2) Karatsuba decomposition used by GEMM-path
 * plans created afterwards on this process (DESIGN.md "Karatsuba over the GEMM
 * path"; the identity y = T x is unchanged, only the schedule of tensor-core
 * products).  -1 (default): the planner's cost model chooses; 0: one dense
 * product; d > 0: split whenever allowed down to depth d. */
QRNG_API void        qrng_debug_set_karatsuba(int max_depth);

/* TEST ONLY, host-only (no GPU): the planner's decomposition of an m x n
 * extraction with max_depth as in qrng_debug_set_karatsuba.  counts[0..3] =
 * leaves, terms, combine entries, depth.  If the buffers are large enough
 * (leaf_cap >= leaves, term_cap >= terms, comb_cap >= words + 1 + entries,
 * words = ceil(m/32)) they receive, per leaf l, leaf_rw[6l..6l+5] = {r, w,
 * out_off, first term, seed terms, input terms}; terms = the seed-term bit
 * offsets into s followed by the input-term bit offsets into the block; comb
 * = CSR row pointers (words + 1) then Y-row word offsets: output word j of a
 * block is the XOR of Y[comb[...]] where leaf l's parities occupy words
 * [out_off, out_off + ceil(r/32)) of Y, row i at bit 31 - (i % 32).
 * Leaf l computes y_l[i] = XOR_j d_l[i - j + w - 1] x_l[j] (i < r, j < w) with
 * d_l[k] = XOR over seed terms t of s[t + k] (0 past n+m-1) and
 * x_l[j] = XOR over input terms u of x[u + j].  Errors: E_UNSUPPORTED when no
 * decomposition exists (n % 128 != 0, m >= n). */
QRNG_API qrng_status qrng_debug_karatsuba_plan(uint64_t n, uint64_t m, int max_depth, uint32_t *leaf_rw,
                                               uint32_t leaf_cap, uint32_t *terms, uint32_t term_cap,
                                               uint32_t *comb, uint32_t comb_cap, uint32_t *counts);
/* TEST ONLY (no GPU needed): the one-pass Q-buffer form of the same plan
 * (karatsuba.cu qslice_kernel).  Every Q buffer (x0 ^ x1 of a Karatsuba node,
 * stored in a block's X row of info[3] 32-bit words) is cut into chunks of
 * s = n / info[0] bits; chunk e is written at 16-byte unit ent[e] >> 16 of the
 * X row as the XOR of the block's aligned s-bit slices i (x[i s, (i+1) s))
 * with bit i of ent[e] & 0xFFFF set.  info = {slices (0: the tree is not
 * covered and ent is empty), log2(s / 128), chunks, X-row words, leaves};
 * leaf_x[2l..2l+1] = {input is the X row (1) or the raw block (0), word offset
 * of leaf l's input window}, leaves in qrng_debug_karatsuba_plan's order.
 * Buffers too small (ent_cap < chunks, leaf_cap < leaves): sizes only.
 * Errors: E_INVALID for a NULL info, E_UNSUPPORTED as above. */
QRNG_API qrng_status qrng_debug_qslice_plan(uint64_t n, uint64_t m, int max_depth, uint32_t *ent, uint32_t ent_cap,
                                            uint32_t *leaf_x, uint32_t leaf_cap, uint32_t *info);

/* BENCH / TEST ONLY instrumentation.
 * qrng_debug_launch_count: number of kernels this library has launched in the
 * process so far (plan preparation and extraction kernels alike).
 * qrng_debug_kernel_timing(1) makes every subsequent main extraction-kernel
 * launch record CUDA events on its own stream, (2) also every auxiliary
 * kernel (Karatsuba Q buffers / combine, modified-Toeplitz repack / XOR;
 * read with qrng_debug_kernel_time_split), (0) none; qrng_debug_kernel_time_ms
 * synchronises those events, returns the summed device time in ms, stores the
 * number of timed launches in *launches (if not NULL) and clears the record. */
QRNG_API uint64_t    qrng_debug_launch_count(void);
/* TEST ONLY: one-CTA probe of the tcgen05 operand layouts used by the GEMM
 * path: D (128 x N int32, row-major, device) = A (128 x K uint8 0/1 or any
 * u8, row-major, device) times B^T with the Hankel B[i][k] = h[i + k]
 * (h: N+K bytes, device).  N in [16, 256] multiple of 16, K multiple of 128. */
/* BENCH ONLY: launch the register-resident radix-32 modular-butterfly
 * microbenchmark (the NTT path's butterfly code, no memory traffic) on every
 * SM; *butterflies receives the number of radix-2 butterflies it performs.
 * Time it with CUDA events on `stream` to get the achievable butterfly rate
 * (SURVEY.md 8(d) "R_bfly"). */
QRNG_API qrng_status qrng_debug_butterfly_rate(int iters, uint64_t *butterflies, cudaStream_t stream);
/* BENCH ONLY: the same microbenchmark with every radix-32 DFT followed by the
 * inter-pass twiddle multiplication (Montgomery power chains), i.e. the full
 * register-resident instruction mix of a non-final NTT pass.  *butterflies
 * counts the same 160 butterflies per iteration, so the rate is directly
 * comparable with qrng_debug_butterfly_rate. */
QRNG_API qrng_status qrng_debug_pass_rate(int iters, uint64_t *butterflies, cudaStream_t stream);
/* BENCH ONLY: operand width of the tensor-core path this library was built
 * with: 4 = tcgen05 kind::mxf4 (E2M1 0/1 operands, FP32 accumulation, the
 * default), 8 = kind::i8 (S32 accumulation, -DQRNG_GEMM_FP4=0). */
QRNG_API int         qrng_debug_gemm_operand_bits(void);
/* TEST ONLY: the same product on kind::mxf4 (E2M1 0/1 operands, both in shared
 * memory, unit UE8M0 block scales, FP32 accumulation): D (128 x N float,
 * row-major, device).  hi_first selects the nibble order of the packed
 * operands.  N in [16, 256] multiple of 16, K in [64, 1024] multiple of 64. */
QRNG_API qrng_status qrng_debug_mxf4_probe(const uint8_t *d_A, const uint8_t *d_h, float *d_D, int N, int K,
                                           int hi_first, cudaStream_t stream);
QRNG_API qrng_status qrng_debug_umma_probe(const uint8_t *d_A, const uint8_t *d_h, int32_t *d_D,
                                           int N, int K, cudaStream_t stream);
QRNG_API void        qrng_debug_kernel_timing(int enable);
/* PROFILING ONLY: the MMA-issue timeline of CTA 0 of the last packed-mode
 * tcgen05 launches (gemm_tc.cu "MMA-issue timeline"): h_out receives 6144
 * uint64 = 512 stages x {tile << 8 | stage, clock64 at the stage's start
 * (stage 0: the tile's start), after the tile lookup, after the accumulator
 * wait, after the B wait, after the A wait, after issue + commits, 0}, then
 * 256 CTAs x {globaltimer ns at entry, first A stage ready, last MMA commit,
 * exit; tile count, 0, 0, 0};
 * E_UNSUPPORTED unless the library was built with -DQRNG_GEMM_TIMELINE.
 * reset != 0 clears the record. */
QRNG_API qrng_status qrng_debug_gemm_trace(uint64_t *h_out, int reset);
/* PROFILING ONLY: back-to-back int8 MMAs on fixed operands, one CTA per SM
 * (form 0: int8 cta_group::1 A in TMEM; 1: int8 cta_group::1 A in SMEM;
 * 3: int8 stage shape, 4 K32 steps x two N tiles per elected issue + one
 * commit; 4: kind::mxf4 M128 N=n K64 back to back; 5: the E2M1 kernel's stage
 * shape, 2 K64 steps x two N tiles (N0 = n & 511 <= 224, N1 = n >> 9 or N0 if
 * 0, <= 224) per elected issue + one commit; form 2 (cta_group::2) was removed
 * with the 2-SM kernel and returns E_UNSUPPORTED); *macs = work done.
 * form + 16k (forms 0-1): a commit every k MMAs; (form 5): a second warp
 * stores k bytes per clock to other shared memory while the MMAs run
 * (shared-memory contention probe).
 * Time with CUDA events on `stream`. */
QRNG_API qrng_status qrng_debug_mma_rate(int form, int iters, int n, uint64_t *macs, cudaStream_t stream);
QRNG_API double      qrng_debug_kernel_time_ms(uint64_t *launches);
/* As qrng_debug_kernel_time_ms, also returning the auxiliary launches timed on
 * channel 1 (Karatsuba Q buffers and combine/pack kernels) in *aux_ms. */
QRNG_API double      qrng_debug_kernel_time_split(double *aux_ms, uint64_t *launches, uint64_t *aux_launches);

#ifdef __cplusplus
}
#endif
#endif /* QRNG_H_ */
