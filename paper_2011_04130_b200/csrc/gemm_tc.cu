// gemm_tc.cu -- batched Toeplitz products on the sm_100a tensor cores
// (tcgen05.mma kind::mxf4, E2M1 0/1 operands, exact FP32 accumulation in TMEM).
//
// Method: the direct O(mn) product k = T r of PAPER.md:189-197 (Listing 1 at
// PAPER.md:388-400) for ALL blocks at once.  Every block shares the seed, so
// the blocks form the columns of one matrix and the extraction is one dense
// contraction  D[b][i] = sum_j T[i][j] x_b[j]  (an exact integer <= n),
// followed by parity: y_i = D[b][i] & 1 (C1).  The same kernel runs the leaf
// products of the GF(2) Karatsuba decomposition (karatsuba.cu) as one grouped
// launch ("grouped" mode: tiles walk a leaf table, parities go to a word-aligned
// workspace).
//
// B200 design:
//  * Re-indexed as a Hankel product with K reversed, j'' = n-1-j:
//        T[i][j] = s[i + j'']            A[b][j''] = x_b[n-1-j'']
//    so a row of B is a window of the seed and a row of A a reversed window of
//    the raw block.
//  * Operands: E2M1 0/1 (0x0 / 0x2) with unit UE8M0 block scales, both in
//    shared memory (K-major, no swizzle).  Every product is exactly 0 or 1 and
//    every partial sum an integer < 2^24, so FP32 accumulation is exact
//    (pinned by tests/test_gpu_mxf4.py and the all-ones / adversarial parity
//    tests); parity = lowest mantissa bit of the sum + 2^23.
//  * B operand (2 N tiles x 224 output rows) generated on chip from the packed
//    seed: a core matrix (8 rows x 32 K) at (row group g, K group q) depends
//    only on g + 4q, so ONE linear array of core matrices (SBO 128 B, LBO
//    512 B) serves every MMA as an overlapping window -- no HBM/L2 traffic for T.
//  * A operand (M = 128 blocks): 4 transform warps load the packed block bytes
//    (prefetch ring across tiles), bit-reverse each big-endian word and write
//    the same E2M1 spread; 2 stages of 512 K.
//  * One elected lane of the MMA warp issues, per 512-K stage, 8 x K64 x 2 N
//    tiles of M128 N224 into FP32 accumulators in TMEM.  N tile 1 of the next
//    tile is deferred DEFER stages so the epilogue's drain of N tile 0 overlaps.
//  * Packed accumulators (grouped launches with every leaf K <= 2048): N tile
//    1 accumulates into N tile 0's columns with B scaled by 2^12, one column
//    set holds S0 + 2^12 S1 exactly; two sets alternate between tiles.
//  * Epilogue: 8 warps tcgen05.ld the sums, take parity, pack 32 outputs per
//    MSB-first word and store at bit b*m + i (C4) or into the leaf workspace.
//  * Persistent grid (one CTA per SM), warp-specialised, mbarrier pipelines.
//
// Measured-and-rejected variants of round 1 (int8 kind::i8 with A in TMEM, a
// 2-SM cta_group::2 kernel, one N tile with double-buffered accumulators,
// polling waits, per-stage warp reconvergence, timing-experiment switches and
// the cycle-trace build) are described in DESIGN.md 6.1 and were removed from
// the product source; git history keeps them.
#include <algorithm>
#include <cstdlib>
#include "qrng_internal.cuh"
#include "tc_ptx.cuh"

namespace qrng {
namespace gemm {
using namespace tc;

constexpr int BM = 128;          // blocks per tile (TMEM lanes)
constexpr int BN = 224;          // output rows per N tile
constexpr int NT = 2;            // N tiles per A stage (A reuse factor)
constexpr int KS = 512;          // K per A stage: KS / 64 MMAs of K64 per N tile
constexpr int KS128 = KS / 128;  // 128-bit raw chunks per A stage
#ifndef QRNG_GEMM_ASTAGES
#define QRNG_GEMM_ASTAGES 2
#endif
constexpr int A_STAGES = QRNG_GEMM_ASTAGES;  // A ring slots (2 measured faster than 3 / 4: more L1 for the loads)
constexpr int A_STAGE_BYTES = BM * KS / 2;  // A stage: BM rows x KS nibbles
constexpr int A_SBO = KS / 32 * 128;        // A stage: byte stride between 8-row core-matrix groups
constexpr int KC = 1024;         // K per B chunk
constexpr int SPC = KC / KS;     // A stages per B chunk
#ifndef QRNG_GEMM_BSLOTS
#define QRNG_GEMM_BSLOTS 3
#endif
constexpr int B_SLOTS = QRNG_GEMM_BSLOTS;  // B chunk ring slots
constexpr int CM_PER_CHUNK = KC / 8 + NT * BN / 8 - 1;  // core matrices per chunk
constexpr int CHUNK_BYTES = CM_PER_CHUNK * 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t ACC_COL0 = 0;                  // accumulators: N tile t at columns [t BN, (t+1) BN)
constexpr uint32_t SF_COL = ACC_COL0 + NT * BN;   // unit block scales (16 columns of 0x7F)
// Packed-accumulator mode (tiles with K <= 2048, i.e. Karatsuba leaves of
// w <= 2048): N tile 1's MMAs accumulate into N tile 0's FP32 accumulator with
// B scaled by 2^PACK_SHIFT, so one 224-column set holds both sums exactly
// (S0 + 2^12 S1 <= 2048 + 2^12 * 2048 < 2^24; every partial sum is an integer
// of that form): bit 0 and bit 12 of the integer are the two parities.  Two
// such sets alternate between tiles, so the drain -- half the TMEM reads --
// overlaps the next tile's MMAs.
constexpr int PACK_SHIFT = 12;
constexpr uint32_t kMaxPackedK = 2048;
constexpr uint32_t SF2_COL = SF_COL + 16;  // block scales 2^PACK_SHIFT (UE8M0 127 + 12)
constexpr int ACC_FULL = 2;
constexpr int ACC_EMPTY = 2;
static_assert(NT * BN + 32 <= (int)TMEM_COLS, "TMEM budget");
// Deferred second N tile: the epilogue drains N tile 0 and then N tile 1 (all
// 8 warps, half the columns each); the next tile's MMAs start on N tile 0 as
// soon as it is drained and catch up N tile 1 DEFER A stages later.
constexpr int DEFER = 1;
static_assert(DEFER < A_STAGES && DEFER < SPC, "deferred stages stay resident in one chunk");
// epilogue: warp group h drains columns [GC_LO(h), GC_LO(h) + GC_N(h)) of an N
// tile (128 + 96), at most NWG words each
constexpr uint32_t GC0 = 32 * ((BN / 32 + 1) / 2);
constexpr int NWG = GC0 / 32;
// Warp roles.
// Warp roles: MMA issuer, NBG B generators (3; 4 for grouped launches with
// many leaves, whose B generators switch leaf seeds often: measured config 3
// 206 -> 212 Gbit/s, config 2 716 -> 700 with 4), 4 A transformers, 8
// epilogue warps (they use warp % 4 as their TMEM lane quadrant, so any
// offset works).  NBG is a template parameter of the kernel.
constexpr int W_MMA = 0, W_BGEN0 = 1, N_XFORM = 4, N_EPI = 8;
__host__ __device__ constexpr int nthreads_for(int nbg) { return (1 + nbg + N_XFORM + N_EPI) * 32; }
#ifndef QRNG_GEMM_PF
#define QRNG_GEMM_PF 2
#endif
constexpr int PF = QRNG_GEMM_PF;  // A-transform prefetch depth (stages)
constexpr int MAX_N = 1 << 16;
static_assert(kTileRows == NT * BN, "leaf tables assume NT*BN rows per work tile");

// ---- optional MMA-issue timeline (profiling builds: -DQRNG_GEMM_TIMELINE) ----------
// The elected MMA lane of CTA 0 records, per stage, clock64 before its waits,
// after its waits and after its issue + commits (tag = tile << 8 | stage);
// read back with qrng_debug_gemm_trace.  Row 512 + c holds, for CTA c < 256,
// globaltimer ns at kernel entry, when the first A stage is ready, after the
// last MMA commit and at exit, then its tile count and SM id (packed mode).
// Compiled out of the product build.
#ifdef QRNG_GEMM_TIMELINE
constexpr int kTimelineStages = 512, kTimelineCtaRows = 256;
__device__ unsigned long long g_timeline[8 * (kTimelineStages + kTimelineCtaRows)];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TL_CTA(k)                                                                               \
    if (blockIdx.x < kTimelineCtaRows) g_timeline[8 * kTimelineStages + 8 * blockIdx.x + (k)] = gtimer()
#define TL_T(v) const unsigned long long v = clock64()
#define TL_REC(idx, tag, a, b, c, d, e, f)                                                     \
    if (blockIdx.x == 0 && (idx) < kTimelineStages) {                                         \
        unsigned long long *g_ = g_timeline + 8 * (idx);                                      \
        g_[0] = (tag); g_[1] = (a); g_[2] = (b); g_[3] = (c); g_[4] = (d); g_[5] = (e); g_[6] = (f); \
    }
#else
#define TL_CTA(k)
#define TL_T(v)
#define TL_REC(idx, tag, a, b, c, d, e, f)
#endif

// ---- the extraction kernel -----------------------------------------------------
struct Args {
    const uint32_t *raw;       // packed raw stream (MSB-first bytes) as words
    uint64_t n_blocks;
    uint32_t n, m;
    uint32_t kst;              // K stages per tile = ceil(n / KS)
    uint32_t k128;             // 128-bit raw chunks per block = n / 128
    uint32_t nchunks;          // B chunks per tile = ceil(kst / SPC)
    uint32_t n_mtiles, n_npairs;  // M tiles; pairs of N tiles (NT = 2 per work tile)
    uint32_t prows;            // plain mode: output rows per N pair (448, fewer for small batches)
    const uint32_t *seed_words;  // logical big-endian seed words, zero padded
    uint32_t seed_words_n;
    const uint8_t *seed_bytes;   // plain mode, one-shot calls: the caller's MSB-first seed (seed_words unused)
    uint64_t seed_bits;          // L = n + m - 1 (seed_bytes mode)
    OutStream out;
    // grouped (Karatsuba leaf) mode only: tiles walk the leaf table, operands
    // come from per-leaf inputs and parities go to a word-aligned workspace
    const Leaf *leaves;
    uint32_t n_leaves;
    const uint32_t *xws;       // workspace of XOR-combined leaf inputs
    uint32_t x_stride;         // words per block in xws
    uint32_t *yws;             // leaf parity workspace
    uint32_t y_stride;         // words per block in yws
    uint64_t mt_magic;         // ceil(2^64 / n_mtiles) (0 when n_mtiles == 1): q = umul64hi(x, magic)
    uint32_t n_runs, run_q, run_rem;  // tile runs (work distribution, set at launch): count, ntiles / n_runs, ntiles % n_runs
};

// Leaf table row as the kernel reads it (grouped mode, staged in shared memory
// at kernel start: the per-tile lookup is on the MMA issuer's critical path).
struct TLeaf {
    uint32_t tile_base, tile_end;  // work tiles [tile_base, tile_end) of this leaf
    uint32_t prows, k128, r;       // rows per N pair, 128-bit input chunks (w / 128), output rows
    uint32_t seed_off;             // leaf seed (word offset in the plan's seed buffer)
    uint32_t x_off_src;            // input word offset | (1 << 31) when it is in the X workspace
    uint32_t out_off;              // word offset of the leaf parities in a block's Y row
};
static_assert(sizeof(TLeaf) == 32, "TLeaf is 8 words");

__device__ __forceinline__ uint32_t div_mtiles(const Args &a, uint32_t x) {
    return a.mt_magic ? (uint32_t)__umul64hi((uint64_t)x, a.mt_magic) : x;
}

// Geometry of one work tile (M tile of BM blocks x up to NT*BN output rows).
struct Tile {
    uint32_t mt, n0;           // M tile; first output row of the N pair
    uint32_t kst, nchunks;     // K stages of KS (the last one zero-padded), B chunks of KC
    uint32_t k128;             // 128-bit input chunks per block row
    uint32_t r;                // valid output rows of the product this tile belongs to
    uint32_t ntc, nlast;       // N tiles used (1..NT); N of the last one (multiple of 16)
    const uint32_t *seed;      // seed words of the product (smem in plain mode)
    const uint32_t *xb;        // block-0 input words of the product
    uint32_t xs;               // words per block of the input
    uint32_t out_off;          // grouped: word offset of the leaf in a block's yws row
};

__device__ __forceinline__ void tile_rows(Tile &ti, uint32_t cap = NT * BN) {
    const uint32_t left = ti.r > ti.n0 ? min(cap, ti.r - ti.n0) : 16u;
    ti.ntc = (left + BN - 1) / BN;
    const uint32_t lastrows = left - (ti.ntc - 1) * BN;
    ti.nlast = (lastrows + 15) & ~15u;
}

// Plain mode: one product (the whole extraction), tiles (N pair, M tile).
// Grouped mode: tiles of leaf l are [npair_base*n_mtiles, (npair_base+npairs)*n_mtiles);
// `cur` is a per-role cursor into the leaf table (tiles only increase).
template <bool GROUPED>
__device__ __forceinline__ Tile tile_info(const Args &a, const uint32_t *seed_s, uint32_t t, uint32_t &cur) {
    Tile ti;
    if (!GROUPED) {
        ti.mt = t % a.n_mtiles;
        ti.n0 = (t / a.n_mtiles) * a.prows;
        ti.kst = a.kst;
        ti.k128 = a.k128;
        ti.nchunks = a.nchunks;
        ti.r = a.m;
        ti.seed = seed_s;
        ti.xb = a.raw;
        ti.xs = a.n >> 5;
        ti.out_off = 0;
        tile_rows(ti, a.prows);
        return ti;
    } else {
        const TLeaf *lv = reinterpret_cast<const TLeaf *>(seed_s);  // shared-memory leaf table
        while (cur + 1 < a.n_leaves && t >= lv[cur].tile_end) ++cur;
        const TLeaf L = lv[cur];
        const uint32_t tl = t - L.tile_base, q = div_mtiles(a, tl);
        ti.mt = tl - q * a.n_mtiles;
        ti.n0 = q * L.prows;
        ti.k128 = L.k128;
        ti.kst = (L.k128 + KS128 - 1) / KS128;
        ti.nchunks = (ti.kst + SPC - 1) / SPC;
        ti.r = L.r;
        ti.seed = a.seed_words + L.seed_off;
        const uint32_t xo = L.x_off_src & 0x7FFFFFFFu;
        if (!(L.x_off_src >> 31)) { ti.xb = a.raw + xo; ti.xs = a.n >> 5; }
        else { ti.xb = a.xws + xo; ti.xs = a.x_stride; }
        ti.out_off = L.out_off;
        tile_rows(ti, L.prows);
        return ti;
    }
    tile_rows(ti);
    return ti;
}

// ---- work distribution ----------------------------------------------------------
// The tiles [0, ntiles) are cut into a.n_runs contiguous runs of equal
// length (+-1); CTA c takes runs c, c + G, c + 2G, ... (G = gridDim.x).  Runs of
// consecutive tiles share their N pair (M tile varies fastest), so one B
// operand set serves the whole run (see `same_b`); a few runs per CTA keep the
// CTAs working on nearby tiles (A-operand reuse in L2) and the per-CTA tile
// counts within a few tiles of each other.  n_runs == ntiles gives the
// plain strided order t = c, c + G, ...
constexpr uint32_t kNoTile = 0xFFFFFFFFu;
struct TCur {
    uint32_t t, hi, i;  // current tile, end of the current run, run index
};
// first tile of run i: runs [0, run_rem) have run_q + 1 tiles, the rest run_q
// (host-computed quotient / remainder: no division on the device)
__device__ __forceinline__ uint32_t run_lo(const Args &a, uint32_t i) { return i * a.run_q + min(i, a.run_rem); }
__device__ __forceinline__ void tcur_skip(const Args &a, TCur &c) {
    while (c.t >= c.hi) {  // past the run's end (or an empty run): the CTA's next run
        c.i += gridDim.x;
        if (c.i >= a.n_runs) { c.t = kNoTile; return; }
        c.t = run_lo(a, c.i);
        c.hi = run_lo(a, c.i + 1);
    }
}
__device__ __forceinline__ TCur tcur_first(const Args &a) {
    TCur c;
    c.i = blockIdx.x;
    if (c.i >= a.n_runs) { c.t = kNoTile; c.hi = 0; return c; }
    c.t = run_lo(a, c.i);
    c.hi = run_lo(a, c.i + 1);
    tcur_skip(a, c);
    return c;
}
__device__ __forceinline__ void tcur_next(const Args &a, TCur &c) {
    ++c.t;
    tcur_skip(a, c);
}

// Two consecutive tiles of a CTA whose B operands are identical (same seed
// words, N pair, K extent and row count): the second reuses the first one's B
// chunks in shared memory instead of regenerating them.  Only when the tile's
// chunks fit in B_SLOTS - 1 slots, so the next set's first chunk can be built
// while the current set is still in use.
__device__ __forceinline__ bool same_b(const Tile &x, const Tile &y) {
    return x.nchunks <= (uint32_t)(B_SLOTS - 1) && x.seed == y.seed && x.n0 == y.n0 && x.nchunks == y.nchunks &&
           x.k128 == y.k128 && x.r == y.r;
}

// Store the masked parity words of one epilogue thread (its block b, rows
// [n0, n0 + nvalid)): grouped mode into the leaf workspace (word aligned),
// plain mode into the output stream at bit b*m + n0 (C4).
template <bool GROUPED>
__device__ __forceinline__ void store_words(const Args &a, const Tile &ti, uint64_t b, uint32_t n0, uint32_t nvalid,
                                            uint32_t (&words)[NWG]) {
#pragma unroll
    for (int c = 0; c < NWG; ++c) {
        const int vb = (int)nvalid - 32 * c;
        if (vb <= 0) words[c] = 0;
        else if (vb < 32) words[c] &= ~(0xFFFFFFFFu >> vb);
    }
    if (GROUPED) {
        uint32_t *dst = a.yws + b * a.y_stride + ti.out_off + n0 / 32;
#pragma unroll
        for (int c = 0; c < NWG; ++c)
            if ((uint32_t)(32 * c) < nvalid) dst[c] = words[c];
        return;
    }
    const uint64_t G_lo = b * a.m + n0, G_hi = G_lo + nvalid;
    const uint32_t off = (uint32_t)(G_lo & 31);
    const uint64_t W0 = G_lo >> 5;
    uint32_t prev = 0;
#pragma unroll
    for (int c = 0; c <= NWG; ++c) {
        const uint32_t cw = (c < NWG) ? words[c] : 0u;
        const uint32_t ow = off ? ((prev << (32 - off)) | (cw >> off)) : cw;
        prev = cw;
        const uint64_t W = W0 + c;
        if (W * 32 >= G_hi) break;
        const bool excl = (W * 32 >= G_lo) && (W * 32 + 32 <= G_hi);
        emit_word(a.out, W, ow, excl);
    }
}

template <bool GROUPED, bool PACKED = false, int NBG = 3>
__global__ void __launch_bounds__(nthreads_for(NBG), 1) toeplitz_gemm_kernel(Args a) {
    constexpr int N_BGEN = NBG, W_XFORM0 = W_BGEN0 + N_BGEN, W_EPI0 = W_XFORM0 + N_XFORM;
    constexpr int NTHREADS = nthreads_for(NBG);
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *chunks = smem;
    uint8_t *a_ring = smem + B_SLOTS * CHUNK_BYTES;  // A stages (core-matrix layout, LBO 128, SBO A_SBO)
    uint32_t *seed_s = reinterpret_cast<uint32_t *>(a_ring + A_STAGES * A_STAGE_BYTES);
    // plain mode: the seed words; grouped mode: the leaf table (leaf seeds stay in global / L1)
    const uint32_t seed_stage = GROUPED ? a.n_leaves * 8u : a.seed_words_n;
    uint64_t *bars = reinterpret_cast<uint64_t *>(seed_s + ((seed_stage + 3) & ~3u));
    uint64_t *a_full = bars, *a_empty = bars + A_STAGES, *b_full = bars + 2 * A_STAGES;
    uint64_t *b_empty = b_full + B_SLOTS, *acc_full = b_empty + B_SLOTS, *acc_empty = acc_full + ACC_FULL;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + ACC_EMPTY);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TL_CTA(0);
    if (GROUPED) {
        for (uint32_t i = threadIdx.x; i < a.n_leaves; i += NTHREADS) {
            const Leaf &L = a.leaves[i];
            TLeaf o;
            o.tile_base = L.npair_base * a.n_mtiles;
            o.tile_end = (L.npair_base + L.npairs) * a.n_mtiles;
            o.prows = L.pair_rows;
            o.k128 = L.w / 128;
            o.r = L.r;
            o.seed_off = L.seed_off;
            o.x_off_src = L.x_off | (L.x_src ? 0x80000000u : 0u);
            o.out_off = L.out_off;
            reinterpret_cast<TLeaf *>(seed_s)[i] = o;
        }
    } else {
        if (a.seed_bytes) {
            // one-shot calls: the seed words are formed here from the caller's
            // bytes (word w = seed bits [32w, 32w + 32), big-endian, zero at and
            // past L) -- no plan buffer, no separate seed kernel
            const uint64_t nbytes = (a.seed_bits + 7) / 8;
            for (uint32_t i = threadIdx.x; i < seed_stage; i += NTHREADS) {
                uint32_t v = 0;
                const uint64_t b0 = 4ull * i;
                if (b0 + 4 <= nbytes) {
                    v = __byte_perm(__ldg(reinterpret_cast<const uint32_t *>(a.seed_bytes) + i), 0, 0x0123);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) v = (v << 8) | (b0 + k < nbytes ? (uint32_t)a.seed_bytes[b0 + k] : 0u);
                }
                const uint64_t lo = 32ull * i;
                if (lo + 32 > a.seed_bits) v &= a.seed_bits > lo ? (0xFFFFFFFFu << (32 - (uint32_t)(a.seed_bits - lo))) : 0u;
                seed_s[i] = v;
            }
        } else {
            for (uint32_t i = threadIdx.x; i < seed_stage; i += NTHREADS) seed_s[i] = a.seed_words[i];
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < A_STAGES; ++s) { mbar_init(&a_full[s], N_XFORM); mbar_init(&a_empty[s], 1); }
        for (int s = 0; s < B_SLOTS; ++s) { mbar_init(&b_full[s], N_BGEN); mbar_init(&b_empty[s], 1); }
        for (int s = 0; s < ACC_FULL; ++s) mbar_init(&acc_full[s], 1);
        for (int s = 0; s < ACC_EMPTY; ++s) mbar_init(&acc_empty[s], N_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_MMA) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // block scales: UE8M0 127 = 2^0 (SF_COL) and 127 + 12 = 2^12 (SF2_COL) in every byte
    if (warp >= W_EPI0 && warp < W_EPI0 + 4) {
        uint32_t v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = 0x7F7F7F7Fu;
        tmem_st16(tmem + (((uint32_t)(warp & 3) * 32) << 16) + SF_COL, v);
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = (127u + PACK_SHIFT) * 0x01010101u;
        tmem_st16(tmem + (((uint32_t)(warp & 3) * 32) << 16) + SF2_COL, v);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t cur = 0;                                 // leaf cursor of this role
    if (GROUPED) {
        pdl_release();  // the combine kernel may be scheduled as CTAs finish
        pdl_wait();     // the Q buffers (previous kernel) are complete
    }

    if (PACKED && warp == W_MMA) {
        // packed mode: both N tiles into one of two alternating column sets; one
        // elected lane runs the whole loop (no per-stage warp reconvergence)
        if (elect_one()) {
            uint32_t as = 0, aph = 0, it = 0;
            uint32_t gb = 0;        // B chunks of the sets before the current one
            bool first_set = true;  // the current tile starts a B set (its chunks must be waited for)
#ifdef QRNG_GEMM_TIMELINE
            uint32_t tl_i = 0;
#endif
            // the next tile's geometry is looked up while the current tile's first
            // stage is in the tensor pipe (measured: the lookup cost ~400 cycles of
            // pipe idle per tile when done at the tile boundary)
            TCur c = tcur_first(a), nc = c;
            Tile nti{};
            if (c.t != kNoTile) nti = tile_info<GROUPED>(a, seed_s, c.t, cur);
            for (; c.t != kNoTile; c = nc, ++it) {
                TL_T(tl_tile);
                const Tile ti = nti;
                bool last_set = true;  // the next tile needs other B chunks: release ours
                const uint32_t r = it & 1, acc = tmem + ACC_COL0 + r * BN;
                const uint32_t idesc0 = idesc_mxf4(BM, ti.ntc == 1 ? (int)ti.nlast : BN), idesc1 = idesc_mxf4(BM, (int)ti.nlast);
                TL_T(tl_info);
                mbar_wait(&acc_empty[r], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                TL_T(tl_acc);
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    TL_T(tl0);
                    const uint32_t kin = ks % SPC, bc = gb + ks / SPC, bs = bc % B_SLOTS, bph = (bc / B_SLOTS) & 1;
                    if (kin == 0 && first_set) { mbar_wait(&b_full[bs], bph); tc_fence_after(); }
                    TL_T(tlb);
                    mbar_wait(&a_full[as], aph);
                    tc_fence_after();
                    TL_T(tl1);
#ifdef QRNG_GEMM_TIMELINE
                    if (it == 0 && ks == 0) TL_CTA(1);
#endif
                    // descriptors of the stage's first MMA; the others differ only in the
                    // start-address field (addr >> 4, no carry: shared memory < 256 KB)
                    const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + as * A_STAGE_BYTES), 128, A_SBO);
                    const uint64_t bdesc0 =
                        desc_kmajor(smem_u32(chunks + bs * CHUNK_BYTES) + (kin * KS / 8) * 128, 512, 128);
#pragma unroll
                    for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                        const uint64_t adesc = adesc0 + kk * 16;      // + kk * 256 bytes
                        const uint64_t bdesc = bdesc0 + kk * 64;      // + kk * 8 core matrices
                        mma_mxf4_ss(acc, adesc, bdesc, idesc0, tmem + SF_COL, tmem + SF_COL + 8, (ks | kk) != 0);
                        if (ti.ntc == 2)  // N tile 1, B scaled by 2^PACK_SHIFT, same columns
                            mma_mxf4_ss(acc, adesc, bdesc + BN, idesc1, tmem + SF_COL, tmem + SF2_COL, true);  // + BN/8 cm
                    }
                    mma_commit(&a_empty[as]);
                    if (ks == 0) {
                        nc = c;
                        tcur_next(a, nc);
                        if (nc.t != kNoTile) {
                            nti = tile_info<GROUPED>(a, seed_s, nc.t, cur);
                            last_set = !same_b(ti, nti);
                        }
                    }
                    if (last_set && (kin == SPC - 1 || ks == ti.kst - 1)) mma_commit(&b_empty[bs]);
                    TL_T(tl2);
                    TL_REC(tl_i, ((unsigned long long)it << 8) | ks, ks ? tl0 : tl_tile, ks ? tl0 : tl_info,
                           ks ? tl0 : tl_acc, tlb, tl1, tl2);
#ifdef QRNG_GEMM_TIMELINE
                    ++tl_i;
#endif
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                }
                if (last_set) gb += ti.nchunks;
                first_set = last_set;
                mma_commit(&acc_full[r]);
            }
            TL_CTA(2);
#ifdef QRNG_GEMM_TIMELINE
            if (blockIdx.x < kTimelineCtaRows) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                g_timeline[8 * kTimelineStages + 8 * blockIdx.x + 4] = it;
                g_timeline[8 * kTimelineStages + 8 * blockIdx.x + 5] = smid;
            }
#endif
        }
        __syncwarp();
    } else if (!GROUPED && warp == W_MMA) {
        // plain launches: one column set per N tile; N tile 1 of each tile is
        // deferred DEFER stages behind N tile 0; one elected lane runs the loop,
        // with the packed loop's one-tile lookahead and B reuse (consecutive
        // strided tiles often share their N pair: dense n = 1024 2,547 vs 2,447
        // Gbit/s with the grouped loop below)
        if (elect_one()) {
            uint32_t as = 0, aph = 0, it = 0;
            uint32_t gb = 0;        // B chunks of the sets before the current one (as above)
            bool first_set = true;
            TCur c = tcur_first(a), nc = c;
            Tile nti{};  // next tile's geometry, looked up during the current tile (as above)
            if (c.t != kNoTile) nti = tile_info<GROUPED>(a, seed_s, c.t, cur);
            for (; c.t != kNoTile; c = nc, ++it) {
                const Tile ti = nti;
                bool last_set = true;
                const uint32_t idesc_full = idesc_mxf4(BM, BN);
                const uint32_t idesc_last = idesc_mxf4(BM, (int)ti.nlast);
                const uint32_t ph = (it & 1) ^ 1;
                mbar_wait(&acc_empty[0], ph);
                const bool defer = ti.ntc == 2 && ti.kst > (uint32_t)DEFER;
                if (!defer) mbar_wait(&acc_empty[1], ph);
                tc_fence_after();
                bool nt1_on = !defer;
                uint32_t dslot[DEFER];
                uint32_t cb0 = 0;
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC, bc = gb + ks / SPC, bs = bc % B_SLOTS, bph = (bc / B_SLOTS) & 1;
                    if (kin == 0 && first_set) { mbar_wait(&b_full[bs], bph); tc_fence_after(); }
                    mbar_wait(&a_full[as], aph);
                    tc_fence_after();
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                    if (ks == 0) cb0 = cbase;
                    if (!nt1_on && ks == (uint32_t)DEFER) {
                        // N tile 1 drained: its MMAs for the held stages, then release them
                        mbar_wait(&acc_empty[1], ph);
                        tc_fence_after();
#pragma unroll
                        for (int d = 0; d < DEFER; ++d) {
                            const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + dslot[d] * A_STAGE_BYTES), 128, A_SBO);
                            const uint64_t bdesc0 = desc_kmajor(cb0 + (d * KS / 8 + BN / 8) * 128, 512, 128);
#pragma unroll
                            for (uint32_t kk = 0; kk < KS / 64; ++kk)
                                mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc0 + kk * 16, bdesc0 + kk * 64, idesc_last,
                                            tmem + SF_COL, tmem + SF_COL + 8, (d | kk) != 0);
                            mma_commit(&a_empty[dslot[d]]);
                        }
                        nt1_on = true;
                    }
                    // first MMA's descriptors; the others add to the start-address field
                    const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + as * A_STAGE_BYTES), 128, A_SBO);
                    const uint64_t bdesc0 = desc_kmajor(cbase + (kin * KS / 8) * 128, 512, 128);
#pragma unroll
                    for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                        const uint64_t adesc = adesc0 + kk * 16, bdesc = bdesc0 + kk * 64;
                        mma_mxf4_ss(tmem + ACC_COL0, adesc, bdesc, ti.ntc == 1 ? idesc_last : idesc_full,
                                    tmem + SF_COL, tmem + SF_COL + 8, (ks | kk) != 0);
                        if (nt1_on && ti.ntc == 2)
                            mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc, bdesc + BN, idesc_last, tmem + SF_COL,
                                        tmem + SF_COL + 8, (ks | kk) != 0);
                    }
                    if (nt1_on) mma_commit(&a_empty[as]);
                    if (ks == 0) {
                        nc = c;
                        tcur_next(a, nc);
                        if (nc.t != kNoTile) {
                            nti = tile_info<GROUPED>(a, seed_s, nc.t, cur);
                            last_set = !same_b(ti, nti);
                        }
                    }
                    if (last_set && (kin == SPC - 1 || ks == ti.kst - 1)) mma_commit(&b_empty[bs]);
                    if (!nt1_on) dslot[ks] = as;
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                }
                if (last_set) gb += ti.nchunks;
                first_set = last_set;
                mma_commit(&acc_full[0]);
            }
        }
        __syncwarp();
    } else if (warp == W_MMA) {
        // grouped launches with K > 2048 leaves: one column set per N tile; N
        // tile 1 of each tile is deferred DEFER stages behind N tile 0; one
        // elected lane runs the loop; no lookahead and no B reuse (four chunks
        // per tile: nothing to reuse; measured 2^18 leaves 68.1 -> 70.0 Gbit/s
        // against the plain launches' loop)
        if (elect_one()) {
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (TCur c = tcur_first(a); c.t != kNoTile; tcur_next(a, c), ++it) {
                const Tile ti = tile_info<GROUPED>(a, seed_s, c.t, cur);
                const uint32_t idesc_full = idesc_mxf4(BM, BN);
                const uint32_t idesc_last = idesc_mxf4(BM, (int)ti.nlast);
                const uint32_t ph = (it & 1) ^ 1;
                mbar_wait(&acc_empty[0], ph);
                const bool defer = ti.ntc == 2 && ti.kst > (uint32_t)DEFER;
                if (!defer) mbar_wait(&acc_empty[1], ph);
                tc_fence_after();
                bool nt1_on = !defer;
                uint32_t dslot[DEFER];
                uint32_t cb0 = 0;
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC;
                    if (kin == 0) { mbar_wait(&b_full[bs], bph); tc_fence_after(); }
                    mbar_wait(&a_full[as], aph);
                    tc_fence_after();
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                    if (ks == 0) cb0 = cbase;
                    if (!nt1_on && ks == (uint32_t)DEFER) {
                        // N tile 1 drained: its MMAs for the held stages, then release them
                        mbar_wait(&acc_empty[1], ph);
                        tc_fence_after();
#pragma unroll
                        for (int d = 0; d < DEFER; ++d) {
                            const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + dslot[d] * A_STAGE_BYTES), 128, A_SBO);
                            const uint64_t bdesc0 = desc_kmajor(cb0 + (d * KS / 8 + BN / 8) * 128, 512, 128);
#pragma unroll
                            for (uint32_t kk = 0; kk < KS / 64; ++kk)
                                mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc0 + kk * 16, bdesc0 + kk * 64, idesc_last,
                                            tmem + SF_COL, tmem + SF_COL + 8, (d | kk) != 0);
                            mma_commit(&a_empty[dslot[d]]);
                        }
                        nt1_on = true;
                    }
                    // first MMA's descriptors; the others add to the start-address field
                    const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + as * A_STAGE_BYTES), 128, A_SBO);
                    const uint64_t bdesc0 = desc_kmajor(cbase + (kin * KS / 8) * 128, 512, 128);
#pragma unroll
                    for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                        const uint64_t adesc = adesc0 + kk * 16, bdesc = bdesc0 + kk * 64;
                        mma_mxf4_ss(tmem + ACC_COL0, adesc, bdesc, ti.ntc == 1 ? idesc_last : idesc_full,
                                    tmem + SF_COL, tmem + SF_COL + 8, (ks | kk) != 0);
                        if (nt1_on && ti.ntc == 2)
                            mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc, bdesc + BN, idesc_last, tmem + SF_COL,
                                        tmem + SF_COL + 8, (ks | kk) != 0);
                    }
                    if (nt1_on) mma_commit(&a_empty[as]);
                    if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                    if (!nt1_on) dslot[ks] = as;
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                    if (kin == SPC - 1 || ks == ti.kst - 1) {
                        if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                    }
                }
                mma_commit(&acc_full[0]);
            }
        }
        __syncwarp();
    } else if (warp >= W_BGEN0 && warp < W_BGEN0 + N_BGEN) {
        // B generators: core matrix tau of chunk (n0, k0): row r' holds seed bits
        // s[n0 + k0 + 8 tau + r' + c], c = 0..31, as E2M1 0/1.
        const int tb = (warp - W_BGEN0) * 32 + lane;
        uint32_t gb = 0;  // B chunks generated so far (ring position)
        Tile pti{};
        bool have_prev = false;
        for (TCur c = tcur_first(a); c.t != kNoTile; tcur_next(a, c)) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, c.t, cur);
            const bool reuse = (PACKED || !GROUPED) && have_prev && same_b(pti, ti);  // (as the MMA loops)
            pti = ti;
            have_prev = true;
            if (reuse) continue;  // the MMA issuer reads the previous tile's chunks again
            // core-matrix rows the MMAs of this tile read (K chunk + the N rows in use)
            const int ncm = KC / 8 + (int)(((ti.ntc - 1) * BN + ti.nlast) / 8) - 1;
            for (uint32_t ch = 0; ch < ti.nchunks; ++ch, ++gb) {
                const uint32_t base = ti.n0 + ch * KC, bs = gb % B_SLOTS, bph = (gb / B_SLOTS) & 1;
                mbar_wait(&b_empty[bs], bph ^ 1);
                uint8_t *cb = chunks + bs * CHUNK_BYTES;
                for (int r = tb; r < ncm * 8; r += N_BGEN * 32) {
                    const uint32_t p = base + 8 * (r >> 3) + (r & 7);
                    uint32_t w0, w1;
                    if (GROUPED) { w0 = __ldg(ti.seed + (p >> 5)); w1 = __ldg(ti.seed + (p >> 5) + 1); }
                    else { w0 = ti.seed[p >> 5]; w1 = ti.seed[(p >> 5) + 1]; }
                    const uint32_t v = __funnelshift_l(w1, w0, p & 31);
                    *reinterpret_cast<uint4 *>(cb + (r >> 3) * 128 + (r & 7) * 16) = e2m1_row(v);  // seed bits p .. p+31
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&b_full[bs]);
            }
        }
    } else if (warp >= W_XFORM0 && warp < W_XFORM0 + N_XFORM) {
        // A transform: row = block, KS K per stage.  Stages are numbered
        // g = 0, 1, 2, ... over this CTA's (tile, K stage) pairs.  The prefetch
        // ring of input chunks runs continuously across tiles.
        const uint32_t row = (uint32_t)(warp - W_XFORM0) * 32 + lane;
        uint32_t lcur = 0;                      // leaf cursor of the load side
        TCur lc = tcur_first(a);  // load cursor (tile, K stage)
        uint32_t lks = 0;
        Tile lti{};
        if (lc.t != kNoTile) lti = tile_info<GROUPED>(a, seed_s, lc.t, lcur);
        auto step1 = [&]() {
            if (lc.t == kNoTile) return;
            if (++lks == lti.kst) {
                lks = 0;
                tcur_next(a, lc);
                if (lc.t != kNoTile) lti = tile_info<GROUPED>(a, seed_s, lc.t, lcur);
            }
        };
        // Branch-free prefetch: always load from a valid address (clamped block,
        // stale tile past the end) and keep a validity flag, so every ring slot
        // stays in its own registers and the load latency is really hidden.
        // K is reversed: stage lks, quarter hf (128 K each) reads 128-bit chunk
        // k128 - 1 - KS128 lks - hf of the block row (the tail of the last stage
        // may lie before the row start -> zeros)
        auto load = [&](bool &v, uint32_t hf) -> uint4 {
            const uint64_t b = (uint64_t)lti.mt * BM + row;
            const int32_t ci = (int32_t)lti.k128 - 1 - (int32_t)(KS128 * lks + hf);
            v = lc.t != kNoTile && b < a.n_blocks && ci >= 0;
            const uint64_t bc = b < a.n_blocks ? b : a.n_blocks - 1;
            return __ldg(reinterpret_cast<const uint4 *>(lti.xb + bc * lti.xs) + (ci >= 0 ? ci : 0));
        };
        uint4 pf[PF][KS128];
        bool ok[PF], vd[PF][KS128];
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            ok[j] = lc.t != kNoTile;
#pragma unroll
            for (int hf = 0; hf < KS128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
            step1();
        }
        uint32_t g = 0;
        bool more = true;
        while (more) {
#pragma unroll
            for (int j = 0; j < PF; ++j) {
                if (more && !ok[j]) more = false;
                if (more) {
                    uint4 cur4[KS128];
#pragma unroll
                    for (int hf = 0; hf < KS128; ++hf) cur4[hf] = vd[j][hf] ? pf[j][hf] : make_uint4(0, 0, 0, 0);
                    ok[j] = lc.t != kNoTile;
#pragma unroll
                    for (int hf = 0; hf < KS128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
                    step1();
                    const uint32_t as = g % A_STAGES, aph = (g / A_STAGES) & 1;
                    mbar_wait(&a_empty[as], aph ^ 1);
                    tc_fence_after();
                    // K group (32 elements, K reversed) = memory word 3 - q4, element c =
                    // bit c of its big-endian value: bit-reverse so that bit b holds
                    // element 31 - b as in the B rows, then the same nibble spread
                    uint8_t *arow = a_ring + as * A_STAGE_BYTES + (row >> 3) * A_SBO + (row & 7) * 16;
#pragma unroll
                    for (int hf = 0; hf < KS128; ++hf) {
                        const uint32_t M4[4] = {cur4[hf].x, cur4[hf].y, cur4[hf].z, cur4[hf].w};
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            *reinterpret_cast<uint4 *>(arow + (hf * 4 + q4) * 128) =
                                e2m1_row(__brev(__byte_perm(M4[3 - q4], 0, 0x0123)));
                    }
                    fence_proxy_async();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&a_full[as]);
                    ++g;
                }
            }
        }
    } else if (PACKED) {
        // Epilogue (packed mode): warp group h drains columns [GC_LO(h), +GC_N(h))
        // of the tile's column set once; bit 0 of each exact FP32 sum is N tile
        // 0's parity, bit PACK_SHIFT N tile 1's.
        const uint32_t h = (uint32_t)(warp - W_EPI0) >> 2;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t col_lo = h ? GC0 : 0u, col_n = h ? (uint32_t)BN - GC0 : GC0;
        const uint32_t quad = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ACC_COL0 + col_lo;
        uint32_t it = 0;
        for (TCur c = tcur_first(a); c.t != kNoTile; tcur_next(a, c), ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, c.t, cur);
            const uint32_t r = it & 1;
            mbar_wait(&acc_full[r], (it >> 1) & 1);
            tc_fence_after();
            const uint64_t b = (uint64_t)ti.mt * BM + row;
            const uint32_t ncols0 = ti.ntc == 1 ? ti.nlast : (uint32_t)BN, ncols1 = ti.ntc == 2 ? ti.nlast : 0u;
            uint32_t w0[NWG], w1[NWG];
#pragma unroll
            for (int c = 0; c < NWG; ++c) w0[c] = w1[c] = 0u;
            if (col_lo < ncols0) {
#pragma unroll
                for (int c = 0; c < NWG; ++c) {
                    if ((uint32_t)(32 * c) >= col_n) continue;
                    uint32_t v[32];
                    tmem_ld32(quad + r * BN + 32 * c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        // exact integer F < 2^24: with exponent 23 (F < 2^23 lifted by
                        // 2^23) the mantissa is F mod 2^23, whose bits 0 and 12 we need
                        // (F >= 2^23 only when S1 = 2048: then F = 2^23 + S0)
                        const float f = __uint_as_float(v[k]);
                        const uint32_t V = __float_as_uint(f < 8388608.0f ? f + 8388608.0f : f);
                        w0[c] = (w0[c] << 1) | (V & 1u);
                        w1[c] = (w1[c] << 1) | ((V >> PACK_SHIFT) & 1u);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[r]);
            if (b >= a.n_blocks) continue;
#pragma unroll
            for (uint32_t nt = 0; nt < 2; ++nt) {
                const uint32_t ncols = nt ? ncols1 : ncols0;
                const uint32_t n0 = ti.n0 + nt * BN + col_lo;
                if (n0 >= ti.r || col_lo >= ncols) continue;
                const uint32_t nvalid = min(min(col_n, ncols - col_lo), ti.r - n0);
                store_words<GROUPED>(a, ti, b, n0, nvalid, nt ? w1 : w0);
            }
        }
    } else {
        // Epilogue (deferred mode): every warp drains its columns of N tile 0,
        // releases it, then the same columns of N tile 1 (h = warp group, lanes
        // = TMEM quadrant).  The two halves of a tile row meet in one word,
        // which is OR-ed (the output is pre-zeroed in the plain mode).
        const uint32_t h = (uint32_t)(warp - W_EPI0) >> 2;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t col_lo = h ? GC0 : 0u, col_n = h ? (uint32_t)BN - GC0 : GC0;
        const uint32_t quad = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ACC_COL0 + col_lo;
        uint32_t it = 0;
        for (TCur c = tcur_first(a); c.t != kNoTile; tcur_next(a, c), ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, c.t, cur);
            mbar_wait(&acc_full[0], it & 1);
            tc_fence_after();
            const uint64_t b = (uint64_t)ti.mt * BM + row;
#pragma unroll
            for (uint32_t nt = 0; nt < 2; ++nt) {
                const uint32_t ncols = nt < ti.ntc ? (nt + 1 == ti.ntc ? ti.nlast : (uint32_t)BN) : 0u;
                uint32_t words[NWG];
#pragma unroll
                for (int c = 0; c < NWG; ++c) words[c] = 0u;
                if (col_lo < ncols) {
                    // FP32 sums are exact integers < 2^23: adding 2^23 puts their
                    // parity in the lowest mantissa bit; two 32-column loads in flight
#pragma unroll
                    for (int c = 0; c < NWG; c += 2) {
                        uint32_t v[32], v2[32];
                        if ((uint32_t)(32 * c) < col_n) tmem_ld32(quad + nt * BN + 32 * c, v);
                        if (c + 1 < NWG && (uint32_t)(32 * (c + 1)) < col_n) tmem_ld32(quad + nt * BN + 32 * (c + 1), v2);
                        tmem_wait_ld();
                        if ((uint32_t)(32 * c) < col_n) {
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                words[c] = (words[c] << 1) | (__float_as_uint(__uint_as_float(v[k]) + 8388608.0f) & 1u);
                        }
                        if (c + 1 < NWG && (uint32_t)(32 * (c + 1)) < col_n) {
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                words[c + 1] = (words[c + 1] << 1) |
                                               (__float_as_uint(__uint_as_float(v2[k]) + 8388608.0f) & 1u);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[nt]);
                const uint32_t n0 = ti.n0 + nt * BN + col_lo;  // first row of these words
                if (b >= a.n_blocks || n0 >= ti.r || col_lo >= ncols) continue;
                const uint32_t nvalid = min(min(col_n, ncols - col_lo), ti.r - n0);  // tile end, then leaf end
                store_words<GROUPED>(a, ti, b, n0, nvalid, words);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TL_CTA(3);
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

int operand_bits() { return 4; }

qrng_status timeline(uint64_t *h_out, int reset) {
#ifdef QRNG_GEMM_TIMELINE
    QRNG_CUDA_TRY(cudaDeviceSynchronize());
    QRNG_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_timeline, sizeof(g_timeline)));
    if (reset) {
        static unsigned long long z[8 * (kTimelineStages + kTimelineCtaRows)] = {};
        QRNG_CUDA_TRY(cudaMemcpyToSymbol(g_timeline, z, sizeof z));
    }
    return QRNG_OK;
#else
    (void)h_out;
    (void)reset;
    set_error("built without -DQRNG_GEMM_TIMELINE");
    return QRNG_E_UNSUPPORTED;
#endif
}

// ---- host ------------------------------------------------------------------------
static size_t smem_bytes(uint32_t seed_words_n);
// The non-grouped kernel stages all seed words it reads in shared memory next
// to the operand rings, so (n, m) is also bounded by the 227 KB per CTA.
static bool fits_smem(uint64_t n, uint64_t m) { return smem_bytes(seed_words_needed(n, m)) <= 227u * 1024u; }

bool supported(uint64_t n, uint64_t m) { return n % 128 == 0 && n <= MAX_N && m >= 1 && m < n && fits_smem(n, m); }

uint32_t seed_words_needed(uint64_t n, uint64_t m) {
    const uint64_t n_npairs = (m + NT * BN - 1) / (NT * BN), kst = (n + KS - 1) / KS, nchunks = (kst + SPC - 1) / SPC;
    uint64_t pmax = (n_npairs - 1) * NT * BN + (nchunks - 1) * KC + 8 * (CM_PER_CHUNK - 1) + 7;
    // plain launches with narrower N pairs (small batches, plain_prows) reach at
    // most row m - 1 + 448 of the last chunk
    const uint64_t pmax_narrow = (m - 1) + nchunks * KC + NT * BN + 7;
    if (pmax_narrow > pmax) pmax = pmax_narrow;
    return (uint32_t)(pmax / 32 + 2);
}

static size_t smem_bytes(uint32_t seed_words_n) {
    return (size_t)B_SLOTS * CHUNK_BYTES + (size_t)A_STAGES * A_STAGE_BYTES + ((seed_words_n + 3) & ~3u) * 4 +
           (2 * A_STAGES + 2 * B_SLOTS + ACC_FULL + ACC_EMPTY) * 8 + 16;
}

// seed bytes (MSB-first) -> logical big-endian words, zero past L
// seed bits [off, off + L) of an MSB-first byte buffer (off = 1 drops a_1 for
// the modified Toeplitz) -> logical big-endian words, zero past L
__global__ void seed_words_kernel(const uint8_t *seed, uint64_t L, uint32_t off, uint32_t *words, uint64_t nwords) {
    const uint64_t nbytes = (off + L + 7) / 8;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pos = off + w * 32, b0 = pos / 8;
        uint64_t v40 = 0;  // 40 bits starting at byte b0
        for (int k = 0; k < 5; ++k) v40 = (v40 << 8) | (b0 + k < nbytes ? seed[b0 + k] : 0u);
        uint32_t v = (uint32_t)(v40 >> (8 - (pos & 7)));
        const uint64_t lo = w * 32;
        if (lo + 32 > L) v &= (L > lo) ? (0xFFFFFFFFu << (32 - (L - lo))) : 0u;
        words[w] = v;
    }
}

// Modified Toeplitz on this path (api.cu): block b's product input is
// x''_b = [0^pad | x_b[0, n')] (n' = n - m, pad = K - n', K = n' rounded up to
// 128), so the product is a C1 extraction with n = K on a repacked copy; the
// zeros meet seed positions whose values do not matter.  One thread per
// 32-bit word of x'' (memory byte order, like the raw stream).
__global__ void modified_repack_kernel(const uint32_t *raw, uint64_t n_blocks, uint32_t n, uint32_t nprime, uint32_t K,
                                       uint32_t *xws) {
    const uint32_t kw = K / 32, pad = K - nprime;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_blocks * kw;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i / kw;
        const int32_t o = (int32_t)((uint32_t)(i - b * kw) * 32u) - (int32_t)pad;  // first bit of x_b in this word
        const uint32_t *row = raw + b * (n / 32);
        const int32_t w0 = o >= 0 ? o / 32 : -((31 - o) / 32);                      // floor(o / 32)
        const uint32_t sh = (uint32_t)(o - 32 * w0);
        const uint32_t hi = w0 >= 0 ? bswap32(__ldg(row + w0)) : 0u;
        const uint32_t lo = (sh && w0 + 1 >= 0) ? bswap32(__ldg(row + w0 + 1)) : 0u;
        uint32_t v = sh ? ((hi << sh) | (lo >> (32 - sh))) : hi;
        xws[i] = bswap32(v);
    }
}

// y ^= the block's last m raw bits: output bit b m + i takes raw bit b n + n' + i.
// One thread per logical output word; the final partial word lives in the tail scratch.
__global__ void modified_xor_tail_kernel(const uint32_t *raw, uint64_t n_blocks, uint32_t n, uint32_t m,
                                         uint64_t m_magic, OutStream out) {
    const uint32_t nprime = n - m;
    const uint64_t gbits = n_blocks * m, gwords = (gbits + 31) / 32;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < gwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t G = w * 32, end = min(G + 32, gbits);
        uint64_t b = m_magic ? __umul64hi(G, m_magic) : G;  // G / m
        uint32_t i = (uint32_t)(G - b * m);
        uint64_t pos = G;
        uint32_t word = 0;
        while (pos < end) {
            const uint32_t len = (uint32_t)min((uint64_t)(m - i), end - pos);  // 1..32 bits of block b
            const uint64_t rb = b * n + nprime + i;                            // raw bit of y_i
            const uint64_t wi = rb >> 5;
            const uint32_t sh = (uint32_t)(rb & 31);
            const uint32_t hi = bswap32(__ldg(raw + wi));
            const uint32_t lo = (sh && len > 32 - sh) ? bswap32(__ldg(raw + wi + 1)) : 0u;  // inside block b
            const uint32_t bits = sh ? ((hi << sh) | (lo >> (32 - sh))) : hi;
            word |= (bits >> (32 - len)) << (32 - len - (uint32_t)(pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        if (w >= out.full_words) {
            if (word) atomicXor(out.tail, bswap32(word));
        } else {
            out.words[w] ^= bswap32(word);
        }
    }
}

qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s) {
    if (!supported(n, m)) {
        set_error("GEMM path: unsupported n=%llu m=%llu", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    pl.seed_words_n = seed_words_needed(n, m);
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.seed_words, pl.seed_words_n * 4, s));
    count_launch();
    seed_words_kernel<<<(unsigned)((pl.seed_words_n + 255) / 256), 256, 0, s>>>(d_seed, n + m - 1, 0, pl.seed_words,
                                                                              pl.seed_words_n);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

void plan_free(Plan &pl) {
    if (pl.seed_words) cudaFree(pl.seed_words);
    pl = Plan{};
}

// Tile runs of a launch (work distribution above).  Packed Karatsuba launches
// (leaf K <= 2048: two B chunks, reusable) take about QRNG_GEMM_RUNLEN
// (default 32) tiles per run; the others keep the strided order.  Measured
// (tools/runs_ab.sh, tools/runs_ab2.sh; kernel time, strided -> runs):
// config 2 leaves 165 -> 156 us, config 3 1098 -> 1025 us, 2^17 6.63 -> 6.12
// ms; runs of 3-7 tiles regenerate B too often (config 2 189 us at 3.5),
// runs of 100+ tiles spread the CTAs over the whole input (A re-reads miss
// L2: 2^13 leaves 1.24 ms at 221 vs 1.18 at 28); plain dense n = 1024 403
// -> 412 us and 2^18 leaves (K = 4096, no reuse) 13.44 -> 13.56 ms, hence
// strided there.  QRNG_GEMM_RUNS = runs per CTA overrides (0 = strided).
static uint32_t tile_runs(uint32_t ntiles, unsigned grid, bool reuse_b) {
    static const int per_cta = [] {
        const char *e = getenv("QRNG_GEMM_RUNS");
        return (e && *e) ? atoi(e) : -1;
    }();
    static const int run_len = [] {
        const char *e = getenv("QRNG_GEMM_RUNLEN");
        const int v = (e && *e) ? atoi(e) : 32;
        return v > 0 ? v : 32;
    }();
    if (per_cta == 0 || (per_cta < 0 && !reuse_b)) return ntiles;
    uint64_t k = per_cta > 0 ? (uint64_t)per_cta : ((uint64_t)ntiles + (uint64_t)grid * run_len / 2) / ((uint64_t)grid * run_len);
    if (k < 1) k = 1;
    const uint64_t r = (uint64_t)grid * k;
    return r < ntiles ? (uint32_t)r : ntiles;
}

template <bool GROUPED, bool PACKED = false, int NBG = 3>
static qrng_status launch_nbg(const Args &a, cudaStream_t s) {
    if ((uint64_t)a.n_mtiles * a.n_npairs > 0xFFFFFFFFull) {
        set_error("GEMM path: too many tiles");
        return QRNG_E_UNSUPPORTED;
    }
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = smem_bytes(GROUPED ? a.n_leaves * 8u : a.seed_words_n);
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(toeplitz_gemm_kernel<GROUPED, PACKED, NBG>));
        if (st != QRNG_OK) return st;
    }
    const uint32_t ntiles = a.n_mtiles * a.n_npairs;
    const unsigned grid = (unsigned)(ntiles < (uint32_t)sms ? ntiles : (uint32_t)sms);
    Args b = a;
    b.n_runs = tile_runs(ntiles, grid, GROUPED && PACKED);
    b.run_q = ntiles / b.n_runs;
    b.run_rem = ntiles % b.n_runs;
    KernelTimer tm(s, true);
    if (GROUPED) {
        const cudaError_t e = launch_pdl(toeplitz_gemm_kernel<GROUPED, PACKED, NBG>, dim3(grid), dim3(nthreads_for(NBG)), smem, s, b);
        if (e != cudaSuccess) { set_error("grouped GEMM launch: %s", cudaGetErrorString(e)); return QRNG_E_CUDA; }
    } else {
        toeplitz_gemm_kernel<GROUPED, PACKED, NBG><<<grid, nthreads_for(NBG), smem, s>>>(b);
    }
    tm.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

template <bool GROUPED, bool PACKED = false>
static qrng_status launch(const Args &a, cudaStream_t s) {
#ifdef QRNG_GEMM_NBG_FORCE  // A/B builds: one B-generator count for every launch
    return launch_nbg<GROUPED, PACKED, QRNG_GEMM_NBG_FORCE>(a, s);
#endif
    if constexpr (GROUPED && PACKED) {
        // (the deferred-mode kernel with 4 B generators spills: 2^18 leaves 12.9 -> 14.0 ms)
        if (a.n_leaves > 64) return launch_nbg<GROUPED, PACKED, 4>(a, s);
    }
    return launch_nbg<GROUPED, PACKED, 3>(a, s);
}

// Rows per N pair of a plain launch: 448 (two full N tiles) unless the batch
// has too few M tiles to fill the GPU -- then narrower pairs (multiples of 32)
// give ~one work tile per SM (a small batch is latency-bound: more, shorter
// tiles in parallel).
static uint32_t plain_prows(uint32_t n_mtiles, uint64_t m) {
    static const bool narrow = [] {  // QRNG_GEMM_NARROW=0: always 448 (A/B)
        const char *e = getenv("QRNG_GEMM_NARROW");
        return e ? atoi(e) != 0 : true;
    }();
    if (!narrow) return NT * BN;
    const uint32_t want_pairs = 148u / std::max(1u, n_mtiles);
    if (want_pairs <= (m + NT * BN - 1) / (NT * BN)) return NT * BN;
    const uint64_t rows = (m + want_pairs - 1) / want_pairs;
    return (uint32_t)std::min<uint64_t>(NT * BN, std::max<uint64_t>(32, (rows + 31) / 32 * 32));
}

qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                    const OutStream &out, cudaStream_t s) {
    Args a{};
    a.raw = reinterpret_cast<const uint32_t *>(d_raw);
    a.n_blocks = n_blocks;
    a.n = (uint32_t)n;
    a.m = (uint32_t)m;
    a.kst = (uint32_t)((n + KS - 1) / KS);
    a.k128 = (uint32_t)(n / 128);
    a.nchunks = (a.kst + SPC - 1) / SPC;
    a.n_mtiles = (uint32_t)((n_blocks + BM - 1) / BM);
    a.prows = plain_prows(a.n_mtiles, m);
    a.n_npairs = (uint32_t)((m + a.prows - 1) / a.prows);  // work tile t = (N pair t / n_mtiles, M tile t % n_mtiles)
    a.seed_words = pl.seed_words;
    a.seed_words_n = (uint32_t)pl.seed_words_n;
    a.out = out;
    return launch<false>(a, s);
}

// One-shot dense product without a plan: the kernel forms the seed words from
// the caller's seed bytes in its prologue (d_seed must stay valid until the
// kernel has run: stream order on `s`).
qrng_status extract_direct(const uint8_t *d_seed, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                           const OutStream &out, cudaStream_t s) {
    if (!supported(n, m)) {
        set_error("GEMM path: unsupported n=%llu m=%llu", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    Args a{};
    a.raw = reinterpret_cast<const uint32_t *>(d_raw);
    a.n_blocks = n_blocks;
    a.n = (uint32_t)n;
    a.m = (uint32_t)m;
    a.kst = (uint32_t)((n + KS - 1) / KS);
    a.k128 = (uint32_t)(n / 128);
    a.nchunks = (a.kst + SPC - 1) / SPC;
    a.n_mtiles = (uint32_t)((n_blocks + BM - 1) / BM);
    a.prows = plain_prows(a.n_mtiles, m);
    a.n_npairs = (uint32_t)((m + a.prows - 1) / a.prows);
    a.seed_words = nullptr;
    a.seed_words_n = seed_words_needed(n, m);
    a.seed_bytes = d_seed;
    a.seed_bits = n + m - 1;
    a.out = out;
    return launch<false>(a, s);
}

qrng_status extract_grouped(const Leaf *d_leaves, uint32_t n_leaves, uint32_t total_npairs,
                            const uint32_t *d_seeds, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                            const uint32_t *xws, uint32_t x_stride, uint32_t *yws, uint32_t y_stride,
                            uint32_t max_leaf_w, cudaStream_t s) {
    Args a{};
    a.raw = reinterpret_cast<const uint32_t *>(d_raw);
    a.n_blocks = n_blocks;
    a.n = (uint32_t)n;
    a.n_mtiles = (uint32_t)((n_blocks + BM - 1) / BM);
    a.n_npairs = total_npairs;
    a.seed_words = d_seeds;
    a.leaves = d_leaves;
    a.n_leaves = n_leaves;
    a.xws = xws;
    a.x_stride = x_stride;
    a.yws = yws;
    a.y_stride = y_stride;
    // q = floor(x / d) = umul64hi(x, ceil(2^64 / d)) exactly for x, d < 2^32
    a.mt_magic = a.n_mtiles > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / a.n_mtiles) + 1 : 0;
    static const bool packed_ok = [] {
        const char *e = getenv("QRNG_GEMM_PACKED");
        return e ? atoi(e) != 0 : true;
    }();
    if (packed_ok && max_leaf_w <= kMaxPackedK) return launch<true, true>(a, s);
    return launch<true, false>(a, s);
}

bool modified_supported(uint64_t n, uint64_t m) {
    if (m == 0 || m >= n || n % 32) return false;
    const uint64_t K = (n - m + 127) / 128 * 128;
    return K <= MAX_N && fits_smem(K, m);  // m can be far larger than K: the seed window grows with m
}

// Modified Toeplitz (api.cu): the C1 product with n = K (n' = n - m rounded up
// to 128) of the repacked inputs, seed bits a_2 .. a_n (offset 1, n - 1 bits),
// zero beyond -- the prepended zero inputs meet seed positions >= n - 1 or
// values that do not matter.
qrng_status plan_init_modified(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s) {
    if (!modified_supported(n, m)) {
        set_error("GEMM path: unsupported modified Toeplitz n=%llu m=%llu", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    const uint64_t K = (n - m + 127) / 128 * 128;
    pl.seed_words_n = seed_words_needed(K, m);
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.seed_words, pl.seed_words_n * 4, s));
    count_launch();
    seed_words_kernel<<<(unsigned)((pl.seed_words_n + 255) / 256), 256, 0, s>>>(d_seed, n - 1, 1, pl.seed_words,
                                                                              pl.seed_words_n);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

qrng_status extract_modified(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                             const OutStream &out, cudaStream_t s) {
    const uint64_t nprime = n - m, K = (nprime + 127) / 128 * 128;
    uint32_t *xws = nullptr;
    const size_t xbytes = (size_t)n_blocks * (K / 8);
    QRNG_CUDA_TRY(cudaMallocAsync(&xws, xbytes, s));
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const auto grid_for = [&](uint64_t items) {
        const uint64_t want = (items + 255) / 256, cap = (uint64_t)sms * 16;
        return (unsigned)(want < cap ? want : cap);
    };
    const uint32_t *raw = reinterpret_cast<const uint32_t *>(d_raw);
    {
        KernelTimer t(s, true, 1);
        modified_repack_kernel<<<grid_for(n_blocks * (K / 32)), 256, 0, s>>>(raw, n_blocks, (uint32_t)n,
                                                                             (uint32_t)nprime, (uint32_t)K, xws);
        t.stop();
    }
    cudaError_t e = cudaGetLastError();
    qrng_status st = e == cudaSuccess ? extract(pl, reinterpret_cast<const uint8_t *>(xws), n_blocks, K, m, out, s)
                                      : QRNG_E_CUDA;
    if (e != cudaSuccess) set_error("modified_repack_kernel: %s", cudaGetErrorString(e));
    if (st == QRNG_OK) {
        const uint64_t gwords = (n_blocks * m + 31) / 32;
        const uint64_t m_magic = m > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / m) + 1 : 0;
        KernelTimer t(s, true, 1);
        modified_xor_tail_kernel<<<grid_for(gwords), 256, 0, s>>>(raw, n_blocks, (uint32_t)n, (uint32_t)m, m_magic, out);
        t.stop();
        e = cudaGetLastError();
        if (e != cudaSuccess) { set_error("modified_xor_tail_kernel: %s", cudaGetErrorString(e)); st = QRNG_E_CUDA; }
    }
    cudaFreeAsync(xws, s);
    return st;
}

}  // namespace gemm
}  // namespace qrng