// gemm_tc.cu -- batched dense Toeplitz product on tcgen05 int8 tensor cores.
//
// Method: the direct O(mn) product k = T r of PAPER.md:189-197 (Listing 1 at
// PAPER.md:388-400) for ALL blocks at once.  Every block shares the seed, so
// the blocks form the columns of one matrix and the extraction is one dense
// contraction  D[b][i] = sum_j T[i][j] x_b[j]  (exact int32, max value n),
// followed by parity: y_i = D[b][i] & 1 (C1).
//
// B200 design:
//  * Rewritten as a Hankel product with the K index reversed, j'' = n-1-j:
//        T[i][j] = s[i + j'']            A[b][j''] = x_b[n-1-j'']
//    so the B operand (rows i, K j'') is a sliding window of the seed with
//    positive unit strides in both directions.
//  * B operand (N = 192 output rows) in shared memory, generated on chip from
//    the packed seed, never read from HBM/L2: in the K-major no-swizzle
//    canonical layout a core matrix (8 rows x 16 K-bytes) at (row group g,
//    K chunk q) only depends on g + 2q, so ONE linear array of core matrices
//    with SBO = 128 B (row-group stride) and LBO = 256 B (K-chunk stride)
//    describes every B tile; the MMA simply reads overlapping windows of it.
//  * A operand (M = 128 blocks) in TMEM: "transform" warps load 16 packed
//    bytes per block and K-stage, expand bits to int8 0/-1 with SHF + PRMT
//    (sign-replicate) in registers and tcgen05.st them (32 columns = 128 K per
//    stage, 4-stage ring).
//  * tcgen05.mma.cta_group::1.kind::i8 M128 N192 K32, S32 accumulators in
//    TMEM.  Each expanded A stage feeds TWO N tiles (two accumulators, 8 MMAs
//    per stage), halving the bit-expansion work per tensor-core op; the B
//    chunk for the second tile is the first one shifted by 24 core matrices.
//  * Epilogue warps tcgen05.ld the accumulators, take parity, pack 32 outputs
//    per word MSB-first and store them at bit b*m + i (C4).
//  * Persistent grid (one CTA per SM), warp-specialised, mbarrier pipelines.
#include <algorithm>
#include <cstdlib>
#include "qrng_internal.cuh"

namespace qrng {
namespace gemm {

#ifndef QRNG_GEMM_DEFER
#define QRNG_GEMM_DEFER 2  // MMAs of N tile 1 of the next tile start this many A stages late (0: off)
#endif
#ifndef QRNG_GEMM_KS_FP4
#define QRNG_GEMM_KS_FP4 512  // K per A stage of the E2M1 kernel (256 or 512; 512 measured faster)
#endif

constexpr int BM = 128;        // blocks per tile (TMEM lanes)
constexpr int BN = QRNG_GEMM_BN;  // output rows per N tile
// Operand format.  FP4 (default): tcgen05.mma kind::mxf4 -- E2M1 0/1 operands
// (0x0 / 0x2 = 0.0 / 1.0, two per byte) with unit UE8M0 block scales, both
// operands in shared memory, FP32 accumulators (exact: every product is 0 or 1
// and every partial sum an integer <= n <= 2^16 < 2^24), twice the int8 MMA
// rate.  Otherwise kind::i8 with A in TMEM and S32 accumulators.
constexpr bool FP4 = QRNG_GEMM_FP4 != 0;
constexpr int KS = FP4 ? QRNG_GEMM_KS_FP4 : 128;  // K per A stage (FP4: KS/64 MMAs of K64 per N tile per stage)
constexpr int KS128 = KS / 128;      // 128-bit raw chunks per A stage
#ifndef QRNG_GEMM_ASTAGES_FP4
#define QRNG_GEMM_ASTAGES_FP4 2
#endif
constexpr int A_STAGES = FP4 ? QRNG_GEMM_ASTAGES_FP4 : QRNG_GEMM_ASTAGES;  // A ring slots (FP4: smem; i8: TMEM, 32 columns each)
constexpr int A_STAGE_BYTES = 128 * KS / 2;  // FP4 A stage in smem: BM rows x KS nibbles
constexpr int A_SBO = KS / 32 * 128;          // FP4 A stage: byte stride between 8-row core-matrix groups
#ifndef QRNG_GEMM_KC
#define QRNG_GEMM_KC 1024
#endif
constexpr int KC = QRNG_GEMM_KC;  // K per B chunk
constexpr int SPC = KC / KS;   // A stages per B chunk
#ifndef QRNG_GEMM_BSLOTS
#define QRNG_GEMM_BSLOTS 3
#endif
constexpr int B_SLOTS = QRNG_GEMM_BSLOTS;  // B chunk ring slots
constexpr int NT = QRNG_GEMM_NT;  // N tiles per A stage (A reuse factor)
// accumulator sets in TMEM (2 lets the MMAs of tile k+1 overlap the drain of tile k; needs NT = 1)
constexpr int ACC_BUFS = QRNG_GEMM_ACCBUFS;
constexpr int CM_PER_CHUNK = KC / 8 + NT * BN / 8 - 1;  // core matrices per chunk
constexpr int CHUNK_BYTES = CM_PER_CHUNK * 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t A_COL0 = 0;    // i8: A stages in columns [0, 32 A_STAGES)
constexpr uint32_t ACC_COL0 = FP4 ? 0u : 32u * A_STAGES;  // accumulator sets (buffer x N tile)
constexpr uint32_t SF_COL = ACC_COL0 + ACC_BUFS * NT * BN;  // FP4: unit block scales (16 columns of 0x7F)
// FP4 packed-accumulator mode (tiles with K <= 2048, i.e. Karatsuba leaves of
// w <= 2048): N tile 1's MMAs accumulate into N tile 0's FP32 accumulator with
// B scaled by 2^PACK_SHIFT, so one 192-column set holds both sums exactly
// (S0 + 2^12 S1 <= 2048 + 2^12 * 2048 < 2^24; every partial sum is an integer
// of that form): bit 0 and bit 12 of the integer are the two parities.  Two such sets alternate between tiles, so
// the drain -- half the TMEM reads -- overlaps the next tile's MMAs.
constexpr int PACK_SHIFT = 12;
constexpr uint32_t kMaxPackedK = 2048;
constexpr uint32_t SF2_COL = SF_COL + 16;  // FP4: block scales 2^PACK_SHIFT (UE8M0 127 + 12)
constexpr int ACC_FULL = FP4 ? 2 : ACC_BUFS;
static_assert((FP4 ? 32 : A_STAGES * 32) + ACC_BUFS * NT * BN <= (int)TMEM_COLS, "TMEM budget");
constexpr bool PACK_OK = FP4 && NT == 2 && ACC_BUFS == 1;  // packed mode alternates the two N-tile column sets
static_assert(ACC_BUFS == 1 || NT == 1, "epilogue warp groups: one per buffer (NT = 1) or one per N tile");
// Deferred second N tile (NT = 2, one accumulator set): the epilogue drains
// N tile 0 and then N tile 1 (all 8 warps, half the columns each); the next
// tile's MMAs start on N tile 0 as soon as it is drained and catch up N tile 1
// after QRNG_GEMM_DEFER A stages, so half of the drain overlaps the MMAs.
constexpr bool DEFER_ON = QRNG_GEMM_DEFER > 0 && NT == 2 && ACC_BUFS == 1 && (BN == 192 || (FP4 && BN == 224));
// deferred / packed epilogues: warp group h drains columns [GC_LO(h), GC_LO(h) + GC_N(h))
// of an N tile (BN = 192: 96 + 96; BN = 224: 128 + 96), at most NWG words each
constexpr uint32_t GC0 = 32 * ((BN / 32 + 1) / 2);
constexpr int NWG = GC0 / 32;
constexpr int DEFER = QRNG_GEMM_DEFER > 0 ? (QRNG_GEMM_DEFER < KC / KS ? QRNG_GEMM_DEFER : KC / KS - 1) : 1;
static_assert(!DEFER_ON || (DEFER < A_STAGES && DEFER < KC / KS), "deferred stages stay resident in one chunk");
static_assert(!FP4 || DEFER_ON || (NT == 1 && ACC_BUFS == 2),
              "the FP4 operand path: deferred NT = 2 / BN = 192, or one N tile with double-buffered accumulators");
constexpr int ACC_EMPTY = DEFER_ON ? 2 : ACC_BUFS;
// Warp roles.  The A transform uses XF_PAR warps per TMEM lane quadrant, each
// taking every XF_PAR-th stage, so the per-stage latency chain (wait slot ->
// expand -> tcgen05.st -> wait::st -> arrive) of one warp is overlapped.
#ifndef QRNG_GEMM_XFPAR
#define QRNG_GEMM_XFPAR 1
#endif
constexpr int XF_PAR = QRNG_GEMM_XFPAR;
constexpr int W_MMA = 0, W_BGEN0 = 1, N_BGEN = 3, W_XFORM0 = 4, N_XFORM = 4 * XF_PAR, W_EPI0 = W_XFORM0 + N_XFORM,
              N_EPI = 8;
constexpr int NTHREADS = (W_EPI0 + N_EPI) * 32;
static_assert(A_STAGES % XF_PAR == 0, "each transform warp owns fixed ring slots");
#ifndef QRNG_GEMM_PF
#define QRNG_GEMM_PF (KS > 256 ? 2 : 4)
#endif
constexpr int PF = QRNG_GEMM_PF;  // A-transform prefetch depth (stages)
constexpr int MAX_N = 1 << 16;
#if !QRNG_GEMM_2CTA
static_assert(kTileRows == NT * BN, "leaf tables assume NT*BN rows per work tile");
#endif

// ---- PTX helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
#ifndef QRNG_GEMM_POLL
#define QRNG_GEMM_POLL 0  // 1: spin on mbarrier.test_wait instead of the suspending try_wait
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t done;
    do {
#if QRNG_GEMM_POLL
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
#else
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
#endif
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
                 : "memory");
}
// true in exactly one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, int8 x int8 -> s32, M128, N from idesc, K32
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

#define QRNG_R8(i) "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]), "r"(v[i + 3]), "r"(v[i + 4]), "r"(v[i + 5]), "r"(v[i + 6]), "r"(v[i + 7])
#define QRNG_W8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])

// Each thread writes 32 consecutive 32-bit columns of its own TMEM lane.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        QRNG_R8(0), QRNG_R8(8), QRNG_R8(16), QRNG_R8(24)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16};" ::"r"(taddr),
        QRNG_R8(0), QRNG_R8(8)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : QRNG_W8(0), QRNG_W8(8), QRNG_W8(16), QRNG_W8(24)
        : "r"(taddr)
        : "memory");
}
// 64 consecutive S32 columns of this thread's lane, the low 16 bits of columns
// 2k and 2k+1 packed into register k (bit 0 and bit 16 carry their parities)
__device__ __forceinline__ void tmem_ld32_pack16(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : QRNG_W8(0), QRNG_W8(8), QRNG_W8(16), QRNG_W8(24)
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16_pack16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15}, [%16];"
        : QRNG_W8(0), QRNG_W8(8)
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, no swizzle (canonical layout:
// 8x16-byte core matrices; LBO = K-direction stride, SBO = 8-row-group stride).
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version for sm_100
    return d;         // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// kind::i8 instruction descriptor: S32 accumulate, S8 x S8, both K-major.
// Operand bytes are 0x00 / 0xFF = 0 / -1, so every product is 0 or +1 and the
// S32 sum is exactly the count sum_j T[i][j] x_j (at most n <= 2^16).
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool is_signed = true) {
    return (2u << 4) | ((is_signed ? 1u : 0u) << 7) | ((is_signed ? 1u : 0u) << 10) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_mxf4_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, bool acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"((uint32_t)acc), "r"(sfa), "r"(sfb)
        : "memory");
}
// 32 E2M1 elements (one core-matrix row, 16 bytes) from a 32-bit window v:
// slot 8i + j (word i, nibble j) takes bit 4j + i of v as 0x0 / 0x2.  A and B
// use the same slot order, so the K permutation cancels in the dot product.
__device__ __forceinline__ uint4 e2m1_row(uint32_t v) {
    return make_uint4((v << 1) & 0x22222222u, v & 0x22222222u, (v >> 1) & 0x22222222u, (v >> 2) & 0x22222222u);
}

// prmt.b32 with sign-replicate selectors: each output byte is 0x00 or 0xFF,
// the MSB of the selected byte of {b, a} replicated.
template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL));
    return d;
}

// K order inside every 16-slot core-matrix chunk (any fixed permutation is
// allowed because A and B use the same one and a chunk's core matrix still
// depends only on g + 2q):  slot s = 4*cc + f holds chunk element
//     r(s) = 15 - 8*(f & 1) - 2*cc - (f >> 1)
// (elements counted along the reversed K index j'').  This is the order in
// which 8 shifted copies of a raw word expose their bits at byte MSBs, so both
// operands are built with SHF + PRMT only.

#ifndef QRNG_GEMM_PACK16
#define QRNG_GEMM_PACK16 1  // epilogue: tcgen05.ld .pack::16b (two S32 columns per register, low halves)
#endif
#ifndef QRNG_GEMM_EXP
#define QRNG_GEMM_EXP 0  // timing experiments only (results wrong when != 0)
#endif

// ---- optional cycle tracing (build with -DQRNG_GEMM_TRACE; qrng_debug_gemm_trace) ----
// Slots: 0 MMA wait a_full, 1 MMA wait b_full, 2 MMA wait acc_empty, 3 MMA total,
// 4 xform wait a_empty, 5 xform expand+st+wait::st, 6 xform total, 7 B-gen wait b_empty,
// 8 B-gen total, 9 epilogue wait acc_full, 10 epilogue total, 11 stages (MMA side),
// 12 MMA wait acc_empty[1], 13 prologue, 14/15 CTA span (globaltimer), 16 MMA
// elected issue blocks, 17 MMA per-tile setup (tile_info + descriptors)
#ifdef QRNG_GEMM_TRACE
__device__ unsigned long long g_trace[32];
// counters accumulate in registers (constant slots) and are flushed once per
// warp at exit, so tracing does not put global atomics inside the pipeline
#define TRACE_DECL unsigned long long trl[32] = {}
#define TRACE_T0(v) const long long v = clock64()
#define TRACE_ADD(slot, t0) (trl[slot] += (unsigned long long)(clock64() - (t0)))
#define TRACE_ADDV(slot, v) (trl[slot] += (unsigned long long)(v))
#else
#define TRACE_DECL
#define TRACE_T0(v)
#define TRACE_ADD(slot, t0)
#define TRACE_ADDV(slot, v)
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
    const uint32_t *seed_words;  // logical big-endian seed words, zero padded
    uint32_t seed_words_n;
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
        ti.n0 = (t / a.n_mtiles) * (NT * BN);
        ti.kst = a.kst;
        ti.k128 = a.k128;
        ti.nchunks = a.nchunks;
        ti.r = a.m;
        ti.seed = seed_s;
        ti.xb = a.raw;
        ti.xs = a.n >> 5;
        ti.out_off = 0;
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

// One stage: 128 K elements of one block from its 16 raw bytes (memory words
// M_0..M_3, stream order, MSB-first bytes).  S_a = M_q << a puts stream bit
// 32q + 8k + a (bit a of byte k) at the MSB of byte k.  Chunk G of the stage
// (16 reversed-K elements) is bytes k0, k0+1 of word q = 3 - G/2, k0 = 2 - 2(G&1);
// its column cc takes bytes {k0, k0+1} of S_2cc and S_2cc+1 (order of r(s)).
__device__ __forceinline__ void xform_stage(uint32_t taddr, uint4 w) {
    const uint32_t M[4] = {w.x, w.y, w.z, w.w};
    uint32_t v[32];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t S[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) S[a] = M[q] << a;
        const int G0 = 2 * (3 - q);  // chunk of bytes {2,3}; G0 + 1 is bytes {0,1}
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            v[4 * G0 + cc] = prmt_sign<0xFEBA>(S[2 * cc], S[2 * cc + 1]);
            v[4 * (G0 + 1) + cc] = prmt_sign<0xDC98>(S[2 * cc], S[2 * cc + 1]);
        }
    }
    tmem_st32(taddr, v);
}

template <bool GROUPED, bool PACKED = false>
__global__ void __launch_bounds__(NTHREADS, 1) toeplitz_gemm_kernel(Args a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *chunks = smem;
    uint8_t *a_ring = smem + B_SLOTS * CHUNK_BYTES;  // FP4: A stages (core-matrix layout, LBO 128, SBO 512)
    uint32_t *seed_s = reinterpret_cast<uint32_t *>(a_ring + (FP4 ? A_STAGES * A_STAGE_BYTES : 0));
    // plain mode: the seed words; grouped mode: the leaf table (leaf seeds stay in global / L1)
    const uint32_t seed_stage = GROUPED ? a.n_leaves * 8u : a.seed_words_n;
    uint64_t *bars = reinterpret_cast<uint64_t *>(seed_s + ((seed_stage + 3) & ~3u));
    uint64_t *a_full = bars, *a_empty = bars + A_STAGES, *b_full = bars + 2 * A_STAGES;
    uint64_t *b_empty = b_full + B_SLOTS, *acc_full = b_empty + B_SLOTS, *acc_empty = acc_full + ACC_FULL;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + ACC_EMPTY);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef QRNG_GEMM_TRACE
    const long long t_entry = clock64();
    if (threadIdx.x == 0) {  // CTA span in global ns: slot 14 max end (set at exit), slot 15 max ~start
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        atomicMax(&g_trace[15], ~g);
    }
#endif
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
        for (uint32_t i = threadIdx.x; i < seed_stage; i += NTHREADS) seed_s[i] = a.seed_words[i];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < A_STAGES; ++s) { mbar_init(&a_full[s], N_XFORM / XF_PAR); mbar_init(&a_empty[s], 1); }
        for (int s = 0; s < B_SLOTS; ++s) { mbar_init(&b_full[s], N_BGEN); mbar_init(&b_empty[s], 1); }
        for (int s = 0; s < ACC_FULL; ++s) mbar_init(&acc_full[s], 1);
        for (int s = 0; s < ACC_EMPTY; ++s) mbar_init(&acc_empty[s], DEFER_ON ? N_EPI : N_EPI / ACC_BUFS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_MMA) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (FP4) {
        // unit block scales: UE8M0 127 = 2^0 in every byte of the scale-factor columns
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
    }
    const uint32_t ntiles = a.n_mtiles * a.n_npairs;  // n_npairs: total over leaves in grouped mode
    uint32_t cur = 0;                                 // leaf cursor of this role
    if (GROUPED) {
        pdl_release();  // the combine kernel may be scheduled as CTAs finish
        pdl_wait();     // the Q buffers (previous kernel) are complete
    }
    TRACE_T0(t_role);
    TRACE_DECL;

#ifndef QRNG_GEMM_SOLO
#define QRNG_GEMM_SOLO 1  // one elected lane runs the whole MMA loop (no per-stage warp reconvergence)
#endif
    if (PACKED && QRNG_GEMM_SOLO && warp == W_MMA) {
        if (elect_one()) {
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
                const uint32_t r = it & 1, acc = tmem + ACC_COL0 + r * BN;
                const uint32_t idesc0 = idesc_mxf4(BM, ti.ntc == 1 ? (int)ti.nlast : BN), idesc1 = idesc_mxf4(BM, (int)ti.nlast);
                mbar_wait(&acc_empty[r], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC;
                    if (kin == 0) { mbar_wait(&b_full[bs], bph); tc_fence_after(); }
                    mbar_wait(&a_full[as], aph);
                    tc_fence_after();
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
                        if (ti.ntc == 2)
                            mma_mxf4_ss(acc, adesc, bdesc + BN, idesc1, tmem + SF_COL, tmem + SF2_COL, true);  // + BN/8 cm
                    }
                    mma_commit(&a_empty[as]);
                    if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                    if (kin == SPC - 1 || ks == ti.kst - 1) {
                        if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                    }
                }
                mma_commit(&acc_full[r]);
            }
        }
        __syncwarp();
    } else if (PACKED && warp == W_MMA) {
        // packed mode: both N tiles into one of two alternating column sets
        uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            const uint32_t r = it & 1, acc = tmem + ACC_COL0 + r * BN;
            const uint32_t idesc0 = idesc_mxf4(BM, ti.ntc == 1 ? (int)ti.nlast : BN), idesc1 = idesc_mxf4(BM, (int)ti.nlast);
            { TRACE_T0(tw); mbar_wait(&acc_empty[r], ((it >> 1) & 1) ^ 1); if (lane == 0) TRACE_ADD(2, tw); }
            tc_fence_after();
            for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                const uint32_t kin = ks % SPC;
                if (kin == 0) {
                    { TRACE_T0(tw); mbar_wait(&b_full[bs], bph); if (lane == 0) TRACE_ADD(1, tw); }
                    tc_fence_after();
                }
                { TRACE_T0(tw); mbar_wait(&a_full[as], aph); if (lane == 0) TRACE_ADD(0, tw); }
                tc_fence_after();
                const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                const uint32_t abase = smem_u32(a_ring + as * A_STAGE_BYTES);
                if (lane == 0) TRACE_ADDV(11, 1);
                TRACE_T0(tiss);
                if (elect_one()) {
#pragma unroll
                    for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                        const uint32_t koff = kin * KS + kk * 64;
                        const uint64_t adesc = desc_kmajor(abase + kk * 256, 128, A_SBO);
                        mma_mxf4_ss(acc, adesc, desc_kmajor(cbase + (koff / 8) * 128, 512, 128), idesc0,
                                    tmem + SF_COL, tmem + SF_COL + 8, (ks | kk) != 0);
                        if (ti.ntc == 2)  // N tile 1, B scaled by 2^PACK_SHIFT, same columns
                            mma_mxf4_ss(acc, adesc, desc_kmajor(cbase + (koff / 8 + BN / 8) * 128, 512, 128), idesc1,
                                        tmem + SF_COL, tmem + SF2_COL, true);
                    }
                    mma_commit(&a_empty[as]);
                    if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                }
                __syncwarp();
                if (lane == 0) TRACE_ADD(16, tiss);
                if (++as == A_STAGES) { as = 0; aph ^= 1; }
                if (kin == SPC - 1 || ks == ti.kst - 1) {
                    if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                }
            }
            if (elect_one()) mma_commit(&acc_full[r]);
            __syncwarp();
        }
    } else if (DEFER_ON && FP4 && QRNG_GEMM_SOLO && warp == W_MMA) {
        // the same loop run by one elected lane (no per-stage warp reconvergence)
        if (elect_one()) {
            // converged warp, elected issue; N tile 1 of each tile is deferred DEFER stages
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                TRACE_T0(tsetup);
                const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
                const uint32_t idesc_full = FP4 ? idesc_mxf4(BM, BN) : idesc_i8(BM, BN);
                const uint32_t idesc_last = FP4 ? idesc_mxf4(BM, (int)ti.nlast) : idesc_i8(BM, (int)ti.nlast);
                const uint32_t ph = (it & 1) ^ 1;
                if (lane == 0) TRACE_ADD(17, tsetup);
                { TRACE_T0(tw); mbar_wait(&acc_empty[0], ph); if (lane == 0) TRACE_ADD(2, tw); }
                const bool defer = ti.ntc == 2 && ti.kst > (uint32_t)DEFER;
                if (!defer) { TRACE_T0(tw); mbar_wait(&acc_empty[1], ph); if (lane == 0) TRACE_ADD(12, tw); }
                tc_fence_after();
                bool nt1_on = !defer;
                uint32_t dslot[DEFER];
                uint32_t cb0 = 0;
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC;
                    if (kin == 0) {
                        { TRACE_T0(tw); mbar_wait(&b_full[bs], bph); if (lane == 0) TRACE_ADD(1, tw); }
                        tc_fence_after();
                    }
                    { TRACE_T0(tw); mbar_wait(&a_full[as], aph); if (lane == 0) TRACE_ADD(0, tw); }
                    if (lane == 0) TRACE_ADDV(11, 1);
                    tc_fence_after();
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                    if (ks == 0) cb0 = cbase;
                    if (!nt1_on && ks == (uint32_t)DEFER) {
                        // N tile 1 drained: its MMAs for the held stages, then release them
                        { TRACE_T0(tw); mbar_wait(&acc_empty[1], ph); if (lane == 0) TRACE_ADD(12, tw); }
                        tc_fence_after();
                        {
    #pragma unroll
                            for (int d = 0; d < DEFER; ++d) {
                                if constexpr (FP4) {
                                    const uint64_t adesc0 = desc_kmajor(smem_u32(a_ring + dslot[d] * A_STAGE_BYTES), 128, A_SBO);
                                    const uint64_t bdesc0 = desc_kmajor(cb0 + (d * KS / 8 + BN / 8) * 128, 512, 128);
    #pragma unroll
                                    for (uint32_t kk = 0; kk < KS / 64; ++kk)
                                        mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc0 + kk * 16, bdesc0 + kk * 64, idesc_last,
                                                    tmem + SF_COL, tmem + SF_COL + 8, (d | kk) != 0);
                                } else {
    #pragma unroll
                                    for (uint32_t kk = 0; kk < 4; ++kk) {
                                        const uint32_t koff = d * KS + kk * 32;
                                        const uint64_t bdesc = desc_kmajor(cb0 + (koff / 8 + BN / 8) * 128, 256, 128);
                                        mma_i8_ts(tmem + ACC_COL0 + BN, tmem + A_COL0 + dslot[d] * 32 + kk * 8, bdesc,
                                                  idesc_last, (d | kk) != 0);
                                    }
                                }
                                mma_commit(&a_empty[dslot[d]]);
                            }
                        }
                    
                        nt1_on = true;
                    }
                    const uint32_t a_tmem = tmem + A_COL0 + as * 32;
                    TRACE_T0(tiss);
                    {
                        if constexpr (FP4) {
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
                        } else {
    #pragma unroll
                        for (uint32_t kk = 0; kk < 4; ++kk) {
                            const uint32_t koff = kin * KS + kk * 32;
                            const uint64_t bdesc0 = desc_kmajor(cbase + (koff / 8) * 128, 256, 128);
                            mma_i8_ts(tmem + ACC_COL0, a_tmem + kk * 8, bdesc0, ti.ntc == 1 ? idesc_last : idesc_full,
                                      (ks | kk) != 0);
                            if (nt1_on && ti.ntc == 2) {
                                const uint64_t bdesc1 = desc_kmajor(cbase + (koff / 8 + BN / 8) * 128, 256, 128);
                                mma_i8_ts(tmem + ACC_COL0 + BN, a_tmem + kk * 8, bdesc1, idesc_last, (ks | kk) != 0);
                            }
                        }
                        }
                        if (nt1_on) mma_commit(&a_empty[as]);
                        if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                    }
                
                    if (lane == 0) TRACE_ADD(16, tiss);
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
    } else if (DEFER_ON && warp == W_MMA) {
        // converged warp, elected issue; N tile 1 of each tile is deferred DEFER stages
        uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            TRACE_T0(tsetup);
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            const uint32_t idesc_full = FP4 ? idesc_mxf4(BM, BN) : idesc_i8(BM, BN);
            const uint32_t idesc_last = FP4 ? idesc_mxf4(BM, (int)ti.nlast) : idesc_i8(BM, (int)ti.nlast);
            const uint32_t ph = (it & 1) ^ 1;
            if (lane == 0) TRACE_ADD(17, tsetup);
            { TRACE_T0(tw); mbar_wait(&acc_empty[0], ph); if (lane == 0) TRACE_ADD(2, tw); }
            const bool defer = ti.ntc == 2 && ti.kst > (uint32_t)DEFER;
            if (!defer) { TRACE_T0(tw); mbar_wait(&acc_empty[1], ph); if (lane == 0) TRACE_ADD(12, tw); }
            tc_fence_after();
            bool nt1_on = !defer;
            uint32_t dslot[DEFER];
            uint32_t cb0 = 0;
            for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                const uint32_t kin = ks % SPC;
                if (kin == 0) {
                    { TRACE_T0(tw); mbar_wait(&b_full[bs], bph); if (lane == 0) TRACE_ADD(1, tw); }
                    tc_fence_after();
                }
                { TRACE_T0(tw); mbar_wait(&a_full[as], aph); if (lane == 0) TRACE_ADD(0, tw); }
                if (lane == 0) TRACE_ADDV(11, 1);
                tc_fence_after();
                const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                if (ks == 0) cb0 = cbase;
                if (!nt1_on && ks == (uint32_t)DEFER) {
                    // N tile 1 drained: its MMAs for the held stages, then release them
                    { TRACE_T0(tw); mbar_wait(&acc_empty[1], ph); if (lane == 0) TRACE_ADD(12, tw); }
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int d = 0; d < DEFER; ++d) {
                            if constexpr (FP4) {
                                const uint32_t abase = smem_u32(a_ring + dslot[d] * A_STAGE_BYTES);
#pragma unroll
                                for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                                    const uint32_t koff = d * KS + kk * 64;
                                    mma_mxf4_ss(tmem + ACC_COL0 + BN, desc_kmajor(abase + kk * 256, 128, A_SBO),
                                                desc_kmajor(cb0 + (koff / 8 + BN / 8) * 128, 512, 128), idesc_last,
                                                tmem + SF_COL, tmem + SF_COL + 8, (d | kk) != 0);
                                }
                            } else {
#pragma unroll
                                for (uint32_t kk = 0; kk < 4; ++kk) {
                                    const uint32_t koff = d * KS + kk * 32;
                                    const uint64_t bdesc = desc_kmajor(cb0 + (koff / 8 + BN / 8) * 128, 256, 128);
                                    mma_i8_ts(tmem + ACC_COL0 + BN, tmem + A_COL0 + dslot[d] * 32 + kk * 8, bdesc,
                                              idesc_last, (d | kk) != 0);
                                }
                            }
                            mma_commit(&a_empty[dslot[d]]);
                        }
                    }
                    __syncwarp();
                    nt1_on = true;
                }
                const uint32_t a_tmem = tmem + A_COL0 + as * 32;
                TRACE_T0(tiss);
                if (elect_one()) {
                    if constexpr (FP4) {
                        const uint32_t abase = smem_u32(a_ring + as * A_STAGE_BYTES);
#pragma unroll
                        for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                            const uint32_t koff = kin * KS + kk * 64;
                            const uint64_t adesc = desc_kmajor(abase + kk * 256, 128, A_SBO);
                            mma_mxf4_ss(tmem + ACC_COL0, adesc, desc_kmajor(cbase + (koff / 8) * 128, 512, 128),
                                        ti.ntc == 1 ? idesc_last : idesc_full, tmem + SF_COL, tmem + SF_COL + 8,
                                        (ks | kk) != 0);
                            if (nt1_on && ti.ntc == 2)
                                mma_mxf4_ss(tmem + ACC_COL0 + BN, adesc,
                                            desc_kmajor(cbase + (koff / 8 + BN / 8) * 128, 512, 128), idesc_last,
                                            tmem + SF_COL, tmem + SF_COL + 8, (ks | kk) != 0);
                        }
                    } else {
#pragma unroll
                    for (uint32_t kk = 0; kk < 4; ++kk) {
                        const uint32_t koff = kin * KS + kk * 32;
                        const uint64_t bdesc0 = desc_kmajor(cbase + (koff / 8) * 128, 256, 128);
                        mma_i8_ts(tmem + ACC_COL0, a_tmem + kk * 8, bdesc0, ti.ntc == 1 ? idesc_last : idesc_full,
                                  (ks | kk) != 0);
                        if (nt1_on && ti.ntc == 2) {
                            const uint64_t bdesc1 = desc_kmajor(cbase + (koff / 8 + BN / 8) * 128, 256, 128);
                            mma_i8_ts(tmem + ACC_COL0 + BN, a_tmem + kk * 8, bdesc1, idesc_last, (ks | kk) != 0);
                        }
                    }
                    }
                    if (nt1_on) mma_commit(&a_empty[as]);
                    if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                }
                __syncwarp();
                if (lane == 0) TRACE_ADD(16, tiss);
                if (!nt1_on) dslot[ks] = as;
                if (++as == A_STAGES) { as = 0; aph ^= 1; }
                if (kin == SPC - 1 || ks == ti.kst - 1) {
                    if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                }
            }
            if (elect_one()) mma_commit(&acc_full[0]);
            __syncwarp();
        }
    } else if (FP4 && warp == W_MMA) {
        // E2M1, double-buffered accumulator sets (NT = 1): one elected lane runs the loop
        if (elect_one()) {
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
                const uint32_t idesc_full = idesc_mxf4(BM, BN), idesc_last = idesc_mxf4(BM, (int)ti.nlast);
                const uint32_t ab = it % ACC_BUFS, acc0 = ACC_COL0 + ab * NT * BN;
                mbar_wait(&acc_empty[ab], ((it / ACC_BUFS) & 1) ^ 1);
                tc_fence_after();
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC;
                    if (kin == 0) { mbar_wait(&b_full[bs], bph); tc_fence_after(); }
                    mbar_wait(&a_full[as], aph);
                    tc_fence_after();
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                    const uint32_t abase = smem_u32(a_ring + as * A_STAGE_BYTES);
#pragma unroll
                    for (uint32_t kk = 0; kk < KS / 64; ++kk) {
                        const uint32_t koff = kin * KS + kk * 64;
                        const uint64_t adesc = desc_kmajor(abase + kk * 256, 128, A_SBO);
#pragma unroll
                        for (uint32_t nt = 0; nt < NT; ++nt)
                            if (nt < ti.ntc)
                                mma_mxf4_ss(tmem + acc0 + nt * BN, adesc,
                                            desc_kmajor(cbase + (koff / 8 + nt * (BN / 8)) * 128, 512, 128),
                                            nt + 1 == ti.ntc ? idesc_last : idesc_full, tmem + SF_COL, tmem + SF_COL + 8,
                                            (ks | kk) != 0);
                    }
                    mma_commit(&a_empty[as]);
                    if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                    if (kin == SPC - 1 || ks == ti.kst - 1) {
                        if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                    }
                }
                mma_commit(&acc_full[ab]);
            }
        }
        __syncwarp();
    } else if (warp == W_MMA) {
        // the whole warp runs the issue loop converged (operands stay warp-uniform);
        // one elected lane issues each tcgen05.mma / commit
        {
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
                // N tiles before the last use N = BN; the last one only the rows it needs
                const uint32_t idesc_full = idesc_i8(BM, BN), idesc_last = idesc_i8(BM, (int)ti.nlast);
                const uint32_t ab = it % ACC_BUFS, acc0 = ACC_COL0 + ab * NT * BN;
                { TRACE_T0(tw); mbar_wait(&acc_empty[ab], ((it / ACC_BUFS) & 1) ^ 1); if (lane == 0) TRACE_ADD(2, tw); }
                tc_fence_after();
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC;
                    if (kin == 0) {
                        { TRACE_T0(tw); mbar_wait(&b_full[bs], bph); if (lane == 0) TRACE_ADD(1, tw); }
                        tc_fence_after();
                    }
                    { TRACE_T0(tw); mbar_wait(&a_full[as], aph); if (lane == 0) TRACE_ADD(0, tw); }
                    if (lane == 0) TRACE_ADDV(11, 1);
                    tc_fence_after();
                    const uint32_t a_tmem = tmem + A_COL0 + as * 32;
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK_BYTES);
                    if (elect_one()) {
#pragma unroll
                        for (uint32_t kk = 0; kk < 4; ++kk) {
                            const uint32_t koff = kin * KS + kk * 32;  // K offset inside the chunk
#pragma unroll
                            for (uint32_t nt = 0; nt < NT; ++nt) {  // N tile nt starts 24*nt core matrices later
                                if (nt < ti.ntc) {
                                    const uint64_t bdesc = desc_kmajor(cbase + (koff / 8 + nt * (BN / 8)) * 128, 256, 128);
#if QRNG_GEMM_EXP != 1  // experiment 1: no MMAs (transform / B-gen / epilogue throughput alone)
                                    mma_i8_ts(tmem + acc0 + nt * BN, a_tmem + kk * 8, bdesc,
                                              nt + 1 == ti.ntc ? idesc_last : idesc_full, (ks | kk) != 0);
#endif
                                }
                            }
                        }
                        mma_commit(&a_empty[as]);
                        if (kin == SPC - 1 || ks == ti.kst - 1) mma_commit(&b_empty[bs]);
                    }
                    __syncwarp();
                    if (++as == A_STAGES) { as = 0; aph ^= 1; }
                    if (kin == SPC - 1 || ks == ti.kst - 1) {
                        if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                    }
                }
                if (elect_one()) mma_commit(&acc_full[ab]);
                __syncwarp();
            }
        }
        __syncwarp();
    } else if (warp >= W_BGEN0 && warp < W_BGEN0 + N_BGEN) {
        // B generators: core matrix tau of chunk (n0, k0): row r' holds seed bits
        // s[n0 + k0 + 8 tau + r' + c], c = 0..15, as int8 0/1.
        const int tb = (warp - W_BGEN0) * 32 + lane;
        uint32_t bs = 0, bph = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            // core-matrix rows the MMAs of this tile read (K chunk + the N rows in use)
            const int ncm = KC / 8 + (int)(((ti.ntc - 1) * BN + ti.nlast) / 8) - 1;
            for (uint32_t c = 0; c < ti.nchunks; ++c) {
                const uint32_t base = ti.n0 + c * KC;
                { TRACE_T0(tw); mbar_wait(&b_empty[bs], bph ^ 1); if (lane == 0) TRACE_ADD(7, tw); }
                uint8_t *cb = chunks + bs * CHUNK_BYTES;
#if QRNG_GEMM_EXP >= 16 && (QRNG_GEMM_EXP & 8)  // experiment 8 (bitmask >= 16): no B generation
                if (ncm < 0)
#endif
                for (int r = tb; r < ncm * 8; r += N_BGEN * 32) {
                    // row holds seed bits p + r(s); in v (seed bit p + d at bit 31 - d) the
                    // bit of slot s = 4cc + f sits at byte 2 + (f&1), bit 2cc + (f>>1)
                    const uint32_t p = base + 8 * (r >> 3) + (r & 7);
                    uint32_t w0, w1;
                    if (GROUPED) { w0 = __ldg(ti.seed + (p >> 5)); w1 = __ldg(ti.seed + (p >> 5) + 1); }
                    else { w0 = ti.seed[p >> 5]; w1 = ti.seed[(p >> 5) + 1]; }
                    const uint32_t v = __funnelshift_l(w1, w0, p & 31);
                    uint4 o;
                    if constexpr (FP4) {
                        o = e2m1_row(v);  // 32 elements: seed bits p .. p + 31
                    } else {
                        o.x = prmt_sign<0xFEBA>(v << 7, v << 6);
                        o.y = prmt_sign<0xFEBA>(v << 5, v << 4);
                        o.z = prmt_sign<0xFEBA>(v << 3, v << 2);
                        o.w = prmt_sign<0xFEBA>(v << 1, v);
                    }
                    *reinterpret_cast<uint4 *>(cb + (r >> 3) * 128 + (r & 7) * 16) = o;
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&b_full[bs]);
                if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
            }
        }
    } else if (warp >= W_XFORM0 && warp < W_XFORM0 + N_XFORM) {
        // A transform: TMEM lane = block, 128 K per stage.  Stages are numbered
        // g = 0, 1, 2, ... over this CTA's (tile, K stage) pairs; this warp takes
        // g = par (mod XF_PAR) for its lane quadrant.  The prefetch ring of input
        // chunks runs continuously across tiles.
        const uint32_t xw = (uint32_t)(warp - W_XFORM0), par = xw / 4;
        const uint32_t row = (xw & 3) * 32 + lane;  // warp % 4 == xw % 4: TMEM lane quadrant
        const uint32_t lane_addr = tmem + (((uint32_t)(warp & 3) * 32) << 16);
        uint32_t lcur = 0;                      // leaf cursor of the load side
        uint32_t lt = blockIdx.x, lks = 0;      // load cursor (tile, K stage)
        Tile lti{};
        if (lt < ntiles) lti = tile_info<GROUPED>(a, seed_s, lt, lcur);
        auto step1 = [&]() {
            if (lt >= ntiles) return;
            if (++lks == lti.kst) {
                lks = 0;
                lt += gridDim.x;
                if (lt < ntiles) lti = tile_info<GROUPED>(a, seed_s, lt, lcur);
            }
        };
        // Branch-free prefetch: always load from a valid address (clamped block,
        // stale tile past the end) and keep a validity flag, so every ring slot
        // stays in its own registers and the load latency is really hidden.
        // K is reversed: stage lks, half hf (128 K each) reads 128-bit chunk
        // k128 - 1 - KS128 lks - hf of the block row (FP4: the second half of the
        // last stage may lie before the row start -> zeros)
        auto load = [&](bool &v, uint32_t hf) -> uint4 {
            const uint64_t b = (uint64_t)lti.mt * BM + row;
            const int32_t ci = (int32_t)lti.k128 - 1 - (int32_t)(KS128 * lks + hf);
            v = lt < ntiles && b < a.n_blocks && ci >= 0;
#if QRNG_GEMM_EXP == 3  // experiment 3: every lane reads block 0 (coalesced broadcast loads)
            const uint64_t bc = 0;
#else
            const uint64_t bc = b < a.n_blocks ? b : a.n_blocks - 1;
#endif
            return __ldg(reinterpret_cast<const uint4 *>(lti.xb + bc * lti.xs) + (ci >= 0 ? ci : 0));
        };
        for (uint32_t i = 0; i < par; ++i) step1();
        uint4 pf[PF][KS128];
        bool ok[PF], vd[PF][KS128];
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            ok[j] = lt < ntiles;
#pragma unroll
            for (int hf = 0; hf < KS128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
#pragma unroll
            for (int i = 0; i < XF_PAR; ++i) step1();
        }
        uint32_t g = par;
        bool more = true;
        while (more) {
#pragma unroll
            for (int j = 0; j < PF; ++j) {
                if (more && !ok[j]) more = false;
                if (more) {
                    uint4 cur[KS128];
#pragma unroll
                    for (int hf = 0; hf < KS128; ++hf) cur[hf] = vd[j][hf] ? pf[j][hf] : make_uint4(0, 0, 0, 0);
                    const uint4 cur4 = cur[0];
                    ok[j] = lt < ntiles;
#pragma unroll
                    for (int hf = 0; hf < KS128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
#pragma unroll
                    for (int i = 0; i < XF_PAR; ++i) step1();
                    const uint32_t as = g % A_STAGES, aph = (g / A_STAGES) & 1;
                    { TRACE_T0(tw); mbar_wait(&a_empty[as], aph ^ 1); if (lane == 0) TRACE_ADD(4, tw); }
                    tc_fence_after();
                    TRACE_T0(tx);
#if !(QRNG_GEMM_EXP == 2 || (QRNG_GEMM_EXP >= 16 && (QRNG_GEMM_EXP & 2)))  // experiment 2: no A expansion/TMEM store
                    if constexpr (FP4) {
                        // K group g (32 elements, K reversed) = memory word 3 - g, element c = bit c
                        // of its big-endian value: bit-reverse so that bit b holds element 31 - b
                        // as in the B rows, then the same nibble spread
                        uint8_t *arow = a_ring + as * A_STAGE_BYTES + (row >> 3) * A_SBO + (row & 7) * 16;
#pragma unroll
                        for (int hf = 0; hf < KS128; ++hf) {
                            const uint32_t M4[4] = {cur[hf].x, cur[hf].y, cur[hf].z, cur[hf].w};
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4)
                                *reinterpret_cast<uint4 *>(arow + (hf * 4 + q4) * 128) =
                                    e2m1_row(__brev(__byte_perm(M4[3 - q4], 0, 0x0123)));
                        }
                        fence_proxy_async();
                    } else {
                        xform_stage(lane_addr + A_COL0 + as * 32, cur4);
                        tmem_wait_st();
                    }
#else
                    if (cur4.x == 0x12345678u) __nanosleep(1);
#endif
                    if (lane == 0) TRACE_ADD(5, tx);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&a_full[as]);
                    g += XF_PAR;
                }
            }
        }
    } else if (PACKED) {
        // Epilogue (packed mode): every warp drains columns [96 h, 96 h + 96) of
        // the tile's column set once; bit 0 of each exact FP32 sum is N tile 0's
        // parity, bit PACK_SHIFT N tile 1's.
        const uint32_t h = (uint32_t)(warp - W_EPI0) >> 2;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t col_lo = h ? GC0 : 0u, col_n = h ? (uint32_t)BN - GC0 : GC0;
        const uint32_t quad = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ACC_COL0 + col_lo;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            const uint32_t r = it & 1;
            { TRACE_T0(tw); mbar_wait(&acc_full[r], (it >> 1) & 1); if (lane == 0) TRACE_ADD(9, tw); }
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
                uint32_t *words = nt ? w1 : w0;
                const uint32_t n0 = ti.n0 + nt * BN + col_lo;
                if (n0 >= ti.r || col_lo >= ncols) continue;
                const uint32_t nvalid = min(min(col_n, ncols - col_lo), ti.r - n0);
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
                    continue;
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
        }
    } else if (DEFER_ON) {
        // Epilogue (deferred mode): every warp drains columns [96 h, 96 h + 96) of
        // N tile 0, releases it, then the same columns of N tile 1 (h = warp
        // group, lanes = TMEM quadrant).  Parity of the S32 sums, 32 outputs per
        // MSB-first word; the two halves of a tile row meet in one word, which is
        // OR-ed (the output is pre-zeroed in the plain mode).
        const uint32_t h = (uint32_t)(warp - W_EPI0) >> 2;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t col_lo = h ? GC0 : 0u, col_n = h ? (uint32_t)BN - GC0 : GC0;
        const uint32_t quad = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ACC_COL0 + col_lo;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            { TRACE_T0(tw); mbar_wait(&acc_full[0], it & 1); if (lane == 0) TRACE_ADD(9, tw); }
            tc_fence_after();
            const uint64_t b = (uint64_t)ti.mt * BM + row;
#pragma unroll
            for (uint32_t nt = 0; nt < 2; ++nt) {
                const uint32_t ncols = nt < ti.ntc ? (nt + 1 == ti.ntc ? ti.nlast : (uint32_t)BN) : 0u;
                uint32_t words[NWG];
#pragma unroll
                for (int c = 0; c < NWG; ++c) words[c] = 0u;
                if (col_lo < ncols) {
                    uint32_t v[32];
                    uint32_t u[16];
#if QRNG_GEMM_EXP == 4 || (QRNG_GEMM_EXP >= 16 && (QRNG_GEMM_EXP & 4))  // experiment 4: no accumulator reads
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = row + k;
#pragma unroll
                    for (int k = 0; k < 16; ++k) u[k] = row ^ k;
#else
                    if constexpr (FP4) {
                        // FP32 sums are exact integers < 2^23: adding 2^23 puts their
                        // parity in the lowest mantissa bit; two 32-column loads in flight
#pragma unroll
                        for (int c = 0; c < NWG; c += 2) {
                            uint32_t v2[32];
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
                    } else {
                        tmem_ld32_pack16(quad + nt * BN, v);
                        tmem_ld16_pack16(quad + nt * BN + 64, u);
                        tmem_wait_ld();
                    }
#endif
                    if constexpr (!FP4) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) words[0] = (words[0] << 2) | ((v[k] & 1u) << 1) | ((v[k] >> 16) & 1u);
#pragma unroll
                    for (int k = 16; k < 32; ++k) words[1] = (words[1] << 2) | ((v[k] & 1u) << 1) | ((v[k] >> 16) & 1u);
#pragma unroll
                    for (int k = 0; k < 16; ++k) words[2] = (words[2] << 2) | ((u[k] & 1u) << 1) | ((u[k] >> 16) & 1u);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[nt]);
                const uint32_t n0 = ti.n0 + nt * BN + col_lo;  // first row of these words
                if (b >= a.n_blocks || n0 >= ti.r || col_lo >= ncols) continue;
                const uint32_t nvalid = min(min(col_n, ncols - col_lo), ti.r - n0);  // tile end, then leaf end
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
                    continue;
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
        }
    } else {
        // Epilogue: with ACC_BUFS = 2 warp group g = (w - W_EPI0) / 4 drains the
        // tiles k = g mod 2 of this CTA (accumulator set g) while the MMAs of the
        // next tile fill the other set; with one set, group g drains N tile g.
        // Parity of the S32 sums, 32 outputs per MSB-first word.
        const uint32_t grp = (uint32_t)(warp - W_EPI0) >> 2;
        const uint32_t nt = ACC_BUFS == 1 ? grp : 0u, ab = ACC_BUFS == 1 ? 0u : grp;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t lane_addr = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ACC_COL0 + ab * NT * BN + nt * BN;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x + ab * gridDim.x; t < ntiles; t += ACC_BUFS * gridDim.x, ++it) {
            const Tile ti = tile_info<GROUPED>(a, seed_s, t, cur);
            { TRACE_T0(tw); mbar_wait(&acc_full[ab], it & 1); if (lane == 0) TRACE_ADD(9, tw); }
            tc_fence_after();
            const uint32_t ncols = nt < ti.ntc ? (nt + 1 == ti.ntc ? ti.nlast : (uint32_t)BN) : 0u;
            uint32_t words[BN / 32];
#if QRNG_GEMM_PACK16
            if constexpr (FP4) {
                // FP32 sums: exact integers < 2^23, parity = lowest mantissa bit of F + 2^23
#pragma unroll
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t w = 0;
                    if ((uint32_t)(32 * c) < ncols) {
                        uint32_t v[32];
                        tmem_ld32(lane_addr + 32 * c, v);
                        tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            w = (w << 1) | (__float_as_uint(__uint_as_float(v[k]) + 8388608.0f) & 1u);
                    }
                    words[c] = w;
                }
            } else
            // 64 columns per load: only the parity (bit 0) of each S32 sum is
            // needed and it survives truncation to 16 bits
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) {
                uint32_t w0 = 0, w1 = 0;
                if ((uint32_t)(64 * c) < ncols) {
                    uint32_t v[32];
                    tmem_ld32_pack16(lane_addr + 64 * c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 16; ++k) w0 = (w0 << 2) | ((v[k] & 1u) << 1) | ((v[k] >> 16) & 1u);
#pragma unroll
                    for (int k = 16; k < 32; ++k) w1 = (w1 << 2) | ((v[k] & 1u) << 1) | ((v[k] >> 16) & 1u);
                }
                words[2 * c] = w0;
                words[2 * c + 1] = w1;
            }
#else
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t w = 0;
                if ((uint32_t)(32 * c) < ncols) {
                    uint32_t v[32];
                    tmem_ld32(lane_addr + 32 * c, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 32; ++k) w = (w << 1) | (v[k] & 1u);
                }
                words[c] = w;
            }
#endif
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
            const uint64_t b = (uint64_t)ti.mt * BM + row;
            const uint32_t n0 = ti.n0 + nt * BN;
            if (b >= a.n_blocks || n0 >= ti.r) continue;
            const uint32_t nvalid = min(ncols, ti.r - n0);
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) {
                const int vb = (int)nvalid - 32 * c;  // valid bits in word c
                if (vb <= 0) words[c] = 0;
                else if (vb < 32) words[c] &= ~(0xFFFFFFFFu >> vb);
            }
            if (GROUPED) {
                // word-aligned leaf parities (n0 % 32 == 0), logical words
                uint32_t *dst = a.yws + b * a.y_stride + ti.out_off + n0 / 32;
#pragma unroll
                for (int c = 0; c < BN / 32; ++c)
                    if ((uint32_t)(32 * c) < nvalid) dst[c] = words[c];
                continue;
            }
            const uint64_t G_lo = b * a.m + n0, G_hi = G_lo + nvalid;
            const uint32_t off = (uint32_t)(G_lo & 31);
            const uint64_t W0 = G_lo >> 5;
            uint32_t prev = 0;
#pragma unroll
            for (int c = 0; c <= BN / 32; ++c) {
                const uint32_t cw = (c < BN / 32) ? words[c] : 0u;
                const uint32_t ow = off ? ((prev << (32 - off)) | (cw >> off)) : cw;
                prev = cw;
                const uint64_t W = W0 + c;
                if (W * 32 >= G_hi) break;
                const bool excl = (W * 32 >= G_lo) && (W * 32 + 32 <= G_hi);
                emit_word(a.out, W, ow, excl);
            }
        }
    }

#ifdef QRNG_GEMM_TRACE
    if (lane == 0) {
        const int slot = warp == W_MMA ? 3 : (warp < W_XFORM0 ? 8 : (warp < W_EPI0 ? 6 : 10));
        atomicAdd(&g_trace[slot], (unsigned long long)(clock64() - t_role));
        if (warp == W_MMA) atomicAdd(&g_trace[13], (unsigned long long)(t_role - t_entry));  // prologue
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (trl[i]) atomicAdd(&g_trace[i], trl[i]);
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
#ifdef QRNG_GEMM_TRACE
    if (threadIdx.x == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        atomicMax(&g_trace[14], g);
    }
#endif
}



// ---- 2-SM variant (build with -DQRNG_GEMM_2CTA=1) ---------------------------------
// A CTA pair (cluster of 2, one per SM of a TPC) runs tcgen05.mma.cta_group::2
// M256 N256 K32: each CTA holds 128 blocks of the A operand (expanded in its
// own shared memory, K-major canonical layout) and 128 of the 256 output rows
// of the Toeplitz B operand (generated on chip as in the 1-SM kernel); each
// CTA's TMEM receives its 128 blocks x all 256 rows.  With A out of TMEM the
// 512 TMEM columns hold two 256-column accumulator sets, so the MMAs of tile
// k+1 run while the epilogue drains tile k.  The leader CTA (rank 0) issues
// the MMAs; the full barriers live in the leader and count both CTAs'
// producers (remote arrives), the empty barriers are signalled in both CTAs
// by a multicast commit.
#if QRNG_GEMM_2CTA
namespace two {
constexpr int BM2 = 256, BH = 128;          // blocks per tile, per CTA
// FP4 (kind::mxf4): 224-row tiles (whole 32-bit words, so leaf parities stay
// word aligned) so that two FP32 accumulator sets (448 columns) and the
// scale-factor columns fit in TMEM; 512-K stages (8 MMAs per handshake)
constexpr int BN2 = FP4 ? 224 : 256;        // output rows per tile (N of one MMA)
constexpr int KS2 = FP4 ? 512 : KS;         // K per A stage
constexpr int KS2_128 = KS2 / 128;
constexpr int SPC2 = KC / KS2;              // A stages per B chunk
constexpr int A2_STAGES = FP4 ? 3 : 4;      // A ring in shared memory
constexpr int A2_BYTES = FP4 ? BH * KS2 / 2 : BH * KS;  // 128 rows x the stage's K (nibbles / bytes)
constexpr int A2_SBO = FP4 ? KS2 / 32 * 128 : 1024;     // bytes between 8-row core-matrix groups
constexpr uint32_t SF2_COL = 2 * BN2;       // FP4: unit block scales after the two accumulator sets
static_assert(!FP4 || 2 * BN2 + 16 <= (int)TMEM_COLS, "TMEM budget (2-SM)");
constexpr int PF2 = FP4 ? 2 : PF;           // transform prefetch depth (stages)
constexpr int CM2 = KC / 8 + (BN2 / 2) / 8 - 1;  // core matrices per B chunk per CTA
constexpr int CHUNK2_BYTES = CM2 * 128;
constexpr int W2_MMA = 0, W2_BGEN0 = 1, N2_BGEN = 3, W2_XF0 = 4, N2_XF = 8, W2_EPI0 = 12, N2_EPI = 8;
constexpr int NTHREADS2 = 20 * 32;
constexpr int XF2_PAR = 2;                  // transform warps per 32-row quarter, alternating stages
static_assert(kTileRows == BN2, "leaf tables assume BN2 rows per work tile");

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_rank(uint64_t *b, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(b)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void mma2_mxf4_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}
__device__ __forceinline__ void mma2_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive once on `bar` (same offset) in both CTAs when the issued MMAs complete
__device__ __forceinline__ void mma2_commit_both(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

struct Tile2 {
    uint32_t mt, n0, kst, nchunks, r, ntile;  // ntile: rows of this tile (N, multiple of 16)
    uint32_t k128;                            // 128-bit input chunks per block row
    const uint32_t *seed, *xb;
    uint32_t xs, out_off;
};

template <bool GROUPED>
__device__ __forceinline__ Tile2 tile2_info(const Args &a, const uint32_t *seed_s, uint32_t t, uint32_t &cur) {
    Tile2 ti;
    uint32_t tl;
    if (!GROUPED) {
        ti.k128 = a.n / 128;
        ti.kst = (ti.k128 + KS2_128 - 1) / KS2_128;
        ti.r = a.m;
        ti.seed = seed_s;
        ti.xb = a.raw;
        ti.xs = a.n >> 5;
        ti.out_off = 0;
        tl = t;
    } else {
        while (cur + 1 < a.n_leaves && t >= (__ldg(&a.leaves[cur].npair_base) + __ldg(&a.leaves[cur].npairs)) * a.n_mtiles)
            ++cur;
        const Leaf &L = a.leaves[cur];
        tl = t - __ldg(&L.npair_base) * a.n_mtiles;
        ti.k128 = __ldg(&L.w) / 128;
        ti.kst = (ti.k128 + KS2_128 - 1) / KS2_128;
        ti.r = __ldg(&L.r);
        ti.seed = a.seed_words + __ldg(&L.seed_off);
        if (__ldg(&L.x_src) == 0) { ti.xb = a.raw + __ldg(&L.x_off); ti.xs = a.n >> 5; }
        else { ti.xb = a.xws + __ldg(&L.x_off); ti.xs = a.x_stride; }
        ti.out_off = __ldg(&L.out_off);
    }
    ti.mt = tl % a.n_mtiles;
    ti.n0 = (tl / a.n_mtiles) * BN2;
    ti.nchunks = (ti.kst + SPC2 - 1) / SPC2;
    const uint32_t left = ti.r > ti.n0 ? min((uint32_t)BN2, ti.r - ti.n0) : 16u;
    ti.ntile = (left + 15) & ~15u;
    return ti;
}

template <bool GROUPED>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS2, 1) toeplitz_gemm2_kernel(Args a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *abuf = smem;                                   // A2_STAGES x 16 KB
    uint8_t *chunks = smem + A2_STAGES * A2_BYTES;          // B_SLOTS x CHUNK2_BYTES
    uint32_t *seed_s = reinterpret_cast<uint32_t *>(chunks + B_SLOTS * CHUNK2_BYTES);
    const uint32_t seed_stage = GROUPED ? 0u : a.seed_words_n;
    uint64_t *bars = reinterpret_cast<uint64_t *>(seed_s + ((seed_stage + 3) & ~3u));
    uint64_t *a_full = bars, *a_empty = bars + A2_STAGES, *b_full = bars + 2 * A2_STAGES;
    uint64_t *b_empty = b_full + B_SLOTS, *acc_full = b_empty + B_SLOTS, *acc_empty = acc_full + 2;
    uint64_t *a_local = acc_empty + 2;  // peer CTA: its transform warps' arrivals, relayed to the leader
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_local + A2_STAGES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    for (uint32_t i = threadIdx.x; i < seed_stage; i += NTHREADS2) seed_s[i] = a.seed_words[i];
    if (threadIdx.x == 0) {
        // leader a_full: its own 4 transform warps of the stage + one relayed arrive from the peer
        for (int s = 0; s < A2_STAGES; ++s) {
            mbar_init(&a_full[s], 4 + 1);
            mbar_init(&a_empty[s], 1);
            mbar_init(&a_local[s], 4);
        }
        for (int s = 0; s < B_SLOTS; ++s) { mbar_init(&b_full[s], 2 * N2_BGEN); mbar_init(&b_empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], 2 * 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W2_MMA) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (FP4) {
        // unit block scales (UE8M0 127) in this CTA's scale-factor columns
        if (warp >= W2_EPI0 && warp < W2_EPI0 + 4) {
            uint32_t v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = 0x7F7F7F7Fu;
            tmem_st16(tmem + (((uint32_t)(warp & 3) * 32) << 16) + SF2_COL, v);
            tmem_wait_st();
        }
        tc_fence_before();
        cluster_sync();
        tc_fence_after();
    }
    const uint32_t pair = blockIdx.x >> 1, npairs_grid = gridDim.x >> 1;
    const uint32_t ntiles = a.n_mtiles * a.n_npairs;  // n_npairs: N tiles of 256 rows (total over leaves)
    uint32_t cur = 0;

    if (warp == W2_MMA) {
        if (rank == 0) {  // converged warp, one elected lane issues
            uint32_t as = 0, aph = 0, bs = 0, bph = 0, it = 0;
            for (uint32_t t = pair; t < ntiles; t += npairs_grid, ++it) {
                const Tile2 ti = tile2_info<GROUPED>(a, seed_s, t, cur);
                const uint32_t idesc = FP4 ? idesc_mxf4(BM2, (int)ti.ntile) : idesc_i8(BM2, (int)ti.ntile);
                const uint32_t ab = it & 1, acc = ab * BN2;
                mbar_wait_cluster(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
                tc_fence_after();
                for (uint32_t ks = 0; ks < ti.kst; ++ks) {
                    const uint32_t kin = ks % SPC2;
                    if (kin == 0) {
                        mbar_wait_cluster(&b_full[bs], bph);
                        tc_fence_after();
                    }
                    mbar_wait_cluster(&a_full[as], aph);
                    tc_fence_after();
                    const uint32_t abase = smem_u32(abuf + as * A2_BYTES);
                    const uint32_t cbase = smem_u32(chunks + bs * CHUNK2_BYTES);
                    if (elect_one()) {
                        if constexpr (FP4) {
#pragma unroll
                            for (uint32_t kk = 0; kk < KS2 / 64; ++kk) {
                                // A: core matrix (row group g, K group q of 32) at g*A2_SBO + q*128
                                const uint64_t adesc = desc_kmajor(abase + kk * 256, 128, A2_SBO);
                                const uint32_t koff = kin * KS2 + kk * 64;
                                const uint64_t bdesc = desc_kmajor(cbase + (koff / 8) * 128, 512, 128);
                                mma2_mxf4_ss(tmem + acc, adesc, bdesc, idesc, tmem + SF2_COL, tmem + SF2_COL + 8,
                                             (ks | kk) != 0);
                            }
                        } else {
#pragma unroll
                            for (uint32_t kk = 0; kk < 4; ++kk) {
                                // A: core matrix (row group g, K chunk q) at g*1024 + q*128: SBO 1024, LBO 128
                                const uint64_t adesc = desc_kmajor(abase + kk * 2 * 128, 128, 1024);
                                const uint32_t koff = kin * KS + kk * 32;
                                const uint64_t bdesc = desc_kmajor(cbase + (koff / 8) * 128, 256, 128);
                                mma2_i8_ss(tmem + acc, adesc, bdesc, idesc, (ks | kk) != 0);
                            }
                        }
                        mma2_commit_both(&a_empty[as]);
                        if (kin == SPC2 - 1 || ks == ti.kst - 1) mma2_commit_both(&b_empty[bs]);
                    }
                    __syncwarp();
                    if (++as == A2_STAGES) { as = 0; aph ^= 1; }
                    if (kin == SPC2 - 1 || ks == ti.kst - 1) {
                        if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
                    }
                }
                if (elect_one()) mma2_commit_both(&acc_full[ab]);
                __syncwarp();
            }
        } else if (rank == 1 && lane == 0) {
            // relay: the peer's transform warps arrive on a_local (CTA scope, no
            // memory barrier); this thread, which has no loads in flight, forwards
            // each completed stage to the leader's a_full with one cluster-release arrive
            uint32_t g = 0;
            for (uint32_t t = pair; t < ntiles; t += npairs_grid) {
                const Tile2 ti = tile2_info<GROUPED>(a, seed_s, t, cur);
                for (uint32_t ks = 0; ks < ti.kst; ++ks, ++g) {
                    mbar_wait(&a_local[g % A2_STAGES], (g / A2_STAGES) & 1);
                    mbar_arrive_rank(&a_full[g % A2_STAGES], 0);
                }
            }
        }
        __syncwarp();
    } else if (warp >= W2_BGEN0 && warp < W2_BGEN0 + N2_BGEN) {
        // this CTA's half of the B tile: rows n0 + rank*ntile/2 .. + ntile/2
        const int tb = (warp - W2_BGEN0) * 32 + lane;
        uint32_t bs = 0, bph = 0;
        for (uint32_t t = pair; t < ntiles; t += npairs_grid) {
            const Tile2 ti = tile2_info<GROUPED>(a, seed_s, t, cur);
            const uint32_t half = ti.ntile / 2;
            const int ncm = KC / 8 + (int)(half / 8) - 1;
            for (uint32_t c = 0; c < ti.nchunks; ++c) {
                const uint32_t base = ti.n0 + rank * half + c * KC;
                mbar_wait(&b_empty[bs], bph ^ 1);
                uint8_t *cb = chunks + bs * CHUNK2_BYTES;
                for (int r = tb; r < ncm * 8; r += N2_BGEN * 32) {
                    const uint32_t p = base + 8 * (r >> 3) + (r & 7);
                    uint32_t w0, w1;
                    if (GROUPED) { w0 = __ldg(ti.seed + (p >> 5)); w1 = __ldg(ti.seed + (p >> 5) + 1); }
                    else { w0 = ti.seed[p >> 5]; w1 = ti.seed[(p >> 5) + 1]; }
                    const uint32_t v = __funnelshift_l(w1, w0, p & 31);
                    uint4 o;
                    if constexpr (FP4) {
                        o = e2m1_row(v);
                    } else {
                        o.x = prmt_sign<0xFEBA>(v << 7, v << 6);
                        o.y = prmt_sign<0xFEBA>(v << 5, v << 4);
                        o.z = prmt_sign<0xFEBA>(v << 3, v << 2);
                        o.w = prmt_sign<0xFEBA>(v << 1, v);
                    }
                    *reinterpret_cast<uint4 *>(cb + (r >> 3) * 128 + (r & 7) * 16) = o;
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive_rank(&b_full[bs], 0);
                if (++bs == B_SLOTS) { bs = 0; bph ^= 1; }
            }
        }
    } else if (warp >= W2_XF0 && warp < W2_XF0 + N2_XF) {
        // A transform into shared memory: row = block (this CTA's 128 of the
        // tile's 256), 128 K per stage, chunk G (16 K-bytes) of row r goes to
        // core matrix (r/8, G): offset (r/8)*1024 + G*128 + (r%8)*16.
        const uint32_t xw = (uint32_t)(warp - W2_XF0), par = xw / 4;
        const uint32_t row = (xw & 3) * 32 + lane;
        uint32_t lcur = 0, lt = pair, lks = 0;
        Tile2 lti{};
        if (lt < ntiles) lti = tile2_info<GROUPED>(a, seed_s, lt, lcur);
        auto step1 = [&]() {
            if (lt >= ntiles) return;
            if (++lks == lti.kst) {
                lks = 0;
                lt += npairs_grid;
                if (lt < ntiles) lti = tile2_info<GROUPED>(a, seed_s, lt, lcur);
            }
        };
        // K reversed: stage lks, part hf (128 K each) is 128-bit chunk
        // k128 - 1 - KS2_128 lks - hf of the block row (zeros before the row start)
        auto load = [&](bool &v, uint32_t hf) -> uint4 {
            const uint64_t b = (uint64_t)lti.mt * BM2 + rank * BH + row;
            const int32_t ci = (int32_t)lti.k128 - 1 - (int32_t)(KS2_128 * lks + hf);
            v = lt < ntiles && b < a.n_blocks && ci >= 0;
            const uint64_t bc = b < a.n_blocks ? b : a.n_blocks - 1;
            return __ldg(reinterpret_cast<const uint4 *>(lti.xb + bc * lti.xs) + (ci >= 0 ? ci : 0));
        };
        for (uint32_t i = 0; i < par; ++i) step1();
        uint4 pf[PF2][KS2_128];
        bool ok[PF2], vd[PF2][KS2_128];
#pragma unroll
        for (int j = 0; j < PF2; ++j) {
            ok[j] = lt < ntiles;
#pragma unroll
            for (int hf = 0; hf < KS2_128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
#pragma unroll
            for (int i = 0; i < XF2_PAR; ++i) step1();
        }
        uint32_t g = par;
        bool more = true;
        while (more) {
#pragma unroll
            for (int j = 0; j < PF2; ++j) {
                if (more && !ok[j]) more = false;
                if (more) {
                    const uint4 cur4 = vd[j][0] ? pf[j][0] : make_uint4(0, 0, 0, 0);
                    const uint32_t as = g % A2_STAGES, aph = (g / A2_STAGES) & 1;
                    mbar_wait(&a_empty[as], aph ^ 1);
                    if constexpr (FP4) {
                        // 16 core-matrix rows of 32 E2M1 elements: K group gk of the stage is
                        // word 3 - (gk & 3) of 128-bit part gk / 4 (same slot order as B)
                        uint8_t *dst = abuf + as * A2_BYTES + (row >> 3) * A2_SBO + (row & 7) * 16;
#pragma unroll
                        for (int hf = 0; hf < KS2_128; ++hf) {
                            const uint4 c4 = vd[j][hf] ? pf[j][hf] : make_uint4(0, 0, 0, 0);
                            const uint32_t M4[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                *reinterpret_cast<uint4 *>(dst + (hf * 4 + q) * 128) =
                                    e2m1_row(__brev(__byte_perm(M4[3 - q], 0, 0x0123)));
                        }
                    } else {
                    // expand the 16 raw bytes (same K order as the 1-SM kernel's TMEM stage)
                    const uint32_t M[4] = {cur4.x, cur4.y, cur4.z, cur4.w};
                    uint8_t *dst = abuf + as * A2_BYTES + (row >> 3) * 1024 + (row & 7) * 16;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t S[8];
#pragma unroll
                        for (int b2 = 0; b2 < 8; ++b2) S[b2] = M[q] << b2;
                        const int G0 = 2 * (3 - q);
                        uint4 lo, hi;
                        lo.x = prmt_sign<0xFEBA>(S[0], S[1]);
                        lo.y = prmt_sign<0xFEBA>(S[2], S[3]);
                        lo.z = prmt_sign<0xFEBA>(S[4], S[5]);
                        lo.w = prmt_sign<0xFEBA>(S[6], S[7]);
                        hi.x = prmt_sign<0xDC98>(S[0], S[1]);
                        hi.y = prmt_sign<0xDC98>(S[2], S[3]);
                        hi.z = prmt_sign<0xDC98>(S[4], S[5]);
                        hi.w = prmt_sign<0xDC98>(S[6], S[7]);
                        *reinterpret_cast<uint4 *>(dst + G0 * 128) = lo;
                        *reinterpret_cast<uint4 *>(dst + (G0 + 1) * 128) = hi;
                    }
                    }
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(rank == 0 ? &a_full[as] : &a_local[as]);
                    // refill this ring slot after the arrive
                    ok[j] = lt < ntiles;
#pragma unroll
                    for (int hf = 0; hf < KS2_128; ++hf) pf[j][hf] = load(vd[j][hf], hf);
#pragma unroll
                    for (int i = 0; i < XF2_PAR; ++i) step1();
                    g += XF2_PAR;
                }
            }
        }
    } else {
        // Epilogue: group ab = (w - W2_EPI0) / 4 drains accumulator set ab (tiles
        // k = ab mod 2 of this pair); warp % 4 = TMEM lane quadrant.
        const uint32_t ab = (uint32_t)(warp - W2_EPI0) >> 2;
        const uint32_t row = (uint32_t)(warp & 3) * 32 + lane;
        const uint32_t lane_addr = tmem + (((uint32_t)(warp & 3) * 32) << 16) + ab * BN2;
        uint32_t it = 0;
        for (uint32_t t = pair + ab * npairs_grid; t < ntiles; t += 2 * npairs_grid, ++it) {
            const Tile2 ti = tile2_info<GROUPED>(a, seed_s, t, cur);
            mbar_wait(&acc_full[ab], it & 1);
            tc_fence_after();
            constexpr int NW2 = (BN2 + 31) / 32;
            uint32_t words[NW2];
#pragma unroll
            for (int c = 0; c < NW2; ++c) {
                uint32_t w = 0;
                if ((uint32_t)(32 * c) < ti.ntile) {
                    uint32_t v[32];
                    tmem_ld32(lane_addr + 32 * c, v);  // FP4: the last load runs past BN2 (masked below)
                    tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 32; ++k)
                        w = (w << 1) | (FP4 ? (__float_as_uint(__uint_as_float(v[k]) + 8388608.0f) & 1u) : (v[k] & 1u));
                }
                words[c] = w;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_rank(&acc_empty[ab], 0);
            const uint64_t b = (uint64_t)ti.mt * BM2 + rank * BH + row;
            const uint32_t n0 = ti.n0;
            if (b >= a.n_blocks || n0 >= ti.r) continue;
            const uint32_t nvalid = min(min((uint32_t)BN2, ti.ntile), ti.r - n0);
#pragma unroll
            for (int c = 0; c < NW2; ++c) {
                const int vb = (int)nvalid - 32 * c;
                if (vb <= 0) words[c] = 0;
                else if (vb < 32) words[c] &= ~(0xFFFFFFFFu >> vb);
            }
            if (GROUPED) {
                uint32_t *dst = a.yws + b * a.y_stride + ti.out_off + n0 / 32;
#pragma unroll
                for (int c = 0; c < NW2; ++c)
                    if ((uint32_t)(32 * c) < nvalid) dst[c] = words[c];
                continue;
            }
            const uint64_t G_lo = b * a.m + n0, G_hi = G_lo + nvalid;
            const uint32_t off = (uint32_t)(G_lo & 31);
            const uint64_t W0 = G_lo >> 5;
            uint32_t prev = 0;
#pragma unroll
            for (int c = 0; c <= NW2; ++c) {
                const uint32_t cw = (c < NW2) ? words[c] : 0u;
                const uint32_t ow = off ? ((prev << (32 - off)) | (cw >> off)) : cw;
                prev = cw;
                const uint64_t W = W0 + c;
                if (W * 32 >= G_hi) break;
                const bool excl = (W * 32 >= G_lo) && (W * 32 + 32 <= G_hi);
                emit_word(a.out, W, ow, excl);
            }
        }
    }

    tc_fence_before();
    cluster_sync();  // the leader's last MMAs (which read this CTA's smem) are complete
    if (warp == W2_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
    }
}

static size_t smem_bytes2(uint32_t seed_words_n) {
    return (size_t)A2_STAGES * A2_BYTES + (size_t)B_SLOTS * CHUNK2_BYTES + ((seed_words_n + 3) & ~3u) * 4 +
           (3 * A2_STAGES + 2 * B_SLOTS + 4) * 8 + 16;
}

template <bool GROUPED>
static qrng_status launch2(Args a, cudaStream_t s) {
    // tiles of 256 blocks x 256 rows; a.n_npairs counts 256-row N tiles
    a.n_mtiles = (uint32_t)((a.n_blocks + BM2 - 1) / BM2);
    if ((uint64_t)a.n_mtiles * a.n_npairs > 0xFFFFFFFFull) {
        set_error("GEMM path: too many tiles");
        return QRNG_E_UNSUPPORTED;
    }
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = smem_bytes2(GROUPED ? 0u : a.seed_words_n);
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(toeplitz_gemm2_kernel<GROUPED>));
        if (st != QRNG_OK) return st;
    }
    const uint32_t ntiles = a.n_mtiles * a.n_npairs;
    const uint32_t pairs = std::min<uint32_t>(ntiles, (uint32_t)sms / 2);
    KernelTimer tm(s, true);
    toeplitz_gemm2_kernel<GROUPED><<<2 * pairs, NTHREADS2, smem, s>>>(a);
    tm.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}
}  // namespace two
#endif

// ---- MMA-rate microbenchmark (profiling only) ---------------------------------------
// One elected thread per CTA issues `iters` back-to-back int8 MMAs on fixed
// operands (no data movement): form 0 = cta_group::1, A in TMEM, M128 N=n;
// form 1 = cta_group::1, A in SMEM, M128 N=n; form 2 = cta_group::2 (cluster
// pair), A in SMEM, M256 N=n.  Time it with CUDA events; MACs = CTAs x iters x
// (M/ctas) x N x 32.
template <int FORM>
__global__ void __cluster_dims__(FORM == 2 ? 2 : 1, 1, 1) __launch_bounds__(128, 1)
    mma_rate_kernel(int iters, int n, uint32_t *sink, int commit_every) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t &bar = *reinterpret_cast<uint64_t *>(smem + 64 * 1024);
    uint32_t &slot = *reinterpret_cast<uint32_t *>(smem + 64 * 1024 + 16);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (FORM == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc(&slot, 512);
        }
    }
    tc_fence_before();
#if QRNG_GEMM_2CTA
    if (FORM == 2) two::cluster_sync(); else __syncthreads();
#else
    __syncthreads();
#endif
    tc_fence_after();
    const uint32_t tmem = slot;
    uint32_t rank = 0;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (warp == 0 && rank == 0) {  // converged warp, elected issue (as in the kernels)
        const uint32_t idesc = idesc_i8(FORM == 2 ? 256 : 128, n);
        const uint64_t bdesc = desc_kmajor(smem_u32(smem), 256, 128);
        const uint64_t adesc = desc_kmajor(smem_u32(smem + 32768), 128, 1024);
        if (FORM == 4 || FORM == 5) {
            // kind::mxf4 (E2M1, both operands in shared memory, unit scales in TMEM
            // columns [448, 464)): form 4 = back-to-back M128 N=n K64; form 5 = the
            // stage shape, 2 K64 steps x two N tiles (N0 = n & 511, N1 = n >> 9)
            const uint32_t n0 = n & 511, n1 = (n >> 9) ? (n >> 9) : n0;
            const uint32_t id0 = idesc_mxf4(128, n0), id1 = idesc_mxf4(128, n1);
            const uint32_t cb = smem_u32(smem);
            for (int it = 0; it < iters; ++it) {
                if (elect_one()) {
                    if (FORM == 4) {
                        mma_mxf4_ss(tmem + 128, desc_kmajor(cb + 32768, 128, 1024), desc_kmajor(cb, 512, 128), id0,
                                    tmem + 448, tmem + 456, 1);
                    } else {
#pragma unroll
                        for (uint32_t kk = 0; kk < 2; ++kk) {
                            const uint64_t ad = desc_kmajor(cb + 32768 + (it & 3) * 2048 + kk * 256, 128, 512);
                            mma_mxf4_ss(tmem, ad, desc_kmajor(cb + ((it & 3) * 16 + kk * 8) * 128, 512, 128), id0,
                                        tmem + 448, tmem + 456, 1);
                            mma_mxf4_ss(tmem + 192, ad, desc_kmajor(cb + ((it & 3) * 16 + kk * 8 + 24) * 128, 512, 128),
                                        id1, tmem + 448, tmem + 456, 1);
                        }
                        mma_commit(&bar + 1);
                    }
                }
                __syncwarp();
            }
        } else
        if (FORM == 3) {
            // the kernels' stage shape: 4 K32 steps x 2 N tiles (N0 = n & 511,
            // N1 = n >> 9) and one commit per stage, runtime descriptors
            const uint32_t n0 = n & 511, n1 = (n >> 9) ? (n >> 9) : n0;
            const uint32_t id0 = idesc_i8(128, n0), id1 = idesc_i8(128, n1);
            const uint32_t cb = smem_u32(smem);
            for (int it = 0; it < iters; ++it) {
                if (elect_one()) {
#pragma unroll
                    for (uint32_t kk = 0; kk < 4; ++kk) {
                        const uint32_t koff = (it & 3) * 128 + kk * 32;
                        mma_i8_ts(tmem + 128, tmem + (it & 3) * 32 + kk * 8,
                                  desc_kmajor(cb + (koff / 8) * 128, 256, 128), id0, 1);
                        mma_i8_ts(tmem + 128 + 192, tmem + (it & 3) * 32 + kk * 8,
                                  desc_kmajor(cb + (koff / 8 + 24) * 128, 256, 128), id1, 1);
                    }
                    mma_commit(&bar + 1);
                }
                __syncwarp();
            }
        } else
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
                if (commit_every > 0 && it % commit_every == commit_every - 1) {
                    if (FORM == 2)
                        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar + 1)), "h"((uint16_t)3) : "memory");
                    else
                        mma_commit(&bar + 1);
                }
                if (FORM == 0) mma_i8_ts(tmem + 256, tmem, bdesc, idesc, 1);
                else if (FORM == 1)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
                                 "l"(adesc), "l"(bdesc), "r"(idesc) : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
                                 "l"(adesc), "l"(bdesc), "r"(idesc) : "memory");
            }
            __syncwarp();
        }
        __syncwarp();
        if (elect_one()) {
            if (FORM == 2)
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
            else
                mma_commit(&bar);
        }
        __syncwarp();
    }
    if (FORM == 2 || rank == 0) {
        if (threadIdx.x == 0) mbar_wait(&bar, 0);
    }
    tc_fence_before();
#if QRNG_GEMM_2CTA
    if (FORM == 2) two::cluster_sync(); else __syncthreads();
#else
    __syncthreads();
#endif
    if (warp == 0) {
        tc_fence_after();
        if (FORM == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
        else tmem_dealloc(tmem, 512);
    }
    if (threadIdx.x == 0 && iters < 0) sink[0] = tmem;
}

qrng_status mma_rate(int form, int iters, int n, uint64_t *macs, cudaStream_t s) {
    const int commit_every = form / 16;  // form + 16*k: a commit every k MMAs
    form %= 16;
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = 64 * 1024 + 64;
    const unsigned grid = (unsigned)sms;
    count_launch();
    switch (form) {
        case 0: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<0>)); mma_rate_kernel<0><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 1: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<1>)); mma_rate_kernel<1><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 3: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<3>)); mma_rate_kernel<3><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 4: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<4>)); mma_rate_kernel<4><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 5: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<5>)); mma_rate_kernel<5><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
#if QRNG_GEMM_2CTA
        case 2: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<2>)); mma_rate_kernel<2><<<grid & ~1u, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
#endif
        default: set_error("mma_rate: unsupported form"); return QRNG_E_UNSUPPORTED;
    }
    QRNG_CUDA_TRY(cudaGetLastError());
    if (form == 3)
        *macs = (uint64_t)grid * iters * 4ull * 128ull * (uint64_t)((n & 511) + ((n >> 9) ? (n >> 9) : (n & 511))) * 32ull;
    else if (form == 4)
        *macs = (uint64_t)grid * iters * 128ull * (uint64_t)n * 64ull;
    else if (form == 5)
        *macs = (uint64_t)grid * iters * 2ull * 128ull * (uint64_t)((n & 511) + ((n >> 9) ? (n >> 9) : (n & 511))) * 64ull;
    else
        *macs = (uint64_t)(form == 2 ? (grid & ~1u) : grid) * (uint64_t)iters * 128ull * (uint64_t)n * 32ull;
    return QRNG_OK;
}

// ---- layout probe (test only): D = A * B^T with B[i][k] = h[i + k] ----------------
// One CTA, 128 threads.  A: 128 x K int8 row-major (global); h: bytes; D: 128 x N s32.
__global__ void __launch_bounds__(128, 1) umma_probe_kernel(const uint8_t *A, const uint8_t *h, int32_t *D, int N,
                                                           int K) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 8);
    uint8_t *cm = smem + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int ncm = K / 8 + N / 8 - 1;
    for (int r = tid; r < ncm * 8; r += 128) {
        int tau = r >> 3, rr = r & 7;
        for (int c = 0; c < 16; ++c) cm[tau * 128 + rr * 16 + c] = h[8 * tau + rr + c];
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    // A row tid -> TMEM lane tid, columns [0, K/4)
    for (int c0 = 0; c0 < K / 4; c0 += 32) {
        uint32_t v[32];
        for (int c = 0; c < 32; ++c) {
            uint32_t w = 0;
            for (int e = 0; e < 4; ++e) w |= (uint32_t)A[tid * K + 4 * (c0 + c) + e] << (8 * e);
            v[c] = w;
        }
        tmem_st32(lane_addr + c0, v);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        const uint32_t idesc = idesc_i8(128, N, false);  // probe: U8 x U8
        for (int k = 0; k < K; k += 32) {
            const uint64_t bdesc = desc_kmajor(smem_u32(cm) + (k / 8) * 128, 256, 128);
            mma_i8_ts(tmem + 256, tmem + k / 4, bdesc, idesc, k != 0);
        }
        mma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(lane_addr + 256 + c0, v);
        tmem_wait_ld();
        for (int c = 0; c < 32 && c0 + c < N; ++c) D[tid * N + c0 + c] = (int32_t)v[c];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---- FP4 (kind::mxf4) probe (test only) ------------------------------------------
// E2M1 operands, 0 -> 0x0 and 1 -> 0x2 (1.0), two per byte (`hi_first`: element
// 2i in the high nibble), unit block scales (UE8M0 127 = 2^0) in a TMEM region
// filled with 0x7F, FP32 accumulation.  D = A * B^T, B[i][k] = h[i + k] through
// the same overlapping core-matrix windows as the int8 B operand (a core-matrix
// row now holds 32 elements, so the K-direction byte offset LBO is 4 x 128).
__device__ __forceinline__ uint8_t pack_e2m1(uint8_t lo_elem, uint8_t hi_elem, bool hi_first) {
    const uint8_t a = lo_elem ? 2 : 0, b = hi_elem ? 2 : 0;  // element 2i, element 2i + 1
    return hi_first ? (uint8_t)((a << 4) | b) : (uint8_t)((b << 4) | a);
}
__global__ void __launch_bounds__(128, 1) mxf4_probe_kernel(const uint8_t *A, const uint8_t *h, float *D, int N,
                                                           int K, int hi_first) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem);
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 8);
    uint8_t *acm = smem + 1024;                   // A: core matrix (rg, kg) at (rg * K/32 + kg) * 128
    uint8_t *bcm = acm + 128 * (K / 2);           // B windows: core matrix tau row rr = h[8 tau + rr + c], c < 32
    const int warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int ncm = K / 8 + N / 8 - 1;
    for (int r = tid; r < ncm * 8; r += 128) {
        const int tau = r >> 3, rr = r & 7;
        for (int c = 0; c < 16; ++c)
            bcm[tau * 128 + rr * 16 + c] = pack_e2m1(h[8 * tau + rr + 2 * c], h[8 * tau + rr + 2 * c + 1], hi_first);
    }
    for (int kg = 0; kg < K / 32; ++kg)
        for (int c = 0; c < 16; ++c) {
            const int r = tid;
            acm[((r >> 3) * (K / 32) + kg) * 128 + (r & 7) * 16 + c] =
                pack_e2m1(A[r * K + kg * 32 + 2 * c], A[r * K + kg * 32 + 2 * c + 1], hi_first);
        }
    if (tid == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    {
        uint32_t v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = 0x7F7F7F7Fu;
        tmem_st16(lane_addr + 256, v);  // scale-factor region, columns [256, 272)
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        if (elect_one()) {
            const uint32_t idesc = idesc_mxf4(128, N);
            for (int k = 0; k < K; k += 64) {
                const uint64_t adesc = desc_kmajor(smem_u32(acm) + (k / 32) * 128, 128, (K / 32) * 128);
                const uint64_t bdesc = desc_kmajor(smem_u32(bcm) + (k / 8) * 128, 512, 128);
                mma_mxf4_ss(tmem, adesc, bdesc, idesc, tmem + 256, tmem + 264, k != 0);
            }
            mma_commit(bar);
        }
        __syncwarp();
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(lane_addr + c0, v);
        tmem_wait_ld();
        for (int c = 0; c < 32 && c0 + c < N; ++c) D[tid * N + c0 + c] = __uint_as_float(v[c]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int operand_bits() { return FP4 ? 4 : 8; }

qrng_status mxf4_probe(const uint8_t *A, const uint8_t *h, float *D, int N, int K, int hi_first, cudaStream_t s) {
    if (N < 16 || N > 256 || N % 16 || K < 64 || K > 1024 || K % 64) {
        set_error("mxf4 probe: N in [16, 256] multiple of 16, K in [64, 1024] multiple of 64");
        return QRNG_E_INVALID;
    }
    const size_t smem = 1024 + 128 * (K / 2) + (size_t)(K / 8 + N / 8) * 128;
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(mxf4_probe_kernel));
        if (st != QRNG_OK) return st;
    }
    count_launch();
    mxf4_probe_kernel<<<1, 128, smem, s>>>(A, h, D, N, K, hi_first);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
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
    // 2-SM kernel: 256-row tiles, the second CTA's half starts 128 rows later
    const uint64_t T2 = QRNG_GEMM_FP4 ? 224 : 256;  // 2-SM tile rows (kTileRows of a -DQRNG_GEMM_2CTA build)
    const uint64_t nt2 = (m + T2 - 1) / T2, pmax2 = (nt2 - 1) * T2 + T2 / 2 + (nchunks - 1) * KC + 8 * (KC / 8 + T2 / 16 - 1) + 7;
    if (pmax2 > pmax) pmax = pmax2;
    return (uint32_t)(pmax / 32 + 2);
}

static size_t smem_bytes(uint32_t seed_words_n) {
    return (size_t)B_SLOTS * CHUNK_BYTES + (FP4 ? (size_t)A_STAGES * A_STAGE_BYTES : 0) + ((seed_words_n + 3) & ~3u) * 4 + (2 * A_STAGES + 2 * B_SLOTS + ACC_FULL + ACC_EMPTY) * 8 + 16;
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

template <bool GROUPED, bool PACKED = false>
static qrng_status launch(const Args &a, cudaStream_t s) {
    if ((uint64_t)a.n_mtiles * a.n_npairs > 0xFFFFFFFFull) {
        set_error("GEMM path: too many tiles");
        return QRNG_E_UNSUPPORTED;
    }
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t smem = smem_bytes(GROUPED ? a.n_leaves * 8u : a.seed_words_n);
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(toeplitz_gemm_kernel<GROUPED, PACKED>));
        if (st != QRNG_OK) return st;
    }
    const uint32_t ntiles = a.n_mtiles * a.n_npairs;
    const unsigned grid = (unsigned)(ntiles < (uint32_t)sms ? ntiles : (uint32_t)sms);
    KernelTimer tm(s, true);
    if (GROUPED) {
        const cudaError_t e = launch_pdl(toeplitz_gemm_kernel<GROUPED, PACKED>, dim3(grid), dim3(NTHREADS), smem, s, a);
        if (e != cudaSuccess) { set_error("grouped GEMM launch: %s", cudaGetErrorString(e)); return QRNG_E_CUDA; }
    } else {
        toeplitz_gemm_kernel<GROUPED, PACKED><<<grid, NTHREADS, smem, s>>>(a);
    }
    tm.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
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
    a.n_npairs = (uint32_t)((m + NT * BN - 1) / (NT * BN));  // work tile t = (N pair t / n_mtiles, M tile t % n_mtiles)
    a.seed_words = pl.seed_words;
    a.seed_words_n = (uint32_t)pl.seed_words_n;
    a.out = out;
#if QRNG_GEMM_2CTA
    a.n_npairs = (uint32_t)((m + kTileRows - 1) / kTileRows);
    return two::launch2<false>(a, s);
#else
    return launch<false>(a, s);
#endif
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
#if QRNG_GEMM_2CTA
    (void)max_leaf_w;
    return two::launch2<true>(a, s);
#else
    static const bool packed_ok = [] {
        const char *e = getenv("QRNG_GEMM_PACKED");
        return e ? atoi(e) != 0 : true;
    }();
    if constexpr (PACK_OK) {
        if (packed_ok && max_leaf_w <= kMaxPackedK) return launch<true, true>(a, s);
    }
    return launch<true, false>(a, s);
#endif
}

qrng_status trace(uint64_t *h_out, int reset) {
#ifdef QRNG_GEMM_TRACE
    QRNG_CUDA_TRY(cudaDeviceSynchronize());
    QRNG_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_trace, sizeof(g_trace)));
    if (reset) {
        unsigned long long z[32] = {};
        QRNG_CUDA_TRY(cudaMemcpyToSymbol(g_trace, z, sizeof z));
    }
    return QRNG_OK;
#else
    (void)h_out;
    (void)reset;
    set_error("built without -DQRNG_GEMM_TRACE");
    return QRNG_E_UNSUPPORTED;
#endif
}

qrng_status probe(const uint8_t *A, const uint8_t *h, int32_t *D, int N, int K, cudaStream_t s) {
    if (N < 16 || N > 256 || N % 16 || K < 32 || K % 128) {
        set_error("probe: N in [16,256] step 16, K multiple of 128");
        return QRNG_E_INVALID;
    }
    const size_t smem = 1024 + (size_t)(K / 8 + N / 8 - 1) * 128;
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(umma_probe_kernel));
        if (st != QRNG_OK) return st;
    }
    count_launch();
    umma_probe_kernel<<<1, 128, smem, s>>>(A, h, D, N, K);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
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
