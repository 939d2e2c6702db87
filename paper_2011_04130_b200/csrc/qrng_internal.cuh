// qrng_internal.cuh -- internal declarations shared by the libqrng.so sources.
// Product code (sm_100a).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <memory>
#include <cuda_runtime.h>
#include "../../include/qrng.h"

namespace qrng {

// Thread-local error message (qrng_last_error).
void set_error(const char *fmt, ...);

#define QRNG_CUDA_TRY(expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            ::qrng::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                              __FILE__, __LINE__);                                   \
            return QRNG_E_CUDA;                                                      \
        }                                                                            \
    } while (0)

// Opt a kernel into the full 227 KB of dynamic shared memory on the current
// device (once per kernel per device; a process may drive several GPUs).
qrng_status allow_max_smem(const void *func);

// Second stream of the calling thread (per device) plus a fork and a join
// event: multi-pass NTT batches and Karatsuba block chunks alternate between
// the caller's stream and this one so one batch's kernels fill the SMs another
// batch leaves idle.
qrng_status side_stream(cudaStream_t *s2, cudaEvent_t *fork, cudaEvent_t *join);

// Launch accounting / optional per-kernel event timing (qrng_debug_*).
void count_launch();
struct KernelTimer {  // brackets one kernel on its stream (counts every launch)
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    int channel;             // 0: main extraction kernel(s); 1: auxiliary (Karatsuba Q buffers, combine/pack)
    KernelTimer(cudaStream_t st, bool timed, int channel = 0);
    void stop();
};

// ---------------------------------------------------------------------------
// Output bit stream helpers (convention C4: block b's y_i is bit b*m+i,
// MSB-first).  Kernels build "logical big-endian" 32-bit words: global bit g
// sits at position 31-(g&31) of logical word g>>5; memory word = bswap(logical).
struct OutStream {
    uint32_t *words;        // d_out viewed as uint32 (16-byte aligned by contract)
    uint64_t total_bits;    // n_blocks * m
    uint64_t full_words;    // words entirely inside the out buffer (bytes/4)
    uint32_t *tail;         // scratch word for a final partial word (may be null)
};

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Programmatic dependent launch: a kernel launched with launch_pdl() may start
// (prologue) while the previous kernel in the stream finishes; pdl_wait() blocks
// until that kernel has completed and its memory is visible.  pdl_release()
// lets the next PDL-launched kernel be scheduled early.
__device__ __forceinline__ void pdl_wait() {
#ifndef QRNG_NO_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_release() {
#ifndef QRNG_NO_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifdef QRNG_NO_PDL
    cfg.numAttrs = 0;  // plain stream order
#else
    cfg.numAttrs = 1;
#endif
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Write logical word W.  `exclusive` = every bit of W belongs to the caller.
__device__ __forceinline__ void emit_word(const OutStream &o, uint64_t W, uint32_t logical,
                                          bool exclusive) {
    if (W >= o.full_words) {  // partial final word -> scratch, copied by the host afterwards
        if (logical) atomicOr(o.tail, bswap32(logical));
        return;
    }
    if (exclusive) o.words[W] = bswap32(logical);
    else if (logical) atomicOr(&o.words[W], bswap32(logical));
}

// ---------------------------------------------------------------------------
// NTT path (ntt.cu).  Prime p = 119 * 2^23 + 1, primitive root 3.
namespace ntt {
constexpr uint32_t kP = 998244353u;
constexpr uint32_t kP2 = 469762049u;  // 7 * 2^26 + 1: the distributed (NEXT-4) transforms, P up to 2^26
constexpr uint32_t kP3 = 167772161u;  // 5 * 2^25 + 1: third prime of the packed three-prime form
constexpr int kMaxLogP = 23;
constexpr int kMaxLogP2 = 26;
constexpr int kMaxFusedLogP = 15;  // one CTA holds the whole transform in smem

struct Plan {
    int logP = 0;
    uint32_t len = 0;            // raw bits per block entering the product
    bool xor_tail = false;       // modified Toeplitz identity block
    int pack_shift = 0;          // >0: two blocks share one transform (x1 + 2^shift x2)
    int field = 0;               // 0: p = kP (P <= 2^23); 1: p = kP2 (2^23 < P <= 2^26, multi-pass)
    uint32_t *shat = nullptr;    // P words: NTT(seed) * P^-1 * 2^32 mod p, DIF order
    uint32_t *tw = nullptr;      // P words: w_P^e * 2^32 mod p
    uint32_t *itw = nullptr;     // P words: w_P^-e * 2^32 mod p
    uint2 *l1tw = nullptr;       // multi-pass: the segment kernel's level-1 twiddles in Shoup form (ntt.cu)
    uint32_t *work = nullptr;    // multipass scratch (not used by the fused kernel)
    size_t work_words = 0;
    // packed three-prime form (multi-pass, n < 2^21): crt blocks share one
    // transform per prime as sum_g 2^(crt_k g) x_g; the key bits come back by
    // CRT (ntt.cu "Packed three-prime form").  0: one block per transform.
    int crt = 0;
    uint32_t crt_k = 0;
    uint32_t *shat3[3] = {}, *tw3[3] = {}, *itw3[3] = {};  // per prime kP, kP2, kP3
    uint2 *l1tw3[3] = {};
};
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t seed_bit_offset,
                      bool xor_tail, cudaStream_t s);
void plan_free(Plan &pl);
// n = block stride in bits (the product uses the plan's len bits of each block)
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                    uint64_t m, const OutStream &out, cudaStream_t s);
int choose_pack_shift(uint64_t n, int logP);
// NEXT-4: one block across `world` GPUs, distributed four-step NTT with the
// prime kP2 (P = world * N2 <= 2^26).  See ntt.cu "NEXT-4".
struct DistPlan {
    uint64_t n = 0, m = 0;
    uint32_t world = 1, rank = 0;
    int logP = 0, logN2 = 0;
    uint32_t N2 = 0;                   // local transform length = words exchanged per rank
    uint32_t colw[8] = {};             // w_W^(n1 rank), canonical
    uint32_t icolM[8][8] = {};         // w_W^(-n1 k1), Montgomery form
    uint32_t *shat = nullptr;          // seed spectrum slice k1 = rank (N2 words, scaled by P^-1, Montgomery)
    uint32_t *tw = nullptr, *itw = nullptr;    // w_N2^(+-e), e < N2 (Montgomery)
    uint32_t *twr = nullptr, *itwr = nullptr;  // w_P^(+-n2 rank) (null for rank 0)
};
qrng_status dist_plan_init(DistPlan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t world,
                           uint32_t rank, cudaStream_t s);
void dist_plan_free(DistPlan &pl, cudaStream_t s, bool async);
// column DFT of the block bits for k1 = rank, local NTT, * S^, inverse, twist:
// d_buf (N2 words) = this rank's send buffer, chunk r' for peer r'
qrng_status dist_local(const DistPlan &pl, const uint8_t *d_block_bits, uint32_t *d_buf, cudaStream_t s);
// after the all-to-all: radix-W inverse across the received chunks, window
// parities ORed into `out` at global bit g0 + i (out pre-zeroed)
qrng_status dist_finish(const DistPlan &pl, const uint32_t *d_recv, const OutStream &out, uint64_t g0,
                        cudaStream_t s);
qrng_status butterfly_rate(int iters, uint64_t *butterflies, cudaStream_t s, bool with_twiddles);
}  // namespace ntt

// GEMM path (gemm_tc.cu): tcgen05 kind::mxf4 batched Toeplitz product.
namespace gemm {
struct Plan {
    uint32_t *seed_words = nullptr;  // seed as logical big-endian words, zero padded
    uint32_t seed_words_n = 0;
};
// One leaf product of the Karatsuba decomposition (karatsuba.cu): an r x w
// Toeplitz product applied to every block, run as a group of tiles of the
// same tcgen05 kernel.  Device-resident table entry.
struct Leaf {
    uint32_t w, r;              // K (input bits) and output rows; w % 128 == 0
    uint32_t npairs, npair_base;  // N pairs (NT*BN rows) of this leaf; prefix over leaves
    uint32_t seed_off;          // word offset of the leaf seed in the plan's seed buffer
    uint32_t seed_n;            // words of that leaf seed the kernel reads (seed_words_needed)
    uint32_t x_src;             // 0: input is a window of the raw block; 1: XOR combination in the workspace
    uint32_t x_off;             // x_src 0: word offset inside the raw block; 1: word offset in a block's X row
    uint32_t out_off;           // word offset of the leaf parities in a block's Y row
    uint32_t sterm_base, sterm_n;  // seed terms (bit offsets into the root seed) in the term table
    uint32_t iterm_base, iterm_n;  // input terms (bit offsets into the raw block)
    uint32_t pair_rows;         // rows per N pair (<= NT*BN, multiple of 32): r split evenly over npairs
};
// Output rows per work tile of the tcgen05 kernel (gemm_tc.cu: 2 N tiles x 224).
constexpr int kTileRows = 448;
uint32_t seed_words_needed(uint64_t n, uint64_t m);
// Grouped launch over the leaf table (Karatsuba): parities of leaf l, block b,
// row i go to bit 31 - (i & 31) of yws[b * y_stride + out_off + i / 32] (logical words).
qrng_status extract_grouped(const Leaf *d_leaves, uint32_t n_leaves, uint32_t total_npairs,
                            const uint32_t *d_seeds, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                            const uint32_t *xws, uint32_t x_stride, uint32_t *yws, uint32_t y_stride,
                            uint32_t max_leaf_w, cudaStream_t s);
bool supported(uint64_t n, uint64_t m);
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s);
// modified Toeplitz [T | I_m] (n-bit seed): repack x_b[0, n-m) to a multiple of
// 128 bits, the C1 product, then XOR the last m raw bits (api.cu)
bool modified_supported(uint64_t n, uint64_t m);
qrng_status plan_init_modified(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s);
qrng_status extract_modified(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                             const OutStream &out, cudaStream_t s);
void plan_free(Plan &pl);
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                    uint64_t m, const OutStream &out, cudaStream_t s);
// one-shot dense product straight from the caller's seed bytes (no plan)
qrng_status extract_direct(const uint8_t *d_seed, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                           const OutStream &out, cudaStream_t s);
qrng_status probe(const uint8_t *A, const uint8_t *h, int32_t *D, int N, int K, cudaStream_t s);
qrng_status trace(uint64_t *h_out, int reset);     // = timeline (gemm_tc.cu, -DQRNG_GEMM_TIMELINE builds)
qrng_status timeline(uint64_t *h_out, int reset);
int operand_bits();  // 4: kind::mxf4 (E2M1 operands)
qrng_status mxf4_probe(const uint8_t *A, const uint8_t *h, float *D, int N, int K, int hi_first, cudaStream_t s);
// instruments (gemm_probe.cu)
qrng_status mma_rate(int form, int iters, int n, uint64_t *macs, cudaStream_t s);
}  // namespace gemm

// The product on the CUDA cores for small batches (bits.cu): one lane per
// output bit, popcount parity of the seed window AND the reversed block.
namespace bits {
bool supported(uint64_t n, uint64_t m);
// seed words (logical big-endian, zero past n + m - 1) into pl.seed_words
qrng_status plan_init(gemm::Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s);
// seed from d_seed_words (a plan's) or, if null, straight from the caller's bytes;
// every output word is written once (no pre-zeroed output needed)
qrng_status extract(const uint32_t *d_seed_words, const uint8_t *d_seed_bytes, const uint8_t *d_raw,
                    uint64_t n_blocks, uint64_t n, uint64_t m, const OutStream &out, cudaStream_t s);
}  // namespace bits

// Karatsuba decomposition over the GEMM path (karatsuba.cu).
namespace kara {
struct Tables;  // device-resident leaf / term / combine tables, cached per (n, m, depth)
struct Plan {
    std::shared_ptr<const Tables> tab;  // shared with the LRU table cache
    uint32_t *seeds = nullptr;  // leaf seeds (logical big-endian words)
    const uint8_t *pending_seed = nullptr;  // one-shot plans: seeds formed by the first Q-buffer launch
    uint64_t seed_L = 0;
};
// Chooses the decomposition for (n, m); returns false if no leaf split pays off
// (the plain GEMM kernel is then used).  max_depth < 0: cost model decides.
bool choose(uint64_t n, uint64_t m, int max_depth);
// defer_seeds (one-shot calls only: the plan is extracted once, on `s`): the
// leaf seeds are formed by extra CTAs of the first extraction's Q-buffer launch
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, int max_depth, const uint8_t *d_seed, cudaStream_t s,
                      bool defer_seeds = false);
void plan_free(Plan &pl);
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                    const OutStream &out, cudaStream_t s);
// host-side description for bench/tests: depth, number of leaves, leaf MACs per block
void describe(const Plan &pl, int *depth, int *n_leaves, uint64_t *macs_per_block, uint32_t *x_words, uint32_t *y_words);
}  // namespace kara

// Histogram (hist.cu).
qrng_status hist256_launch(const uint8_t *d_samples, uint64_t n, unsigned long long *d_counts,
                           cudaStream_t s);

}  // namespace qrng
