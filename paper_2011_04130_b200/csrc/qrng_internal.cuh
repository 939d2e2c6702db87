// qrng_internal.cuh -- internal declarations shared by the libqrng.so sources.
// Product code (sm_100a).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
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

// Launch accounting / optional per-kernel event timing (qrng_debug_*).
void count_launch();
struct KernelTimer {  // brackets one extraction kernel on its stream (counts every launch)
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    KernelTimer(cudaStream_t st, bool timed);
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
constexpr int kMaxLogP = 23;
constexpr int kMaxFusedLogP = 15;  // one CTA holds the whole transform in smem

struct Plan {
    int logP = 0;
    uint32_t len = 0;            // raw bits per block entering the product
    bool xor_tail = false;       // modified Toeplitz identity block
    int pack_shift = 0;          // >0: two blocks share one transform (x1 + 2^shift x2)
    uint32_t *shat = nullptr;    // P words: NTT(seed) * P^-1 * 2^32 mod p, DIF order
    uint32_t *tw = nullptr;      // P words: w_P^e * 2^32 mod p
    uint32_t *itw = nullptr;     // P words: w_P^-e * 2^32 mod p
    uint32_t *work = nullptr;    // multipass scratch (not used by the fused kernel)
    size_t work_words = 0;
};
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t seed_bit_offset,
                      bool xor_tail, cudaStream_t s);
void plan_free(Plan &pl);
// n = block stride in bits (the product uses the plan's len bits of each block)
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                    uint64_t m, const OutStream &out, cudaStream_t s);
int choose_pack_shift(uint64_t n, int logP);
qrng_status butterfly_rate(int iters, uint64_t *butterflies, cudaStream_t s);
}  // namespace ntt

// GEMM path (gemm_tc.cu): tcgen05 kind::i8 batched Toeplitz product.
namespace gemm {
struct Plan {
    uint32_t *seed_words = nullptr;  // seed as logical big-endian words, zero padded
    uint32_t seed_words_n = 0;
};
bool supported(uint64_t n, uint64_t m);
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s);
void plan_free(Plan &pl);
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                    uint64_t m, const OutStream &out, cudaStream_t s);
qrng_status probe(const uint8_t *A, const uint8_t *h, int32_t *D, int N, int K, cudaStream_t s);
}  // namespace gemm

// Histogram (hist.cu).
qrng_status hist256_launch(const uint8_t *d_samples, uint64_t n, unsigned long long *d_counts,
                           cudaStream_t s);

}  // namespace qrng
