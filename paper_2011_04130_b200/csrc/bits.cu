// bits.cu -- the Toeplitz product on the CUDA cores, for small batches.
//
// y_i = XOR_j (s[i - j + n - 1] AND x_j)   (C1), rewritten with
// the reversed block x'_k = x_{n-1-k}:  y_i = parity(popc(S[i, i+n) AND x')),
// a window of the seed starting at bit i.  One lane per output bit: the
// window's 32-bit words are funnel shifts of two consecutive seed words (seed
// staged in shared memory), AND-ed with x' (read through L1: the lanes of a
// warp share one or two blocks) and XOR-accumulated; the parity of the
// accumulator's popcount is the bit; a warp ballot forms the 32-bit output
// word, written once (no pre-zeroed output, no atomics except the final
// partial word).  Each warp owns a contiguous run of output words, so its
// (block, row) position advances without a division per word.
//
// Why this exists on a tensor-core design: a batch of a few hundred blocks is
// latency-bound on the tcgen05 kernel (~10 us for one tile per SM: TMEM
// allocation, B generation, pipeline fill and drain) while its whole work is
// ~2e8 bit-MACs -- under a microsecond of ALU issue.  The crossover is by
// measurement (api.cu).
#include <algorithm>
#include <cstdlib>
#include "qrng_internal.cuh"

namespace qrng {
namespace bits {

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) bits_kernel(const uint32_t *__restrict__ raw, uint64_t n_blocks, uint32_t n,
                                                        uint32_t m, const uint32_t *__restrict__ seed_words,
                                                        const uint8_t *__restrict__ seed_bytes, uint32_t seed_nw,
                                                        uint64_t words_per_cta, OutStream out) {
    // shared: the seed (seed_nw logical big-endian words + 1 zero word), then
    // the reversed rows x' of the blocks this CTA's output words touch
    extern __shared__ uint32_t S[];
    const uint32_t nw = n / 32;
    const uint64_t L = (uint64_t)n + m - 1;
    const uint64_t total_bits = n_blocks * m, total_words = (total_bits + 31) / 32;
    const uint64_t CW0 = blockIdx.x * words_per_cta;
    const uint64_t CW1 = min(CW0 + words_per_cta, total_words);
    if (CW0 >= CW1) return;
    // bit indices fit 32 bits (n_blocks * m < 2^32, checked by the host)
    const uint32_t b_lo = (uint32_t)(CW0 * 32) / m;
    const uint32_t b_hi = min((uint32_t)(min(CW1 * 32, total_bits) - 1) / m, (uint32_t)n_blocks - 1);
    const uint32_t rows = b_hi - b_lo + 1;
    uint32_t *X = S + ((seed_nw + 1 + 3) & ~3u);
    // every load of the prologue in flight together (one memory round trip):
    // the seed words and the block rows, the rows as 16-byte vectors
    for (uint32_t k = threadIdx.x; k <= seed_nw; k += kThreads) {
        uint32_t v = 0;
        if (k < seed_nw) {
            if (seed_words) {
                v = seed_words[k];
            } else {  // the caller's MSB-first bytes (16-byte aligned): word k = bits [32k, 32k + 32), zero past L
                const uint64_t nbytes = (L + 7) / 8, b0 = 4ull * k;
                if (b0 + 4 <= nbytes) {
                    v = bswap32(__ldg(reinterpret_cast<const uint32_t *>(seed_bytes) + k));
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) v = (v << 8) | (b0 + t < nbytes ? (uint32_t)seed_bytes[b0 + t] : 0u);
                }
                const uint64_t lo = 32ull * k;
                if (lo + 32 > L) v &= L > lo ? (0xFFFFFFFFu << (32 - (uint32_t)(L - lo))) : 0u;
            }
        }
        S[k] = v;
    }
    if (nw % 4 == 0) {  // rows are whole 16-byte vectors (n % 128 == 0; raw is 16-byte aligned)
        const uint4 *src = reinterpret_cast<const uint4 *>(raw + (uint64_t)b_lo * nw);
        const uint32_t nv = rows * nw / 4, nw4 = nw / 4;
        for (uint32_t k = threadIdx.x; k < nv; k += kThreads) {
            const uint4 v = __ldg(src + k);
            // row r, raw words 4c .. 4c+3 -> x' words nw-1-4c .. nw-4-4c: brev of the logical word
            const uint32_t r = k / nw4, c = k - r * nw4;
            uint32_t *dst = X + r * nw + (nw - 1 - 4 * c);
            dst[0] = __brev(bswap32(v.x));
            dst[-1] = __brev(bswap32(v.y));
            dst[-2] = __brev(bswap32(v.z));
            dst[-3] = __brev(bswap32(v.w));
        }
    } else {
        for (uint32_t k = threadIdx.x; k < rows * nw; k += kThreads) {
            const uint32_t r = k / nw, w = k - r * nw;
            X[r * nw + (nw - 1 - w)] = __brev(bswap32(__ldg(raw + (uint64_t)(b_lo + r) * nw + w)));
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t W = CW0 + warp; W < CW1; W += kWarps) {
        // this lane's bit, relative to the CTA's first block: row i of block b_lo + br
        const uint64_t G = W * 32 + lane;
        const bool valid = G < total_bits;
        const uint32_t g = valid ? (uint32_t)G - b_lo * m : 0u;
        const uint32_t br = g / m, i = g - br * m;
        const uint32_t *xr = X + br * nw;
        const uint32_t *sp = S + (i >> 5);
        const uint32_t o = i & 31;
        uint32_t acc = 0, s_prev = sp[0];
#pragma unroll 8
        for (uint32_t w = 0; w < nw; ++w) {
            const uint32_t s_next = sp[w + 1];
            acc ^= __funnelshift_l(s_next, s_prev, o) & xr[w];  // seed bits [i + 32w, i + 32w + 32) AND x'
            s_prev = s_next;
        }
        const uint32_t word = __brev(__ballot_sync(0xFFFFFFFFu, valid && (__popc(acc) & 1u)));  // lane 0 -> MSB
        if (lane == 0) emit_word(out, W, word, true);
    }
}
// seed bytes (MSB-first) -> logical big-endian words, zero at and past L
__global__ void seed_words_kernel(const uint8_t *__restrict__ seed, uint64_t L, uint32_t *__restrict__ words,
                                  uint32_t nw) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nw) return;
    const uint64_t nbytes = (L + 7) / 8, b0 = 4ull * k;
    uint32_t v = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) v = (v << 8) | (b0 + t < nbytes ? (uint32_t)seed[b0 + t] : 0u);
    const uint64_t lo = 32ull * k;
    if (lo + 32 > L) v &= L > lo ? (0xFFFFFFFFu << (32 - (uint32_t)(L - lo))) : 0u;
    words[k] = v;
}
}  // namespace

bool supported(uint64_t n, uint64_t m) {
    // n % 32 == 0 (whole raw words); the seed (n + m - 1 bits) and two block
    // rows in shared memory
    return n % 32 == 0 && m >= 1 && ((n + m - 1 + 31) / 32 + 4 + 2 * (n / 32)) * 4 <= 180u * 1024u;
}

qrng_status plan_init(gemm::Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t s) {
    if (!supported(n, m)) {
        set_error("CUDA-core path: unsupported n=%llu m=%llu", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    pl.seed_words_n = (uint32_t)((n + m - 1 + 31) / 32);
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.seed_words, (size_t)pl.seed_words_n * 4, s));
    count_launch();
    seed_words_kernel<<<(pl.seed_words_n + 255) / 256, 256, 0, s>>>(d_seed, n + m - 1, pl.seed_words,
                                                                    pl.seed_words_n);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

qrng_status extract(const uint32_t *d_seed_words, const uint8_t *d_seed_bytes, const uint8_t *d_raw,
                    uint64_t n_blocks, uint64_t n, uint64_t m, const OutStream &out, cudaStream_t s) {
    if (!supported(n, m)) {
        set_error("CUDA-core path: n %% 32 != 0 or seed too long (n=%llu, m=%llu)", (unsigned long long)n,
                  (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    const uint32_t seed_nw = (uint32_t)((n + m - 1 + 31) / 32), nw = (uint32_t)(n / 32);
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t total_words = (n_blocks * m + 31) / 32;
    // output words per CTA: one per warp while that gives at most 8 CTAs per SM
    // (latency-bound sizes: many CTAs, each one memory round trip; measured at
    // config 1, plan reused: 1 / 2 / 4 / 8 / 16 words per warp 30.5 / 28.9 /
    // 25.3 / 21.8 / 16.3 Gbit/s), more per CTA beyond; capped so the touched
    // block rows fit in ~40 KB
    if (n_blocks * m >= (1ull << 32)) {
        set_error("CUDA-core path: n_blocks * m >= 2^32");
        return QRNG_E_UNSUPPORTED;
    }
    static const int wpw_env = [] {  // QRNG_BITS_WPW: minimum output words per warp (A/B)
        const char *e = getenv("QRNG_BITS_WPW");
        return (e && *e) ? std::max(1, atoi(e)) : 1;
    }();
    uint64_t wpc = std::max<uint64_t>((uint64_t)wpw_env * kWarps, (total_words + (uint64_t)sms * 8 - 1) / ((uint64_t)sms * 8));
    const uint64_t max_rows = std::max<uint64_t>(2, (40u * 1024u) / (nw * 4u));
    wpc = std::min<uint64_t>(wpc, std::max<uint64_t>(1, (max_rows - 1) * m / 32));
    const uint64_t ctas = (total_words + wpc - 1) / wpc;
    const uint64_t rows_max = (wpc * 32 + m - 1) / m + 1;
    const size_t smem = ((size_t)((seed_nw + 1 + 3) & ~3u) + (size_t)rows_max * nw) * 4;
    if (smem > 48 * 1024) {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(bits_kernel));
        if (st != QRNG_OK) return st;
    }
    if (smem > 227 * 1024 || ctas > 0x7FFFFFFFull) {
        set_error("CUDA-core path: launch shape out of range (n=%llu, m=%llu)", (unsigned long long)n,
                  (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    KernelTimer tm(s, true);
    bits_kernel<<<(unsigned)ctas, kThreads, smem, s>>>(reinterpret_cast<const uint32_t *>(d_raw), n_blocks,
                                                       (uint32_t)n, (uint32_t)m, d_seed_words, d_seed_bytes, seed_nw,
                                                       wpc, out);
    tm.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

}  // namespace bits
}  // namespace qrng
