// ntt.cu -- exact number-theoretic-transform path of the Toeplitz extractor.
//
// Method (Sec. III.B, Def. 1-2, Thm. 1-2): embed T in the
// circulant of the seed, so that the key is a window of a cyclic convolution:
//     y_i = c[n-1+i],   c = s * x   (linear convolution).
// The paper computes it with a floating-point FFT followed by round and mod 2
// (Listing 2).  Here the transform is an NTT modulo the prime
// p = 119*2^23 + 1 over a cyclic length P = 2^ceil(log2(n+m-1)) (A20,
// PAPER.md:251): every window value c_t <= n < p, and P >= L rules out
// wrap-around inside the window, so z_t mod p == c_t EXACTLY and y_i is its
// parity (reading A16: no rounding, zero tolerance).
//
// B200 design: one CTA owns one transform of length
// P <= 2^15 in shared memory (padded 1 word per 32 against bank conflicts).
// The transform is a mixed-radix (2^3..2^5) Cooley-Tukey decomposition: each
// pass runs a register-resident radix-2^r DIF sub-DFT with compile-time roots
// in the constant bank (Shoup multiplication), then the inter-pass twiddles
// (Montgomery, powers generated in registers from one table word per thread).
// The deepest pass fuses forward DFT -> pointwise product with the prepared
// seed spectrum -> inverse DFT, so the spectrum never leaves registers.
// For n <= 2^14 two blocks share one transform as x1 + 2^k x2 (2^k > n and
// n (2^k + 1) < p keeps both convolutions exact and separable: parity of c1
// is bit 0, parity of c2 is bit k).  Values are kept lazily in [0, 2p); the
// final residue is made canonical before its parity is taken.
// Larger P run as global radix passes around 2^15-word segment kernels; for
// n < 2^21 four blocks share each transform as sum_g 2^(k g) x_g modulo three
// primes, and the window sums come back by CRT ("Packed three-prime form",
// DESIGN.md 6.3).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "qrng_internal.cuh"

namespace qrng {
namespace ntt {

// The two NTT primes (both < 2^30, so lazy residues in [0, 2p) and sums < 4p
// fit 32 bits; primitive root 3 for both):
//   F = 0: p = 119 * 2^23 + 1 = 998244353 -- every single-GPU transform P <= 2^23;
//   F = 1: p =   7 * 2^26 + 1 = 469762049 -- the distributed four-step NTT of
//          one block (NEXT-4, ntt_dist.cu): roots of unity of order up to 2^26.
template <int F> struct Fld;
template <> struct Fld<0> { static constexpr uint32_t P = kP, PINV = 3296722945u; static constexpr int LOG2 = 23; };
template <> struct Fld<1> { static constexpr uint32_t P = kP2, PINV = 3825205249u; static constexpr int LOG2 = 26; };
//   F = 2: p =   5 * 2^25 + 1 = 167772161 -- third prime of the packed
//          three-prime form (kP kP2 kP3 > 2^86; primitive root 3)
template <> struct Fld<2> { static constexpr uint32_t P = kP3, PINV = 4127195137u; static constexpr int LOG2 = 25; };
static_assert(Fld<0>::P * Fld<0>::PINV == 1u && Fld<1>::P * Fld<1>::PINV == 1u && Fld<2>::P * Fld<2>::PINV == 1u,
              "PINV = p^-1 mod 2^32");
static_assert(4ull * Fld<0>::P < (1ull << 32) && 4ull * Fld<1>::P < (1ull << 32), "lazy [0, 4p) sums fit 32 bits");
constexpr uint32_t P = kP;  // the single-GPU prime (fused kernels, plans of ntt.cu's host code)

constexpr uint64_t powmod_p(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1;
    b %= p;
    while (e) {
        if (e & 1) r = r * b % p;
        b = b * b % p;
        e >>= 1;
    }
    return r;
}
constexpr uint64_t powmod_c(uint64_t b, uint64_t e) { return powmod_p(b, e, P); }

struct RootTab {
    uint32_t w[64], wp[64], iw[64], iwp[64];  // w_64^e, Shoup companions, inverses
};
constexpr RootTab make_roots(uint64_t p) {
    RootTab t{};
    uint64_t w64 = powmod_p(3, (p - 1) / 64, p), iw64 = powmod_p(w64, p - 2, p);
    uint64_t a = 1, b = 1;
    for (int e = 0; e < 64; ++e) {
        t.w[e] = (uint32_t)a;
        t.wp[e] = (uint32_t)((a << 32) / p);
        t.iw[e] = (uint32_t)b;
        t.iwp[e] = (uint32_t)((b << 32) / p);
        a = a * w64 % p;
        b = b * iw64 % p;
    }
    return t;
}
__constant__ RootTab c_roots[3] = {make_roots(Fld<0>::P), make_roots(Fld<1>::P), make_roots(Fld<2>::P)};

// ---- modular arithmetic on lazy residues in [0, 2p) ------------------------
template <int F = 0>
__device__ __forceinline__ uint32_t red2(uint32_t x) { return min(x, x - 2u * Fld<F>::P); }  // [0,4p)->[0,2p)
template <int F = 0>
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wp) {
    uint32_t q = __umulhi(a, wp);
    return a * w - q * Fld<F>::P;  // a*w mod p in [0, 2p), any 32-bit a
}
// Montgomery product a*b/2^32 mod p for a, b < 2p, result in (0, 2p):
// t = a*b < 4p^2 < p 2^32; q = t_lo p^-1 mod 2^32 makes t - q p divisible by
// 2^32, so (t - q p)/2^32 = t_hi - hi(q p) lies in (-p, p); add p.  Written as
// mul.wide / mul.lo / mul.hi / sub so ptxas emits 4 instructions (IMAD.WIDE,
// IMAD, IMAD.HI, IADD3) instead of fusing a 64-bit addend chain.
template <int F = 0>
__device__ __forceinline__ uint32_t mont(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("{\n\t.reg .u64 t;\n\t.reg .u32 lo, hi, q, h;\n\t"
        "mul.wide.u32 t, %1, %2;\n\t"
        "mov.b64 {lo, hi}, t;\n\t"
        "mul.lo.u32 q, lo, %3;\n\t"
        "mul.hi.u32 h, q, %4;\n\t"
        "sub.u32 %0, hi, h;\n\t"
        "add.u32 %0, %0, %4;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "n"(Fld<F>::PINV), "n"(Fld<F>::P));
    return r;
}

__host__ __device__ constexpr int brev(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}

// Radix-2^R DIF on registers: natural order in, bit-reversed order out.
// Every loop has a compile-time trip count so the array stays in registers.
template <int R, int F = 0>
__device__ __forceinline__ void dft_fwd(uint32_t (&x)[1 << R]) {
    constexpr uint32_t P2 = 2u * Fld<F>::P;
    constexpr int N = 1 << R;
#pragma unroll
    for (int t = 0; t < R; ++t) {
#pragma unroll
        for (int k = 0; k < N / 2; ++k) {
            const int half = N >> (t + 1);
            const int e = k & (half - 1);
            const int i = ((k / half) * 2 * half) + e;
            const int step = 64 / (2 * half);
            uint32_t a = x[i], b = x[i + half];
            uint32_t v = a - b + P2;
            x[i] = red2<F>(a + b);
            x[i + half] = (e == 0) ? red2<F>(v) : shoup<F>(v, c_roots[F].w[e * step], c_roots[F].wp[e * step]);
        }
    }
}

// Radix-2^R DIT with inverse roots: bit-reversed order in, natural order out
// (unscaled: returns N times the inverse DFT).
template <int R, int F = 0>
__device__ __forceinline__ void dft_inv(uint32_t (&x)[1 << R]) {
    constexpr uint32_t P2 = 2u * Fld<F>::P;
    constexpr int N = 1 << R;
#pragma unroll
    for (int t = 0; t < R; ++t) {
#pragma unroll
        for (int k = 0; k < N / 2; ++k) {
            const int half = 1 << t;
            const int e = k & (half - 1);
            const int i = ((k / half) * 2 * half) + e;
            const int step = 64 / (2 * half);
            uint32_t a = x[i], b = x[i + half];
            uint32_t tb = (e == 0) ? b : shoup<F>(b, c_roots[F].iw[e * step], c_roots[F].iwp[e * step]);
            x[i] = red2<F>(a + tb);
            x[i + half] = red2<F>(a - tb + P2);
        }
    }
}

// Register q holds spectrum index k1 = brev(q): multiply it by tau^k1
// (tauM = tau * 2^32 mod p, Montgomery form).  The powers come from four
// independent chains tau^(j+1) * (tau^4)^i, so the Montgomery products are not
// one serial dependency chain.
template <int R, int F = 0>
__device__ __forceinline__ void twiddle(uint32_t (&x)[1 << R], uint32_t tauM) {
    constexpr int N = 1 << R;
    if constexpr (N <= 4) {
        uint32_t pw = tauM;
#pragma unroll
        for (int k = 1; k < N; ++k) {
            if (k > 1) pw = mont<F>(pw, tauM);
            x[brev(k, R)] = mont<F>(x[brev(k, R)], pw);
        }
    } else {
        const uint32_t t2 = mont<F>(tauM, tauM), t3 = mont<F>(t2, tauM), t4 = mont<F>(t2, t2);
        uint32_t c[4] = {tauM, t2, t3, t4};
#pragma unroll
        for (int i = 0; i < N / 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = 4 * i + j + 1;
                if (k < N) {
                    if (i > 0) c[j] = mont<F>(c[j], t4);
                    x[brev(k, R)] = mont<F>(x[brev(k, R)], c[j]);
                }
            }
    }
}

// Level-1 twiddles of the 2^15-word segment kernel from shared memory: tab[k * 32 +
// n2] = (tau^k, floor(tau^k 2^32 / p)) for the sub-DFT with n2 = u % 32 (= the
// lane: conflict-free 8-byte loads), a 3-instruction Shoup product per element
// instead of the Montgomery power chain (2 products per element).
template <int R, int F = 0>
__device__ __forceinline__ void twiddle_l1(uint32_t (&x)[1 << R], const uint2 *col) {
    constexpr int N = 1 << R;
#pragma unroll
    for (int k = 1; k < N; ++k) {
        const uint2 t = col[k * 32];
        x[brev(k, R)] = shoup<F>(x[brev(k, R)], t.x, t.y);
    }
}

// ---- pass schedule ---------------------------------------------------------
__host__ __device__ constexpr int np_of(int logP) { return (logP + 4) / 5; }
__host__ __device__ constexpr int radix_of(int logP, int lv) {
    return logP / np_of(logP) + (lv < logP % np_of(logP) ? 1 : 0);
}
__host__ __device__ constexpr int prefix_of(int logP, int lv) {
    int s = 0;
    for (int i = 0; i < lv; ++i) s += radix_of(logP, i);
    return s;
}
#ifndef QRNG_NTT_MAXT
#define QRNG_NTT_MAXT 1024  // threads per transform CTA (each thread takes P / 32 / T sub-DFTs per level)
#endif
__host__ __device__ constexpr int threads_of(int logP) {
    return (1 << logP) / 32 < 32 ? 32 : ((1 << logP) / 32 > QRNG_NTT_MAXT ? QRNG_NTT_MAXT : (1 << logP) / 32);
}
__host__ __device__ constexpr int pidx(int i) { return i + (i >> 5); }

struct FusedArgs {
    const uint32_t *raw;      // raw stream as 32-bit words (MSB-first bytes)
    uint64_t n_blocks;
    uint32_t n, m;
    int shift;                // pack shift (PACK only)
    const uint32_t *shat, *tw, *itw;
    OutStream out;
    uint32_t stage_words;     // per-CTA staging words
    uint32_t tw_shift;        // segment mode: log2(P / segment length) (tables are for w_P)
    uint32_t scaleM;          // forward-only mode: P^-1 * 2^64 mod p
    uint32_t len;             // raw bits used per block (n, or n - m for the modified Toeplitz)
    uint32_t xor_tail;        // modified Toeplitz: output t also XORs raw bit t + 1 of its block
    const uint2 *l1tw;        // SEG mode, 2^15-word segments: level-1 Shoup twiddles [dir][k][n2] (or null)
};

// Level modes: FUSED = one CTA owns a whole transform (bits in, parity bits
// out); SEG = the CTA owns one segment of a multi-pass transform (shared
// memory in and out; the global passes live in ntt_pass_kernel); SEGFWD =
// forward levels only, the last one writes the scaled spectrum (seed prep).
enum { FUSED = 0, SEG = 1, SEGFWD = 2 };

// bit idx of block b (idx < n), stream MSB-first; n % 32 == 0
__device__ __forceinline__ uint32_t raw_bit(const uint32_t *raw, uint64_t b, uint32_t n, uint32_t idx) {
    uint32_t w = __ldg(raw + b * (n >> 5) + (idx >> 5));
    return (bswap32(w) >> (31 - (idx & 31))) & 1u;
}

// Seed spectrum layout: element (sub-DFT u, register q) of a transform's (or
// segment's) last level.  Interleaved (default): the four-word group q / 4 of
// consecutive u is contiguous, so the pointwise product's 16-byte loads (and
// the spectrum's stores) of a warp are consecutive; QRNG_NTT_SHAT_ILV=0: row u
// contiguous (the round-1 layout, for A/B).
#ifndef QRNG_NTT_SHAT_ILV
#define QRNG_NTT_SHAT_ILV 1
#endif
template <int N1, int NSUB>
__device__ __forceinline__ size_t shat4_idx(int u, int q4) {  // uint4 index of words 4 q4 .. 4 q4 + 3
    return QRNG_NTT_SHAT_ILV ? (size_t)q4 * NSUB + u : (size_t)u * (N1 / 4) + q4;
}

template <int LOGP, int LV, bool PACK, int MODE = FUSED, int F = 0>
struct Level {
    static constexpr uint32_t P = Fld<F>::P;
    static constexpr int R = radix_of(LOGP, LV);
    static constexpr int S = prefix_of(LOGP, LV);
    static constexpr int NPASS = np_of(LOGP);
    static constexpr int N1 = 1 << R;
    static constexpr int STRIDE = (1 << LOGP) >> (S + R);
    static constexpr int NSEG = (1 << LOGP) >> S;
    static constexpr int NSUB = (1 << LOGP) >> R;
    static constexpr bool LAST = (LV == NPASS - 1);
    static constexpr int T = threads_of(LOGP);

    __device__ static __forceinline__ int addr(int u, int q) {
        return (u / STRIDE) * NSEG + q * STRIDE + (u % STRIDE);
    }
    // padded smem index of element q of sub-transform u = pbase(u) + poff(q):
    // exact when NSEG % 32 == 0 or STRIDE == 1 (q*STRIDE never carries into
    // the padding of the segment base), so the per-q offsets are immediates.
    static_assert(NSEG % 32 == 0 || STRIDE == 1, "padded addressing needs aligned segments");
    __device__ static __forceinline__ int pbase(int u) { return pidx((u / STRIDE) * NSEG + (u % STRIDE)); }
    static constexpr int poff(int q) { return pidx(q * STRIDE); }

    __device__ static __forceinline__ void load(uint32_t (&x)[N1], int u, uint32_t *data,
                                                const FusedArgs &a, uint64_t b0, int nb) {
        if (LV == 0 && MODE != FUSED) {  // segment already in shared memory
            const int pb = pbase(u);
#pragma unroll
            for (int q = 0; q < N1; ++q) x[q] = data[pb + poff(q)];
        } else if (LV == 0 && STRIDE >= 32) {
            // the warp holds u = u0..u0+31 (u0 % 32 == 0): for each q it needs one
            // 32-bit raw word (idx = q*STRIDE + u0 .. +31).  Lane q fetches word q.
            const int lane = threadIdx.x & 31, u0 = u & ~31;
            const uint32_t *blk = a.raw + b0 * (a.n >> 5);
            uint32_t w1 = 0, w2 = 0;
            const uint32_t myidx = (uint32_t)((lane % N1) * STRIDE + u0);
            if (lane < N1 && myidx < a.len) {
                w1 = bswap32(__ldg(blk + (myidx >> 5)));
                if (PACK && nb > 1) w2 = bswap32(__ldg(blk + (a.n >> 5) + (myidx >> 5)));
                const uint32_t rem = a.len - myidx;  // bits past len are not part of the product
                if (rem < 32) {
                    w1 &= 0xFFFFFFFFu << (32 - rem);
                    w2 &= 0xFFFFFFFFu << (32 - rem);
                }
            }
            const int sh = 31 - lane;
#pragma unroll
            for (int q = 0; q < N1; ++q) {
                uint32_t v = (__shfl_sync(0xffffffffu, w1, q) >> sh) & 1u;
                if (PACK) v |= ((__shfl_sync(0xffffffffu, w2, q) >> sh) & 1u) << a.shift;
                x[q] = v;
            }
        } else if (LV == 0) {  // small P: idx = q*STRIDE + u
#pragma unroll
            for (int q = 0; q < N1; ++q) {
                uint32_t idx = (uint32_t)(q * STRIDE + u), v = 0;
                if (idx < a.len) {
                    v = raw_bit(a.raw, b0, a.n, idx);
                    if (PACK && nb > 1) v |= raw_bit(a.raw, b0 + 1, a.n, idx) << a.shift;
                }
                x[q] = v;
            }
        } else {
            const int pb = pbase(u);
#pragma unroll
            for (int q = 0; q < N1; ++q) x[q] = data[pb + poff(q)];
        }
    }

    // Final inverse output at level 0: element q is z_t, t = q*STRIDE + u.
    __device__ static __forceinline__ void stage_or(uint32_t *stage, uint64_t wfirst, int64_t G, uint32_t bal) {
        if (!bal) return;
        const uint32_t V = __brev(bal);  // ballot bit L (output G+L) -> logical bit 31-L
        const int64_t W0 = G >= 0 ? (G >> 5) : -((31 - G) >> 5);
        const int o = (int)(G - W0 * 32);
        const uint32_t hi = V >> o, lo = o ? (V << (32 - o)) : 0u;
        if (hi) atomicOr(&stage[W0 - (int64_t)wfirst], hi);
        if (lo) atomicOr(&stage[W0 + 1 - (int64_t)wfirst], lo);
    }

    __device__ static __forceinline__ void emit(uint32_t (&x)[N1], int u, uint32_t *stage,
                                                const FusedArgs &a, uint64_t b0, int nb,
                                                uint64_t wfirst) {
        if constexpr (STRIDE >= 32) {
            // lanes hold 32 consecutive t for every q: one ballot per q gives a
            // 32-bit output word; lane q keeps word q and ORs it into the stage.
            const int lane = threadIdx.x & 31, u0 = u & ~31;
            uint32_t mine1 = 0, mine2 = 0;
#pragma unroll
            for (int q = 0; q < N1; ++q) {
                const uint32_t t = (uint32_t)(q * STRIDE + u);
                int64_t i = (int64_t)t - (int64_t)(a.len - 1);
                bool valid = i >= 0 && i < (int64_t)a.m;
                uint32_t z = x[q] >= P ? x[q] - P : x[q];  // canonical residue
                uint32_t x1 = 0, x2 = 0;                   // identity block of [T | I_m]
                if (a.xor_tail && valid) {
                    x1 = raw_bit(a.raw, b0, a.n, t + 1);
                    if (PACK && nb > 1) x2 = raw_bit(a.raw, b0 + 1, a.n, t + 1) << a.shift;
                }
                uint32_t b1 = __ballot_sync(0xffffffffu, valid && ((z ^ x1) & 1u));
                if (lane == (q & 31)) mine1 = b1;
                if (PACK) {
                    uint32_t b2 = __ballot_sync(0xffffffffu, valid && (((z ^ x2) >> a.shift) & 1u));
                    if (lane == (q & 31)) mine2 = b2;
                }
                if ((q & 31) == 31 || q == N1 - 1) {
                    const int qb = q & ~31;
                    if (lane <= (q & 31)) {
                        int64_t i0 = (int64_t)((qb + lane) * STRIDE + u0) - (int64_t)(a.len - 1);
                        stage_or(stage, wfirst, (int64_t)(b0 * a.m) + i0, mine1);
                        if (PACK && nb > 1) stage_or(stage, wfirst, (int64_t)((b0 + 1) * a.m) + i0, mine2);
                    }
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < N1; ++q) {
                const uint32_t t = (uint32_t)(q * STRIDE + u);
                int64_t i = (int64_t)t - (int64_t)(a.len - 1);
                if (i >= 0 && i < (int64_t)a.m) {
                    uint32_t z = x[q] >= P ? x[q] - P : x[q];  // canonical residue
                    if (a.xor_tail) {
                        z ^= raw_bit(a.raw, b0, a.n, t + 1);
                        if (PACK && nb > 1) z ^= raw_bit(a.raw, b0 + 1, a.n, t + 1) << a.shift;
                    }
                    if (z & 1u) {
                        uint64_t g = b0 * a.m + (uint64_t)i;
                        atomicOr(&stage[(g >> 5) - wfirst], 0x80000000u >> (g & 31));
                    }
                    if (PACK && nb > 1 && ((z >> a.shift) & 1u)) {
                        uint64_t g = (b0 + 1) * a.m + (uint64_t)i;
                        atomicOr(&stage[(g >> 5) - wfirst], 0x80000000u >> (g & 31));
                    }
                }
            }
        }
    }

    __device__ static __forceinline__ void fwd(uint32_t *data, uint32_t *stage, const FusedArgs &a,
                                               uint64_t b0, int nb, uint64_t wfirst) {
#pragma unroll
        for (int it = 0; it < (NSUB + T - 1) / T; ++it) {  // independent sub-DFTs: unrolled so they interleave
            const int u = (int)threadIdx.x + it * T;
            if (NSUB % T != 0 && u >= NSUB) break;
            uint32_t x[N1];
            load(x, u, data, a, b0, nb);
            dft_fwd<R, F>(x);
            if (!LAST) {
                const int n2 = u % STRIDE;
                if constexpr (MODE == SEG && LOGP == 15 && LV == 1 && N1 == 32 && STRIDE == 32) {
                    // stage = the shared-memory level-1 table in SEG mode (null: chains)
                    if (n2) {
                        if (stage) twiddle_l1<R, F>(x, reinterpret_cast<const uint2 *>(stage) + n2);
                        else twiddle<R, F>(x, __ldg(a.tw + ((uint32_t)(n2 << S) << a.tw_shift)));
                    }
                } else {
                    if (n2) twiddle<R, F>(x, __ldg(a.tw + ((uint32_t)(n2 << S) << a.tw_shift)));
                }
                {
                    const int pb = pbase(u);
#pragma unroll
                    for (int q = 0; q < N1; ++q) data[pb + poff(q)] = x[q];
                }
            } else if (MODE == SEGFWD) {
                static_assert(N1 % 4 == 0, "last level radix >= 4");
                uint4 *dst4 = reinterpret_cast<uint4 *>(const_cast<uint32_t *>(a.shat));
#pragma unroll
                for (int q4 = 0; q4 < N1 / 4; ++q4)  // * P^-1 * 2^32, 16-byte stores
                    dst4[shat4_idx<N1, NSUB>(u, q4)] =
                        make_uint4(mont<F>(x[4 * q4], a.scaleM), mont<F>(x[4 * q4 + 1], a.scaleM),
                                   mont<F>(x[4 * q4 + 2], a.scaleM), mont<F>(x[4 * q4 + 3], a.scaleM));
            } else {
                // pointwise product with the seed spectrum (DIF order: sub-DFT u, register q)
                const uint4 *sh = reinterpret_cast<const uint4 *>(a.shat);
#pragma unroll
                for (int q4 = 0; q4 < N1 / 4; ++q4) {
                    uint4 s4 = __ldg(sh + shat4_idx<N1, NSUB>(u, q4));
                    x[4 * q4 + 0] = mont<F>(x[4 * q4 + 0], s4.x);
                    x[4 * q4 + 1] = mont<F>(x[4 * q4 + 1], s4.y);
                    x[4 * q4 + 2] = mont<F>(x[4 * q4 + 2], s4.z);
                    x[4 * q4 + 3] = mont<F>(x[4 * q4 + 3], s4.w);
                }
                dft_inv<R, F>(x);
                if (LV == 0 && MODE == FUSED) emit(x, u, stage, a, b0, nb, wfirst);
                else {
                    const int pb = pbase(u);
#pragma unroll
                    for (int q = 0; q < N1; ++q) data[pb + poff(q)] = x[q];
                }
            }
        }
        __syncthreads();
    }

    __device__ static __forceinline__ void inv(uint32_t *data, uint32_t *stage, const FusedArgs &a,
                                               uint64_t b0, int nb, uint64_t wfirst) {
#pragma unroll
        for (int it = 0; it < (NSUB + T - 1) / T; ++it) {  // independent sub-DFTs: unrolled so they interleave
            const int u = (int)threadIdx.x + it * T;
            if (NSUB % T != 0 && u >= NSUB) break;
            uint32_t x[N1];
            {
                const int pb = pbase(u);
#pragma unroll
                for (int q = 0; q < N1; ++q) x[q] = data[pb + poff(q)];
            }
            const int n2 = u % STRIDE;
            if constexpr (MODE == SEG && LOGP == 15 && LV == 1 && N1 == 32 && STRIDE == 32) {
                if (n2) {
                    if (stage) twiddle_l1<R, F>(x, reinterpret_cast<const uint2 *>(stage) + 1024 + n2);
                    else twiddle<R, F>(x, __ldg(a.itw + ((uint32_t)(n2 << S) << a.tw_shift)));
                }
            } else {
                if (n2) twiddle<R, F>(x, __ldg(a.itw + ((uint32_t)(n2 << S) << a.tw_shift)));
            }
            dft_inv<R, F>(x);
            if (LV == 0 && MODE == FUSED) emit(x, u, stage, a, b0, nb, wfirst);
            else {
                {
                    const int pb = pbase(u);
#pragma unroll
                    for (int q = 0; q < N1; ++q) data[pb + poff(q)] = x[q];
                }
            }
        }
        __syncthreads();
    }
};

template <int LOGP, int LV, bool PACK, int MODE = FUSED, int F = 0>
__device__ __forceinline__ void run_levels(uint32_t *data, uint32_t *stage, const FusedArgs &a,
                                           uint64_t b0, int nb, uint64_t wfirst) {
    using L = Level<LOGP, LV, PACK, MODE, F>;
    L::fwd(data, stage, a, b0, nb, wfirst);
    if constexpr (!L::LAST) {
        run_levels<LOGP, LV + 1, PACK, MODE, F>(data, stage, a, b0, nb, wfirst);
        if constexpr (MODE != SEGFWD) L::inv(data, stage, a, b0, nb, wfirst);
    }
}

// ---- multi-pass transform (P > 2^15) ----------------------------------------
// The first levels of the decomposition run as global passes over a
// workspace (ntt_pass_kernel); each remaining 2^LOGS-word segment is an
// independent transform of length 2^LOGS with root w_P^(P/2^LOGS), handled
// entirely in shared memory by ntt_segment_kernel (forward levels, pointwise
// product, inverse levels); the global inverse passes follow, the last one
// emitting parity bits.
#ifndef QRNG_NTT_SEGLOG
#define QRNG_NTT_SEGLOG 15
#endif
constexpr int kSegLog = QRNG_NTT_SEGLOG;  // words per segment-kernel CTA (log2)

template <int LOGS, int MODE, int F = 0>
__global__ void __launch_bounds__(threads_of(LOGS), 1024 / threads_of(LOGS))
    ntt_segment_kernel(FusedArgs a, uint32_t *ws, uint32_t logP) {
    extern __shared__ uint32_t smem[];
    constexpr int NS = 1 << LOGS;
    uint32_t *data = smem;
    const uint64_t seg = blockIdx.x;
    uint32_t *src = ws + ((uint64_t)blockIdx.y << logP) + seg * NS;
    // SEG mode: the level-1 twiddle table (2 x 32 x 32 Shoup pairs) after the data
    uint32_t *tab = nullptr;
    if (MODE == SEG && LOGS == 15 && a.l1tw) {
        uint2 *t2 = reinterpret_cast<uint2 *>(smem + pidx(NS));
        for (int i = threadIdx.x; i < 2048; i += blockDim.x) t2[i] = __ldg(a.l1tw + i);
        tab = reinterpret_cast<uint32_t *>(t2);
    }
    for (int i = threadIdx.x * 4; i < NS; i += blockDim.x * 4) {
        const uint4 v = *reinterpret_cast<const uint4 *>(src + i);
        data[pidx(i)] = v.x;
        data[pidx(i + 1)] = v.y;
        data[pidx(i + 2)] = v.z;
        data[pidx(i + 3)] = v.w;
    }
    __syncthreads();
    FusedArgs b = a;
    b.shat = a.shat + seg * NS;
    run_levels<LOGS, 0, false, MODE, F>(data, tab, b, 0, 1, 0);
    if constexpr (MODE != SEGFWD) {
        for (int i = threadIdx.x * 4; i < NS; i += blockDim.x * 4)
            *reinterpret_cast<uint4 *>(src + i) =
                make_uint4(data[pidx(i)], data[pidx(i + 1)], data[pidx(i + 2)], data[pidx(i + 3)]);
    }
}

struct PassArgs {
    const uint32_t *bits;     // MODE_BITS / MODE_SEED: packed input (raw stream or seed words)
    uint64_t b0;              // first block of the batch (raw stream / output)
    uint32_t n, m, len;       // len: input bits per transform (n for data, L for the seed)
    uint32_t *ws;
    const uint32_t *tw, *itw;
    uint32_t logP, S;         // this pass works on segments of 2^(logP - S) words
    OutStream out;
    uint32_t xor_tail;        // modified Toeplitz: output t also XORs raw bit t + 1 of its block
    // PASS_FWD_PACK (packed three-prime form): transform b of the batch holds
    // blocks (b0 + b) G + g, g < G, as sum_g cg[g] x_g (cg[g] = 2^(k g) mod p)
    uint32_t G;
    uint32_t cg[4];
    uint64_t n_blocks;
    // PASS_INV_CRT: the first two primes' z_t (natural order, same layout as ws)
    const uint32_t *crt0, *crt1;
    uint32_t crt_k;
};
enum { PASS_FWD_BITS = 0, PASS_FWD_SEED = 1, PASS_FWD = 2, PASS_INV = 3, PASS_INV_EMIT = 4, PASS_INV_EMIT_XOR = 5,
       PASS_FWD_PACK = 6, PASS_INV_CRT = 8 };

// ---- packed three-prime form: CRT and key bits ------------------------------
// Garner constants for (p0, p1, p2) = (kP, kP2, kP3); Shoup companions
// floor(c 2^32 / p) so every product is a 3-instruction Shoup multiply.
struct Crt {
    static constexpr uint64_t p0 = kP, p1 = kP2, p2 = kP3;
    static constexpr uint32_t c1 = (uint32_t)powmod_p(p0 % p1, p1 - 2, p1);  // p0^-1 mod p1
    static constexpr uint32_t c1p = (uint32_t)(((uint64_t)c1 << 32) / p1);
    static constexpr uint32_t one2p = (uint32_t)((1ull << 32) / p2);         // reduces r0 mod p2
    static constexpr uint32_t p0m2 = (uint32_t)(p0 % p2);
    static constexpr uint32_t p0m2p = (uint32_t)(((uint64_t)p0m2 << 32) / p2);
    static constexpr uint32_t c2 = (uint32_t)powmod_p(p0 % p2 * (p1 % p2) % p2, p2 - 2, p2);  // (p0 p1)^-1 mod p2
    static constexpr uint32_t c2p = (uint32_t)(((uint64_t)c2 << 32) / p2);
    static constexpr uint64_t p01 = p0 * p1;
};
constexpr int kCrtQ = 32;  // window q per warp staged in shared memory by PASS_INV_CRT (8 warps: 64 KB)
__device__ __forceinline__ uint32_t shoup_p(uint32_t a, uint32_t w, uint32_t wp, uint32_t p) {
    return a * w - __umulhi(a, wp) * p;  // a w mod p in [0, 2p)
}

#ifndef QRNG_NTT_EMIT_SKIP
#define QRNG_NTT_EMIT_SKIP 1  // 0: every q through the window test (A/B)
#endif
// Radix-64 passes: ptxas otherwise spends 214-254 registers (one 256-thread
// CTA per SM); 3 CTAs per SM (85 registers) where that costs at most a few
// bytes of spill, 2 (128 registers) for the forms that spill at 3
#ifndef QRNG_NTT_CRT_CTAS
#define QRNG_NTT_CRT_CTAS 3  // CTAs per SM of the CRT pass (80 registers, 24 B of spill at radix 64)
#endif
#ifndef QRNG_NTT_PASS_BOUND
#define QRNG_NTT_PASS_BOUND 1  // 0: no bound on the radix-64 passes except the emit pass (A/B)
#endif
__host__ __device__ constexpr int ntt_pass_min_ctas(int R, int MODE) {
    return (R == 5 && MODE == 6 && QRNG_NTT_PASS_BOUND) ? 3             // PASS_FWD_PACK at radix 32: 145 -> 85
           : R < 6 ? 1
           : (MODE == 4 || MODE == 5) ? (QRNG_NTT_EMIT_SKIP ? 3 : 1)  // PASS_INV_EMIT[_XOR]
           : !QRNG_NTT_PASS_BOUND ? 1
           : MODE == 6 ? 3                                            // PASS_FWD_PACK
           : MODE == 8 ? QRNG_NTT_CRT_CTAS                            // PASS_INV_CRT
           : MODE == 2 ? 1                                            // PASS_FWD spills even at 2
           : 2;
}
template <int R, int MODE, int F = 0>
__global__ void __launch_bounds__(256, ntt_pass_min_ctas(R, MODE))
    ntt_pass_kernel(PassArgs a) {
    constexpr int N1 = 1 << R;
    constexpr uint32_t P = Fld<F>::P;
    const uint32_t logseg = a.logP - a.S, logstride = logseg - R;
    const uint32_t u = blockIdx.x * 256 + threadIdx.x;  // sub-transform within the block
    const uint64_t bb = blockIdx.y;
    const uint32_t seg = u >> logstride, n2 = u & ((1u << logstride) - 1);
    const uint32_t STRIDE = 1u << logstride;
    uint32_t *base = a.ws + (bb << a.logP) + ((uint64_t)seg << logseg) + n2;
    // PASS_INV_CRT: the first two primes' z_t of the warp's window q (up to
    // kCrtQ of them) are copied into shared memory by cp.async while the
    // transform runs, so the CRT loop finds them there (a load per q inside
    // that loop exposes its latency once per q)
    extern __shared__ uint32_t crt_sm[];
    int crt_qlo = 0, crt_nq = 0;
    if constexpr (MODE == PASS_INV_CRT) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t u0 = u & ~31u;
        const int64_t w_lo = (int64_t)(a.len - 1), w_hi = w_lo + (int64_t)a.m;
        const int64_t ql = (w_lo - (int64_t)(u0 + 31) + (int64_t)STRIDE - 1) / (int64_t)STRIDE;
        const int64_t qh = (w_hi - 1 - (int64_t)u0) / (int64_t)STRIDE;
        crt_qlo = ql < 0 ? 0 : (int)ql;
        const int qhi = qh > N1 - 1 ? N1 - 1 : (int)qh;
        crt_nq = qhi >= crt_qlo ? min(qhi - crt_qlo + 1, kCrtQ) : 0;
        const uint64_t off0 = (bb << a.logP) + u;
        uint32_t *d0 = crt_sm + (warp * 2 * kCrtQ) * 32 + lane;
        for (int j = 0; j < crt_nq; ++j) {
            const uint64_t off = off0 + (uint64_t)(crt_qlo + j) * STRIDE;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(d0 + j * 32)),
                         "l"(a.crt0 + off) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(d0 + (kCrtQ + j) * 32)),
                         "l"(a.crt1 + off) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    uint32_t x[N1];
    if (MODE == PASS_FWD_BITS || MODE == PASS_FWD_SEED) {
        // level 0, STRIDE >= 32: lanes hold 32 consecutive idx = q*STRIDE + u
        const int lane = threadIdx.x & 31;
        const uint32_t u0 = u & ~31u;
        const uint32_t *src = (MODE == PASS_FWD_BITS) ? a.bits + (a.b0 + bb) * (a.n >> 5) : a.bits;
        constexpr int NG = (N1 + 31) / 32;  // lane l fetches the words of q = l + 32 g
        uint32_t w[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            w[g] = 0;
            const uint32_t myidx = (uint32_t)(lane + 32 * g) * STRIDE + u0;
            if (lane + 32 * g < N1 && myidx < a.len) {
                uint32_t v = __ldg(src + (myidx >> 5));
                if (MODE == PASS_FWD_BITS) v = bswap32(v);  // seed words are already logical
                const uint32_t rem = a.len - myidx;         // mask bits past the input length
                if (rem < 32) v &= 0xFFFFFFFFu << (32 - rem);
                w[g] = v;
            }
        }
#pragma unroll
        for (int q = 0; q < N1; ++q) x[q] = (__shfl_sync(0xffffffffu, w[q >> 5], q & 31) >> (31 - lane)) & 1u;
    } else if (MODE == PASS_FWD_PACK) {
        // as PASS_FWD_BITS for each of the G <= 4 blocks of the group, combined
        // as sum_g cg[g] bit_g (< 4p, reduced to [0, 2p)); blocks past the
        // stream contribute nothing
        const int lane = threadIdx.x & 31;
        const uint32_t u0 = u & ~31u;
        constexpr int NG = (N1 + 31) / 32;
        // block by block, so only one block's words are live next to x[]
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint64_t blk = (a.b0 + bb) * a.G + (uint64_t)g;
            const bool have = (uint32_t)g < a.G && blk < a.n_blocks;
            const uint32_t *src = a.bits + blk * (a.n >> 5);
            uint32_t w[NG];
#pragma unroll
            for (int gg = 0; gg < NG; ++gg) {
                w[gg] = 0;
                const uint32_t myidx = (uint32_t)(lane + 32 * gg) * STRIDE + u0;
                if (have && lane + 32 * gg < N1 && myidx < a.len) {
                    uint32_t v = bswap32(__ldg(src + (myidx >> 5)));
                    const uint32_t rem = a.len - myidx;
                    if (rem < 32) v &= 0xFFFFFFFFu << (32 - rem);
                    w[gg] = v;
                }
            }
            const uint32_t c = a.cg[g];
#pragma unroll
            for (int q = 0; q < N1; ++q) {
                const uint32_t bit = (__shfl_sync(0xffffffffu, w[q >> 5], q & 31) >> (31 - lane)) & 1u;
                if (g == 0) x[q] = bit;  // cg[0] = 1
                else x[q] += bit ? c : 0u;
            }
        }
#pragma unroll
        for (int q = 0; q < N1; ++q) x[q] = red2<F>(x[q]);  // < 1 + 3 (p - 1) < 4p -> [0, 2p)
    } else {
#pragma unroll
        for (int q = 0; q < N1; ++q) x[q] = base[(size_t)q * STRIDE];
    }
    if (MODE <= PASS_FWD || MODE == PASS_FWD_PACK) {
        dft_fwd<R, F>(x);
        if (n2) twiddle<R, F>(x, __ldg(a.tw + ((uint64_t)n2 << a.S)));
#pragma unroll
        for (int q = 0; q < N1; ++q) base[(size_t)q * STRIDE] = x[q];
        return;
    }
    if (n2) twiddle<R, F>(x, __ldg(a.itw + ((uint64_t)n2 << a.S)));
    dft_inv<R, F>(x);
    if (MODE == PASS_INV) {
#pragma unroll
        for (int q = 0; q < N1; ++q) base[(size_t)q * STRIDE] = x[q];
        return;
    }
    // level 0 from here: element q is z_t with t = q*STRIDE + u
    const int lane = threadIdx.x & 31;
    const uint32_t u0 = u & ~31u;
    // the warp's t = q*STRIDE + u0..u0+31 meet the key window [len-1, len-1+m)
    // only for q in [q_lo, q_hi] (a third of the q at config 4): the others
    // skip the canonical residue, window test and ballot (warp-uniform)
    const int64_t w_lo = (int64_t)(a.len - 1), w_hi = w_lo + (int64_t)a.m;  // [w_lo, w_hi)
    const int64_t ql = (w_lo - (int64_t)(u0 + 31) + (int64_t)STRIDE - 1) / (int64_t)STRIDE;
    const int64_t qh = (w_hi - 1 - (int64_t)u0) / (int64_t)STRIDE;
    const int q_lo = ql < 0 ? 0 : (int)ql;
    const int q_hi = qh > N1 - 1 ? N1 - 1 : (int)qh;
    if constexpr (MODE == PASS_INV_CRT) {
        // packed form, third prime: with the first two primes' z_t, the CRT
        // value v mod 2^64 (Garner; v < kP kP2 kP3 exactly) holds block g's
        // window sum in bits [k g, k g + k): key bit = bit k g.  Lane (q & 31)
        // keeps the G ballots of its q; every 32 q each lane ORs its words in.
        using C = Crt;
        const uint64_t off0 = (bb << a.logP) + u;
        const uint32_t *s0 = crt_sm + ((threadIdx.x >> 5) * 2 * kCrtQ) * 32 + lane;
        asm volatile("cp.async.wait_all;" ::: "memory");  // this lane's own copies
        uint32_t mine4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < N1; ++q) {
            if (q >= q_lo && q <= q_hi) {
                const uint32_t t = (uint32_t)q * STRIDE + u;
                const int64_t i = (int64_t)t - (int64_t)(a.len - 1);
                const bool valid = i >= 0 && i < (int64_t)a.m;
                uint64_t v = 0;
                if (valid) {
                    const int j = q - crt_qlo;
                    uint32_t r0 = j < crt_nq ? s0[j * 32] : __ldcs(a.crt0 + off0 + (size_t)q * STRIDE);
                    uint32_t r1 = j < crt_nq ? s0[(kCrtQ + j) * 32] : __ldcs(a.crt1 + off0 + (size_t)q * STRIDE);
                    uint32_t r2 = x[q];
                    r0 = r0 >= (uint32_t)C::p0 ? r0 - (uint32_t)C::p0 : r0;
                    r1 = r1 >= (uint32_t)C::p1 ? r1 - (uint32_t)C::p1 : r1;
                    r2 = r2 >= (uint32_t)C::p2 ? r2 - (uint32_t)C::p2 : r2;
                    uint32_t r0m1 = r0 >= (uint32_t)C::p1 ? r0 - (uint32_t)C::p1 : r0;  // r0 < p0 < 3 p1
                    r0m1 = r0m1 >= (uint32_t)C::p1 ? r0m1 - (uint32_t)C::p1 : r0m1;
                    uint32_t y1 = shoup_p(r1 + (uint32_t)C::p1 - r0m1, C::c1, C::c1p, (uint32_t)C::p1);
                    y1 = y1 >= (uint32_t)C::p1 ? y1 - (uint32_t)C::p1 : y1;
                    const uint32_t r0m2 = shoup_p(r0, 1u, C::one2p, (uint32_t)C::p2);     // [0, 2 p2)
                    const uint32_t q02 = shoup_p(y1, C::p0m2, C::p0m2p, (uint32_t)C::p2);  // p0 y1 mod p2
                    uint32_t y2 = shoup_p(r2 + 4u * (uint32_t)C::p2 - r0m2 - q02, C::c2, C::c2p, (uint32_t)C::p2);
                    y2 = y2 >= (uint32_t)C::p2 ? y2 - (uint32_t)C::p2 : y2;
                    v = (uint64_t)r0 + C::p0 * (uint64_t)y1 + C::p01 * (uint64_t)y2;  // mod 2^64
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    uint32_t bit = (uint32_t)(v >> (a.crt_k * g)) & 1u;
                    const uint64_t blk = (a.b0 + bb) * a.G + (uint64_t)g;
                    if (a.xor_tail && valid && (uint32_t)g < a.G && blk < a.n_blocks)
                        bit ^= raw_bit(a.bits, blk, a.n, t + 1);  // identity block of [T | I_m]
                    const uint32_t bal = __ballot_sync(0xffffffffu, valid && bit);
                    if (lane == (q & 31)) mine4[g] = bal;
                }
            }
            if ((q & 31) == 31 || q == N1 - 1) {
                const int qb = q & ~31;
                if (lane <= (q & 31)) {
                    const int64_t i0 = (int64_t)(qb + lane) * STRIDE + u0 - (int64_t)(a.len - 1);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const uint64_t blk = (a.b0 + bb) * a.G + (uint64_t)g;
                        if (mine4[g] && (uint32_t)g < a.G && blk < a.n_blocks) {
                            const int64_t Gb = (int64_t)(blk * a.m) + i0;
                            const uint32_t V = __brev(mine4[g]);
                            const int64_t W0 = Gb >= 0 ? (Gb >> 5) : -((31 - Gb) >> 5);
                            const int o = (int)(Gb - W0 * 32);
                            const uint32_t hi = V >> o, lo = o ? (V << (32 - o)) : 0u;
                            if (hi) emit_word(a.out, (uint64_t)W0, hi, false);
                            if (lo) emit_word(a.out, (uint64_t)(W0 + 1), lo, false);
                        }
                    }
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) mine4[g] = 0;  // a skipped q of the next group leaves its words empty
            }
        }
        return;
    }
    // PASS_INV_EMIT[_XOR]
    uint32_t mine = 0;
#pragma unroll
    for (int q = 0; q < N1; ++q) {
        if (!QRNG_NTT_EMIT_SKIP || (q >= q_lo && q <= q_hi)) {
            const uint32_t t = (uint32_t)q * STRIDE + u;
            const int64_t i = (int64_t)t - (int64_t)(a.len - 1);
            const bool valid = i >= 0 && i < (int64_t)a.m;
            uint32_t z = x[q] >= P ? x[q] - P : x[q];
            if (MODE == PASS_INV_EMIT_XOR && valid) z ^= raw_bit(a.bits, a.b0 + bb, a.n, t + 1);  // identity block
            const uint32_t bal = __ballot_sync(0xffffffffu, valid && (z & 1u));
            if (lane == (q & 31)) mine = bal;
        }
        if ((q & 31) == 31 || q == N1 - 1) {
            const int qb = q & ~31;
            if (lane <= (q & 31) && mine) {
                const int64_t i0 = (int64_t)(qb + lane) * STRIDE + u0 - (int64_t)(a.len - 1);
                const int64_t G = (int64_t)((a.b0 + bb) * a.m) + i0;
                const uint32_t V = __brev(mine);
                const int64_t W0 = G >= 0 ? (G >> 5) : -((31 - G) >> 5);
                const int o = (int)(G - W0 * 32);
                const uint32_t hi = V >> o, lo = o ? (V << (32 - o)) : 0u;
                if (hi) emit_word(a.out, (uint64_t)W0, hi, false);
                if (lo) emit_word(a.out, (uint64_t)(W0 + 1), lo, false);
            }
            mine = 0;  // a skipped q of the next group leaves its lane's word empty
        }
    }
}

template <int LOGP, bool PACK>
__global__ void __launch_bounds__(threads_of(LOGP), 1024 / threads_of(LOGP)) ntt_fused_kernel(FusedArgs a) {
    extern __shared__ uint32_t smem[];
    constexpr int PP = 1 << LOGP;
    uint32_t *data = smem;
    uint32_t *stage = smem + PP + PP / 32;
    const int per = PACK ? 2 : 1;
    const uint64_t b0 = (uint64_t)blockIdx.x * per;
    const int nb = (int)min((uint64_t)per, a.n_blocks - b0);
    const uint64_t g_lo = b0 * a.m, g_hi = (b0 + nb) * a.m;  // [g_lo, g_hi)
    const uint64_t wfirst = g_lo >> 5, wlast = (g_hi - 1) >> 5;
    for (uint32_t i = threadIdx.x; i < a.stage_words; i += blockDim.x) stage[i] = 0;
    __syncthreads();
    run_levels<LOGP, 0, PACK>(data, stage, a, b0, nb, wfirst);
    for (uint64_t w = wfirst + threadIdx.x; w <= wlast; w += blockDim.x) {
        bool excl = (w << 5) >= g_lo && ((w << 5) + 31) < g_hi;
        emit_word(a.out, w, stage[w - wfirst], excl);
    }
}

// ---- plan preparation kernels ----------------------------------------------

// tw[e] = w^e * 2^32 mod p, itw[e] = w^-e * 2^32 mod p for e < P (Montgomery
// form): per thread a first power by Montgomery square-and-multiply, then a
// Montgomery chain (mont(x * R, w * R) = x w R), canonicalised.  (Round 2:
// ~16 exponents per thread and Montgomery powers instead of 64 and a
// 64-bit-modulo power -- the table build was 29 us at P = 2^21, once per
// prime of a one-shot plan.)
constexpr uint32_t kTwChain = 64;  // exponents per thread (the per-thread start powers dominate at 16)
// x^e in Montgomery form (xM = x 2^32 mod p), canonical
template <int F>
__device__ __forceinline__ uint32_t mont_pow(uint32_t xM, uint32_t e) {
    constexpr uint32_t P = Fld<F>::P;
    uint32_t r = (uint32_t)((1ull << 32) % P);  // 1 in Montgomery form
    for (; e; e >>= 1) {  // square-and-multiply, lazy residues in (0, 2p)
        if (e & 1) r = mont<F>(r, xM);
        xM = mont<F>(xM, xM);
    }
    return r >= P ? r - P : r;
}
// Thread t of T takes exponents t, t + T, t + 2T, ... (kTwChain of
// them), so every store instruction of a warp writes 32 consecutive words
// (with chains of consecutive exponents per thread the warp's stores were 64
// bytes apart: 329 us for the two 128 MB tables at P = 2^25).
template <int F = 0>
__global__ void twiddle_table_kernel(uint32_t *tw, uint32_t *itw, uint32_t Pn, uint32_t w, uint32_t iw) {
    constexpr uint32_t P = Fld<F>::P;
    const uint32_t T = gridDim.x * blockDim.x;
    const uint32_t e0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (e0 >= Pn) return;
    const uint32_t wM = (uint32_t)(((uint64_t)w << 32) % P), iwM = (uint32_t)(((uint64_t)iw << 32) % P);
    uint32_t a = mont_pow<F>(wM, e0), b = mont_pow<F>(iwM, e0);
    const uint32_t sa = mont_pow<F>(wM, T), sb = mont_pow<F>(iwM, T);  // w^T, w^-T
    for (uint32_t e = e0; e < Pn; e += T) {
        tw[e] = a;
        itw[e] = b;
        a = mont<F>(a, sa);
        a = a >= P ? a - P : a;
        b = mont<F>(b, sb);
        b = b >= P ? b - P : b;
    }
}

// The segment kernel's level-1 twiddles (2^15-word segments): l1[dir][k][n2] =
// (w, floor(w 2^32 / p)), w = w_P^(+-(k n2 2^5) << tw_shift), from the Montgomery tables.
template <int F = 0>
__global__ void l1tw_kernel(uint2 *out, const uint32_t *tw, const uint32_t *itw, uint32_t tw_shift, uint32_t Pmask) {
    constexpr uint32_t P = Fld<F>::P;
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= 2048) return;
    const uint32_t dir = idx >> 10, k = (idx >> 5) & 31, n2 = idx & 31;
    const uint32_t e = ((k * n2) << 5 << tw_shift) & Pmask;
    uint32_t w = mont<F>((dir ? itw : tw)[e], 1u);  // out of Montgomery form, in (0, 2p)
    w = w >= P ? w - P : w;
    out[idx] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / P));
}

// Seed spectrum, fused single-CTA version (P <= 2^15): forward passes only.
template <int LOGP, int LV>
__device__ __forceinline__ void seed_levels(uint32_t *data, const uint32_t *seed_words, uint32_t L,
                                            const uint32_t *tw, uint32_t *shat, uint32_t scaleM) {
    constexpr int R = radix_of(LOGP, LV), S = prefix_of(LOGP, LV), N1 = 1 << R;
    constexpr int STRIDE = (1 << LOGP) >> (S + R), NSEG = (1 << LOGP) >> S, NSUB = (1 << LOGP) >> R;
    constexpr bool LAST = (LV == np_of(LOGP) - 1);
    for (int u = threadIdx.x; u < NSUB; u += blockDim.x) {
        uint32_t x[N1];
        const int seg = u / STRIDE, n2 = u % STRIDE;
#pragma unroll
        for (int q = 0; q < N1; ++q) {
            int idx = seg * NSEG + q * STRIDE + n2;
            if (LV == 0) {
                uint32_t v = 0;
                if ((uint32_t)idx < L) v = (seed_words[idx >> 5] >> (31 - (idx & 31))) & 1u;
                x[q] = v;
            } else {
                x[q] = data[pidx(idx)];
            }
        }
        dft_fwd<R>(x);
        if (!LAST) {
            if (n2) twiddle<R>(x, tw[n2 << S]);
#pragma unroll
            for (int q = 0; q < N1; ++q) data[pidx(seg * NSEG + q * STRIDE + n2)] = x[q];
        } else {
            static_assert(N1 % 4 == 0, "last level radix >= 4");
#pragma unroll
            for (int q4 = 0; q4 < N1 / 4; ++q4)  // * P^-1 * 2^32
                reinterpret_cast<uint4 *>(shat)[shat4_idx<N1, NSUB>(u, q4)] =
                    make_uint4(mont(x[4 * q4], scaleM), mont(x[4 * q4 + 1], scaleM), mont(x[4 * q4 + 2], scaleM),
                               mont(x[4 * q4 + 3], scaleM));
        }
    }
    __syncthreads();
    if constexpr (!LAST) seed_levels<LOGP, LV + 1>(data, seed_words, L, tw, shat, scaleM);
}

template <int LOGP>
__global__ void __launch_bounds__(threads_of(LOGP)) seed_fused_kernel(const uint32_t *seed_words, uint32_t L,
                                                                      const uint32_t *tw, uint32_t *shat,
                                                                      uint32_t scaleM) {
    extern __shared__ uint32_t smem[];
    seed_levels<LOGP, 0>(smem, seed_words, L, tw, shat, scaleM);
}

// Seed bits [off, off + L) of an MSB-first byte buffer -> logical big-endian
// words (bit k at 31-(k&31) of word k>>5), zero past L.  off = 1 drops a_1 for
// the modified Toeplitz (its T uses a_2..a_n).
__global__ void seed_words_kernel(const uint8_t *seed, uint64_t L, uint32_t off, uint32_t *words,
                                  uint64_t nwords) {
    const uint64_t nbytes = (off + L + 7) / 8;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pos = off + w * 32, b0 = pos / 8;
        uint64_t v = 0;  // 40 bits starting at byte b0
        for (int k = 0; k < 5; ++k) v = (v << 8) | (b0 + k < nbytes ? seed[b0 + k] : 0u);
        uint32_t r = (uint32_t)(v >> (8 - (pos & 7)));
        const uint64_t lo = w * 32;  // mask bits >= L
        if (lo + 32 > L) r &= (L > lo) ? (0xFFFFFFFFu << (32 - (L - lo))) : 0u;
        words[w] = r;
    }
}

// ---- host side -------------------------------------------------------------
int choose_pack_shift(uint64_t n, int logP) {
    (void)logP;
    int shift = 0;
    while ((1ull << shift) <= n) ++shift;  // 2^shift > n >= any window sum
    if ((unsigned __int128)n * ((1ull << shift) + 1) >= P) return 0;
    return shift;
}

template <int LOGP, bool PACK>
static qrng_status launch_fused(const FusedArgs &a, cudaStream_t s) {
    const int per = PACK ? 2 : 1;
    const size_t smem = ((size_t)(1 << LOGP) + (1 << LOGP) / 32 + a.stage_words) * 4;
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(ntt_fused_kernel<LOGP, PACK>));
        if (st != QRNG_OK) return st;
    }
    uint64_t grid = (a.n_blocks + per - 1) / per;
    KernelTimer t(s, true);
    ntt_fused_kernel<LOGP, PACK><<<(unsigned)grid, threads_of(LOGP), smem, s>>>(a);
    t.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

template <int LOGP>
static qrng_status launch_seed(const uint32_t *seed_words, uint32_t L, const uint32_t *tw,
                               uint32_t *shat, uint32_t scaleM, cudaStream_t s) {
    const size_t smem = ((size_t)(1 << LOGP) + (1 << LOGP) / 32) * 4;
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(seed_fused_kernel<LOGP>));
        if (st != QRNG_OK) return st;
    }
    count_launch();
    seed_fused_kernel<LOGP><<<1, threads_of(LOGP), smem, s>>>(seed_words, L, tw, shat, scaleM);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

#define QRNG_LOGP_CASES(X) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)


// ---- butterfly-rate microbenchmark (the NTT roofline denominator) ----------
// Register-resident radix-32 forward DIF + inverse DIT with the exact butterfly
// code of the kernels above (Shoup with constant-bank roots, lazy [0, 2p)
// reductions, 49 of 80 butterflies per DFT non-trivial), repeated `iters` times
// per thread on every SM; no memory traffic inside the loop.  Counted work:
// 160 radix-2 butterflies per iteration per thread.
__global__ void __launch_bounds__(512, 2) butterfly_rate_kernel(uint32_t *sink, int iters) {
    uint32_t x[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) x[q] = (threadIdx.x * 32u + q) % P;
    for (int it = 0; it < iters; ++it) {
        dft_fwd<5>(x);
        dft_inv<5>(x);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) acc ^= x[q];
    if (acc == 0xFFFFFFFFu) sink[0] = acc;  // keep the work alive
}

// Same loop with each DFT followed by the inter-pass twiddle (twiddle<5>, the
// Montgomery power chains every non-final pass of the transforms runs): the
// rate of the passes' full register-resident instruction mix.  Counted work is
// still 160 butterflies per iteration, so the two rates compare directly.
__global__ void __launch_bounds__(512, 2) pass_rate_kernel(uint32_t *sink, int iters) {
    uint32_t x[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) x[q] = (threadIdx.x * 32u + q) % P;
    for (int it = 0; it < iters; ++it) {
        dft_fwd<5>(x);
        twiddle<5>(x, c_roots[0].w[(it & 31) + 1]);
        dft_inv<5>(x);
        twiddle<5>(x, c_roots[0].iw[(it & 31) + 1]);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) acc ^= x[q];
    if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

qrng_status butterfly_rate(int iters, uint64_t *butterflies, cudaStream_t s, bool with_twiddles) {
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    uint32_t *sink = nullptr;
    QRNG_CUDA_TRY(cudaMallocAsync(&sink, 4, s));
    const unsigned grid = (unsigned)sms * 2, block = 512;
    count_launch();
    if (with_twiddles)
        pass_rate_kernel<<<grid, block, 0, s>>>(sink, iters);
    else
        butterfly_rate_kernel<<<grid, block, 0, s>>>(sink, iters);
    QRNG_CUDA_TRY(cudaGetLastError());
    cudaFreeAsync(sink, s);
    *butterflies = (uint64_t)grid * block * (uint64_t)iters * 160u;
    return QRNG_OK;
}

// ---- multi-pass launch helpers ---------------------------------------------
// Global radices for P = 2^logP > 2^15: g = logP - 15 levels before the segments.
static int global_radices(int logP, int r[2]) {
    const int g = logP - kSegLog;
    if (g <= 6) { r[0] = g; return 1; }
    r[0] = g - g / 2;
    r[1] = g / 2;
    return 2;
}

template <int MODE, int F = 0>
static qrng_status launch_pass(int R, const PassArgs &a, uint64_t nb, cudaStream_t s, bool timed) {
    const uint64_t nsub = 1ull << (a.logP - R);
    dim3 grid((unsigned)(nsub / 256), (unsigned)nb);
    const size_t smem = MODE == PASS_INV_CRT ? (size_t)8 * 2 * kCrtQ * 32 * 4 : 0;
    if (smem) {
        qrng_status st = QRNG_OK;
        switch (R) {
#define X(RR) case RR: st = allow_max_smem(reinterpret_cast<const void *>(ntt_pass_kernel<RR, MODE, F>)); break;
            X(1) X(2) X(3) X(4) X(5) X(6)
#undef X
            default: break;
        }
        if (st != QRNG_OK) return st;
    }
    KernelTimer t(s, timed);
    switch (R) {
#define X(RR) case RR: ntt_pass_kernel<RR, MODE, F><<<grid, 256, smem, s>>>(a); break;
        X(1) X(2) X(3) X(4) X(5) X(6)
#undef X
        default:
            set_error("NTT pass radix 2^%d unsupported", R);
            return QRNG_E_UNSUPPORTED;
    }
    t.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

template <int MODE, int F = 0, int LOGS = kSegLog>
static qrng_status launch_segments(const FusedArgs &a, uint32_t *ws, int logP, uint64_t nb, cudaStream_t s,
                                   bool timed) {
    const size_t smem = ((size_t)(1 << LOGS) + (1 << LOGS) / 32) * 4 + ((MODE == SEG && LOGS == 15) ? 2048 * 8 : 0);
    {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(ntt_segment_kernel<LOGS, MODE, F>));
        if (st != QRNG_OK) return st;
    }
    dim3 grid((unsigned)(1u << (logP - LOGS)), (unsigned)nb);
    KernelTimer t(s, timed);
    ntt_segment_kernel<LOGS, MODE, F><<<grid, threads_of(LOGS), smem, s>>>(a, ws, (uint32_t)logP);
    t.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

// per-prime tables of a plan: seed spectrum and twiddles
struct FieldTabs {
    uint32_t **shat, **tw, **itw;
    uint2 **l1tw;
};

template <int F>
static qrng_status seed_multipass(const FieldTabs &ft, const uint32_t *seed_words, uint64_t n, uint64_t m, uint64_t L,
                                  int logP, uint32_t scaleM, cudaStream_t s);

// twiddle tables, level-1 table and seed spectrum of field F for P = 2^logP
template <int F>
static qrng_status init_field(const FieldTabs &ft, const uint32_t *seed_words, uint64_t n, uint64_t m, uint64_t L,
                              int logP, cudaStream_t s) {
    const uint64_t Pf = Fld<F>::P, Pn = 1ull << logP;
    QRNG_CUDA_TRY(cudaMallocAsync(ft.shat, Pn * 4, s));
    QRNG_CUDA_TRY(cudaMallocAsync(ft.tw, Pn * 4, s));
    QRNG_CUDA_TRY(cudaMallocAsync(ft.itw, Pn * 4, s));
    const uint64_t w = powmod_p(3, (Pf - 1) >> logP, Pf), iw = powmod_p(w, Pf - 2, Pf);
    count_launch();
    twiddle_table_kernel<F><<<(unsigned)(((Pn + kTwChain - 1) / kTwChain + 127) / 128), 128, 0, s>>>(*ft.tw, *ft.itw, (uint32_t)Pn,
                                                                                   (uint32_t)w, (uint32_t)iw);
    QRNG_CUDA_TRY(cudaGetLastError());
    if (logP > kMaxFusedLogP && kSegLog == 15) {  // the segment kernel's level-1 twiddles
        QRNG_CUDA_TRY(cudaMallocAsync(ft.l1tw, 2048 * sizeof(uint2), s));
        count_launch();
        const uint32_t shift = (uint32_t)(logP - kSegLog), mask = (uint32_t)(Pn - 1);
        l1tw_kernel<F><<<8, 256, 0, s>>>(*ft.l1tw, *ft.tw, *ft.itw, shift, mask);
        QRNG_CUDA_TRY(cudaGetLastError());
    }
    // scale = P^-1 * 2^64 mod p, so mont(v, scale) = v * P^-1 * 2^32 (Montgomery form for the pointwise product)
    const uint64_t pinvP = powmod_p(Pn % Pf, Pf - 2, Pf);
    const uint64_t r2 = (uint64_t)(((unsigned __int128)1 << 64) % Pf);
    const uint32_t scaleM = (uint32_t)((unsigned __int128)pinvP * r2 % Pf);
    if (logP > kMaxFusedLogP) return seed_multipass<F>(ft, seed_words, n, m, L, logP, scaleM, s);
    if constexpr (F == 0) {
        switch (logP) {
#define X(LP) case LP: return launch_seed<LP>(seed_words, (uint32_t)L, *ft.tw, *ft.shat, scaleM, s);
            QRNG_LOGP_CASES(X)
#undef X
            default: break;
        }
    }
    set_error("NTT plan: no transform for P = 2^%d", logP);
    return QRNG_E_UNSUPPORTED;
}

// Packed three-prime form: G blocks per transform as v = sum_g 2^(k g) x_g,
// k = bit length of n (every window sum c_g <= n < 2^k, so the convolution of v
// with the seed holds each c_g in its own k-bit field), transformed modulo
// each of kP, kP2, kP3 and recombined by CRT (M = kP kP2 kP3 > 2^86 > max v).
// Pays when G >= 4 (4 blocks for 3 transforms per direction): n < 2^21 with
// (G - 1) k <= 63 (the key bits 0, k, 2k, 3k are read from v mod 2^64).
// Multi-pass sizes from P = 2^17 to 2^23; QRNG_NTT_CRT=0 disables it.
int choose_crt(uint64_t n, int logP, bool /*xor_tail: the CRT pass XORs the identity block too*/, uint32_t *k_out) {
    static const bool on = [] {
        const char *e = getenv("QRNG_NTT_CRT");
        return !(e && *e && atoi(e) == 0);
    }();
    // P = 2^16 (one global pass of radix 2, 2 segments): measured slower packed
    // (modified config 3: 78.1 -> 72.1 Gbit/s), so from P = 2^17
    if (!on || logP < kMaxFusedLogP + 2 || logP > kMaxLogP) return 0;
    uint32_t k = 0;
    while ((1ull << k) <= n) ++k;  // 2^k > n
    const long double M = (long double)kP * kP2 * kP3;
    int G = 1;
    while (G < 4 && (uint64_t)G * k <= 63) {
        long double vmax = 0;  // n * sum_{g <= G} 2^(k g)
        for (int g = 0; g <= G; ++g) vmax += ldexpl((long double)n, (int)(k * g));
        if (vmax >= M * 0.999L) break;
        ++G;
    }
    if (G < 4) return 0;
    *k_out = k;
    return G;
}

qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t seed_bit_offset,
                      bool xor_tail, cudaStream_t s) {
    // n here is the number of raw bits per block that enter the product
    // (n, or n - m for the modified Toeplitz, whose seed starts at bit 1)
    const uint64_t L = n + m - 1;
    pl.len = (uint32_t)n;
    pl.xor_tail = xor_tail;
    int logP = 0;
    while ((1ull << logP) < L) ++logP;
    if (logP < 5) logP = 5;
    // P <= 2^23: p = 119 * 2^23 + 1; 2^23 < P <= 2^26: p = 7 * 2^26 + 1 (its
    // 2-adic limit), same kernels (multi-pass: P > 2^15 here)
    pl.field = logP > kMaxLogP ? 1 : 0;
    if (logP > kMaxLogP2) {
        set_error("NTT path: L = %llu exceeds 2^26", (unsigned long long)L);
        return QRNG_E_UNSUPPORTED;
    }
    pl.logP = logP;
    pl.pack_shift = logP <= kMaxFusedLogP ? choose_pack_shift(n, logP) : 0;  // window sums <= n
    pl.crt = choose_crt(n, logP, xor_tail, &pl.crt_k);
    const uint64_t nwords = (L + 31) / 32 + 1;
    uint32_t *seed_words = nullptr;
    QRNG_CUDA_TRY(cudaMallocAsync(&seed_words, nwords * 4, s));
    count_launch();
    seed_words_kernel<<<(unsigned)((nwords + 255) / 256), 256, 0, s>>>(d_seed, L, seed_bit_offset, seed_words,
                                                                      nwords);
    QRNG_CUDA_TRY(cudaGetLastError());
    qrng_status st;
    if (pl.crt) {
        // the three primes' tables on three streams (the caller's, the side
        // stream and a third of this thread's): each chain is a few small
        // launches (a seed-spectrum segment launch is P / 2^15 CTAs), so they
        // fill the SMs together
        cudaStream_t s2, s3;
        cudaEvent_t fork, join;
        st = side_stream(&s2, &fork, &join);
        if (st != QRNG_OK) return st;
        static thread_local cudaStream_t t3 = nullptr;
        static thread_local cudaEvent_t j3 = nullptr;
        static thread_local int t3dev = -1;
        int dev = 0;
        QRNG_CUDA_TRY(cudaGetDevice(&dev));
        if (t3dev != dev) {  // (a stream per device and thread, as side_stream)
            if (t3) { cudaStreamDestroy(t3); cudaEventDestroy(j3); }
            t3 = nullptr;
            QRNG_CUDA_TRY(cudaStreamCreateWithFlags(&t3, cudaStreamNonBlocking));
            QRNG_CUDA_TRY(cudaEventCreateWithFlags(&j3, cudaEventDisableTiming));
            t3dev = dev;
        }
        s3 = t3;
        QRNG_CUDA_TRY(cudaEventRecord(fork, s));
        QRNG_CUDA_TRY(cudaStreamWaitEvent(s2, fork, 0));
        QRNG_CUDA_TRY(cudaStreamWaitEvent(s3, fork, 0));
        st = init_field<1>(FieldTabs{&pl.shat3[1], &pl.tw3[1], &pl.itw3[1], &pl.l1tw3[1]}, seed_words, n, m, L, logP, s2);
        const qrng_status st2 =
            init_field<2>(FieldTabs{&pl.shat3[2], &pl.tw3[2], &pl.itw3[2], &pl.l1tw3[2]}, seed_words, n, m, L, logP, s3);
        const qrng_status st0 =
            init_field<0>(FieldTabs{&pl.shat3[0], &pl.tw3[0], &pl.itw3[0], &pl.l1tw3[0]}, seed_words, n, m, L, logP, s);
        cudaEventRecord(join, s2);  // always joined: seed_words is freed on s below
        cudaStreamWaitEvent(s, join, 0);
        cudaEventRecord(j3, s3);
        cudaStreamWaitEvent(s, j3, 0);
        if (st == QRNG_OK) st = st2;
        if (st == QRNG_OK) st = st0;
    } else {
        const FieldTabs ft{&pl.shat, &pl.tw, &pl.itw, &pl.l1tw};
        st = pl.field ? init_field<1>(ft, seed_words, n, m, L, logP, s) : init_field<0>(ft, seed_words, n, m, L, logP, s);
    }
    cudaFreeAsync(seed_words, s);
    return st;
}

// seed spectrum through the multi-pass decomposition, forward only
template <int F>
static qrng_status seed_multipass(const FieldTabs &ft, const uint32_t *seed_words, uint64_t n, uint64_t m, uint64_t L,
                                  int logP, uint32_t scaleM, cudaStream_t s) {
    const uint64_t Pn = 1ull << logP;
    qrng_status st = QRNG_OK;
    {
        uint32_t *ws = nullptr;
        QRNG_CUDA_TRY(cudaMallocAsync(&ws, Pn * 4, s));
        int r[2];
        const int np = global_radices(logP, r);
        PassArgs pa{};
        pa.bits = seed_words;
        pa.b0 = 0;
        pa.n = (uint32_t)n;
        pa.m = (uint32_t)m;
        pa.len = (uint32_t)L;
        pa.ws = ws;
        pa.tw = *ft.tw;
        pa.itw = *ft.itw;
        pa.logP = (uint32_t)logP;
        pa.S = 0;
        st = launch_pass<PASS_FWD_SEED, F>(r[0], pa, 1, s, false);
        if (st == QRNG_OK && np == 2) {
            pa.S = (uint32_t)r[0];
            st = launch_pass<PASS_FWD, F>(r[1], pa, 1, s, false);
        }
        if (st == QRNG_OK) {
            FusedArgs fa{};
            fa.shat = *ft.shat;
            fa.tw = *ft.tw;
            fa.itw = *ft.itw;
            fa.tw_shift = (uint32_t)(logP - kSegLog);
            fa.scaleM = scaleM;
            st = launch_segments<SEGFWD, F>(fa, ws, logP, 1, s, false);
        }
        cudaFreeAsync(ws, s);
    }
    return st;
}

void plan_free(Plan &pl) {
    for (void *ptr : {(void *)pl.shat, (void *)pl.tw, (void *)pl.itw, (void *)pl.l1tw, (void *)pl.work})
        if (ptr) cudaFree(ptr);
    for (int f = 0; f < 3; ++f)
        for (void *ptr : {(void *)pl.shat3[f], (void *)pl.tw3[f], (void *)pl.itw3[f], (void *)pl.l1tw3[f]})
            if (ptr) cudaFree(ptr);
    pl = Plan{};
}

template <int F>
static qrng_status extract_multipass(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n,
                                     uint64_t m, const OutStream &out, cudaStream_t s) {
    const int logP = pl.logP;
    // two batches in flight (one per stream), each half the L2-sized budget
    static const int kBatchLog = [] {  // QRNG_NTT_BATCH_LOG: workspace words per batch (experiments)
        const char *e = getenv("QRNG_NTT_BATCH_LOG");
        const int v = e ? atoi(e) : 0;
        return v >= 18 && v <= 27 ? v : 26;
    }();
    uint64_t bb = (1ull << kBatchLog) >> logP;  // 2^26-word (256 MiB) workspace per batch by default
    if (bb < 1) bb = 1;
    if (bb > n_blocks) bb = n_blocks;
    const bool two = n_blocks > bb;
    cudaStream_t s2 = s;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (two) {
        qrng_status st2 = side_stream(&s2, &fork, &join);
        if (st2 != QRNG_OK) return st2;
    }
    uint32_t *wsb[2] = {nullptr, nullptr};
    QRNG_CUDA_TRY(cudaMallocAsync(&wsb[0], (bb << logP) * 4, s));
    if (two) {
        QRNG_CUDA_TRY(cudaMallocAsync(&wsb[1], (bb << logP) * 4, s));
        QRNG_CUDA_TRY(cudaEventRecord(fork, s));
        QRNG_CUDA_TRY(cudaStreamWaitEvent(s2, fork, 0));
    }
    uint32_t *ws = wsb[0];
    const cudaStream_t s_main = s;
    int r[2];
    const int np = global_radices(logP, r);
    PassArgs pa{};
    pa.bits = reinterpret_cast<const uint32_t *>(d_raw);
    pa.n = (uint32_t)n;  // block stride
    pa.m = (uint32_t)m;
    pa.len = pl.len;     // bits per block that enter the product
    pa.xor_tail = pl.xor_tail ? 1u : 0u;
    pa.ws = ws;
    pa.tw = pl.tw;
    pa.itw = pl.itw;
    pa.logP = (uint32_t)logP;
    pa.out = out;
    FusedArgs fa{};
    fa.shat = pl.shat;
    fa.tw = pl.tw;
    fa.itw = pl.itw;
    fa.tw_shift = (uint32_t)(logP - kSegLog);
    static const bool use_l1 = [] {  // QRNG_NTT_L1TW=0: the Montgomery chains at level 1 (A/B)
        const char *e = getenv("QRNG_NTT_L1TW");
        return !(e && *e && atoi(e) == 0);
    }();
    fa.l1tw = use_l1 ? pl.l1tw : nullptr;
    qrng_status st = QRNG_OK;
    for (uint64_t b0 = 0, it = 0; b0 < n_blocks && st == QRNG_OK; b0 += bb, ++it) {
        const uint64_t nb = (n_blocks - b0) < bb ? (n_blocks - b0) : bb;
        const cudaStream_t s = (it & 1) ? s2 : s_main;
        ws = wsb[it & 1];
        pa.ws = ws;
        pa.b0 = b0;
        pa.S = 0;
        st = launch_pass<PASS_FWD_BITS, F>(r[0], pa, nb, s, true);
        if (st == QRNG_OK && np == 2) {
            pa.S = (uint32_t)r[0];
            st = launch_pass<PASS_FWD, F>(r[1], pa, nb, s, true);
        }
        if (st == QRNG_OK) st = launch_segments<SEG, F>(fa, ws, logP, nb, s, true);
        if (st == QRNG_OK && np == 2) {
            pa.S = (uint32_t)r[0];
            st = launch_pass<PASS_INV, F>(r[1], pa, nb, s, true);
        }
        if (st == QRNG_OK) {
            pa.S = 0;
            st = pl.xor_tail ? launch_pass<PASS_INV_EMIT_XOR, F>(r[0], pa, nb, s, true)
                             : launch_pass<PASS_INV_EMIT, F>(r[0], pa, nb, s, true);
        }
    }
    if (two) {  // join the side stream back before the workspaces are released
        cudaEventRecord(join, s2);
        cudaStreamWaitEvent(s_main, join, 0);
        cudaFreeAsync(wsb[1], s_main);
    }
    cudaFreeAsync(wsb[0], s_main);
    return st;
}

// Packed three-prime form: per batch of groups (G blocks each), for each prime
// the forward passes (the first forming the packed input), segments and
// inverse passes down to natural order in that prime's workspace, then the CRT
// kernel.  Batches alternate between two streams as in extract_multipass.
template <int F>
static qrng_status crt_prime(const Plan &pl, PassArgs pa, FusedArgs fa, int logP, uint64_t nb, cudaStream_t s) {
    int r[2];
    const int np = global_radices(logP, r);
    const uint64_t Pf = Fld<F>::P;
    for (int g = 0; g < 4; ++g) pa.cg[g] = (uint32_t)powmod_p(2, (uint64_t)pl.crt_k * g, Pf);
    pa.tw = pl.tw3[F];
    pa.itw = pl.itw3[F];
    fa.shat = pl.shat3[F];
    fa.tw = pl.tw3[F];
    fa.itw = pl.itw3[F];
    fa.l1tw = pl.l1tw3[F];
    pa.S = 0;
    qrng_status st = launch_pass<PASS_FWD_PACK, F>(r[0], pa, nb, s, true);
    if (st == QRNG_OK && np == 2) {
        pa.S = (uint32_t)r[0];
        st = launch_pass<PASS_FWD, F>(r[1], pa, nb, s, true);
    }
    if (st == QRNG_OK) st = launch_segments<SEG, F>(fa, pa.ws, logP, nb, s, true);
    if (st == QRNG_OK && np == 2) {
        pa.S = (uint32_t)r[0];
        st = launch_pass<PASS_INV, F>(r[1], pa, nb, s, true);
    }
    if (st == QRNG_OK) {  // natural order: z_t (F < 2), or CRT + key bits (F = 2)
        pa.S = 0;
        // (storing only the window's q spills at any launch bound for radix 64)
        if constexpr (F < 2) st = launch_pass<PASS_INV, F>(r[0], pa, nb, s, true);
        else st = launch_pass<PASS_INV_CRT, F>(r[0], pa, nb, s, true);
    }
    return st;
}

static qrng_status extract_crt(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                               const OutStream &out, cudaStream_t s) {
    const int logP = pl.logP;
    const uint64_t G = (uint64_t)pl.crt, groups = (n_blocks + G - 1) / G;
    static const int kBatchLog = [] {  // as extract_multipass: workspace words per batch (all three primes)
        const char *e = getenv("QRNG_NTT_BATCH_LOG");
        const int v = e ? atoi(e) : 0;
        return v >= 18 && v <= 27 ? v : 26;
    }();
    // groups per batch: a 2^28-word budget over the three primes (4 GB in all
    // on two streams at most) -- the 2^26 of the one-prime form would leave
    // the segment launches a few waves long, and their tails cost ~15%
    uint64_t bb = ((1ull << (kBatchLog + 2)) >> logP) / 3;
    if (bb < 1) bb = 1;
    if (bb > groups) bb = groups;
    const bool two = groups > bb;
    cudaStream_t s2 = s;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (two) {
        qrng_status st2 = side_stream(&s2, &fork, &join);
        if (st2 != QRNG_OK) return st2;
    }
    const uint64_t wsw = bb << logP;  // words per prime per batch
    uint32_t *wsb[2] = {nullptr, nullptr};
    QRNG_CUDA_TRY(cudaMallocAsync(&wsb[0], 3 * wsw * 4, s));
    if (two) {
        QRNG_CUDA_TRY(cudaMallocAsync(&wsb[1], 3 * wsw * 4, s));
        QRNG_CUDA_TRY(cudaEventRecord(fork, s));
        QRNG_CUDA_TRY(cudaStreamWaitEvent(s2, fork, 0));
    }
    PassArgs pa{};
    pa.bits = reinterpret_cast<const uint32_t *>(d_raw);
    pa.n = (uint32_t)n;
    pa.m = (uint32_t)m;
    pa.len = pl.len;
    pa.logP = (uint32_t)logP;
    pa.out = out;
    pa.G = (uint32_t)G;
    pa.n_blocks = n_blocks;
    pa.crt_k = pl.crt_k;
    pa.xor_tail = pl.xor_tail ? 1u : 0u;  // modified Toeplitz: the CRT pass XORs raw bit t + 1
    FusedArgs fa{};
    fa.tw_shift = (uint32_t)(logP - kSegLog);
    qrng_status st = QRNG_OK;
    for (uint64_t g0 = 0, it = 0; g0 < groups && st == QRNG_OK; g0 += bb, ++it) {
        const uint64_t nb = (groups - g0) < bb ? (groups - g0) : bb;
        const cudaStream_t sb = (it & 1) ? s2 : s;
        uint32_t *ws = wsb[it & 1];
        pa.b0 = g0;
        pa.ws = ws;
        st = crt_prime<0>(pl, pa, fa, logP, nb, sb);
        pa.ws = ws + wsw;
        if (st == QRNG_OK) st = crt_prime<1>(pl, pa, fa, logP, nb, sb);
        pa.ws = ws + 2 * wsw;
        pa.crt0 = ws;
        pa.crt1 = ws + wsw;
        if (st == QRNG_OK) st = crt_prime<2>(pl, pa, fa, logP, nb, sb);
    }
    if (two) {
        cudaEventRecord(join, s2);
        cudaStreamWaitEvent(s, join, 0);
        cudaFreeAsync(wsb[1], s);
    }
    cudaFreeAsync(wsb[0], s);
    return st;
}

qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                    const OutStream &out, cudaStream_t s) {
    if (pl.crt) return extract_crt(pl, d_raw, n_blocks, n, m, out, s);
    if (pl.logP > kMaxFusedLogP)
        return pl.field ? extract_multipass<1>(pl, d_raw, n_blocks, n, m, out, s)
                        : extract_multipass<0>(pl, d_raw, n_blocks, n, m, out, s);
    FusedArgs a{};
    a.raw = reinterpret_cast<const uint32_t *>(d_raw);
    a.n_blocks = n_blocks;
    a.n = (uint32_t)n;
    a.m = (uint32_t)m;
    a.shift = pl.pack_shift;
    a.shat = pl.shat;
    a.tw = pl.tw;
    a.itw = pl.itw;
    a.out = out;
    a.tw_shift = 0;
    a.len = pl.len;
    a.xor_tail = pl.xor_tail ? 1u : 0u;
    const int per = pl.pack_shift ? 2 : 1;
    a.stage_words = (uint32_t)((per * m + 31) / 32 + 2);
    switch (pl.logP) {
#define X(LP)                                                               \
    case LP:                                                                \
        return pl.pack_shift ? launch_fused<LP, true>(a, s) : launch_fused<LP, false>(a, s);
        QRNG_LOGP_CASES(X)
#undef X
        default:
            set_error("NTT path: unsupported P = 2^%d", pl.logP);
            return QRNG_E_UNSUPPORTED;
    }
}


// ---- NEXT-4: one block across W GPUs (distributed four-step NTT) -----------
// ("cut the sequence into several blocks" is
// the opposite move -- here one block too large for a fast single-GPU
// transform is cut across GPUs instead.)  Prime F = 1 (p = 7 * 2^26 + 1,
// P = W * N2 <= 2^26).  Index t = N2 n1 + n2 (n1 < W), k = k1 + W k2:
//   X^[k1 + W k2] = NTT_N2( u_k1 )[k2],
//   u_k1[n2] = w_P^(n2 k1) * sum_{n1<W} x[N2 n1 + n2] w_W^(n1 k1),
// so rank r computes the spectrum slice k1 = r from the (small, replicated)
// block bits with NO communication, multiplies by the matching slice of the
// seed spectrum (plan, same permuted order), runs the local inverse and
// twists:  v_r[n2] = w_P^(-n2 r) * INTT_N2(...)[n2].  Then
//   z[N2 n1 + n2] = sum_{k1<W} w_W^(-n1 k1) v_k1[n2]      (P^-1 folded into S^)
// needs every rank's v at the same n2: ONE all-to-all of N2 words per rank
// (chunk r' = columns [r' N2/W, (r'+1) N2/W)), after which rank r' finishes
// its columns for every n1 and ORs the window parities into the key.  W = 1
// is the single-GPU path for 2^23 < L <= 2^26.

// u[n2] = twist(n2) * sum_{n1 < W} bit(N2 n1 + n2) * c[n1]  (c canonical, sum < W p < 2^32)
struct ColArgs {
    const uint8_t *bits;       // MSB-first bit buffer (block or seed)
    uint64_t len;              // bits that enter the product (n or L); bits past len read as 0
    uint32_t N2, W;
    uint32_t c[8];             // w_W^(n1 r), canonical
    const uint32_t *twM;       // w_P^(n2 r) * 2^32 mod p (Montgomery form), null for r = 0
    uint32_t *u;
};
__global__ void dist_col_dft_kernel(ColArgs a) {
    constexpr uint32_t Pp = Fld<1>::P;
    for (uint32_t n2 = blockIdx.x * blockDim.x + threadIdx.x; n2 < a.N2; n2 += gridDim.x * blockDim.x) {
        uint32_t acc = 0;
        for (uint32_t n1 = 0; n1 < a.W; ++n1) {
            const uint64_t t = (uint64_t)a.N2 * n1 + n2;
            if (t < a.len && ((__ldg(a.bits + (t >> 3)) >> (7 - (t & 7))) & 1u)) acc += a.c[n1];
        }
        acc %= Pp;
        a.u[n2] = a.twM ? mont<1>(acc, __ldg(a.twM + n2)) : acc;
    }
}

// v[n2] = mont(v[n2], itwM[n2]) = v * w_P^(-n2 r) (lazy)
__global__ void dist_twist_kernel(uint32_t *v, const uint32_t *itwM, uint32_t N2) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N2; i += gridDim.x * blockDim.x)
        v[i] = mont<1>(v[i], __ldg(itwM + i));
}

// Rank r' after the all-to-all: recv[k1 * C + j] = v_k1[r' C + j] (C = N2 / W).
// z[N2 n1 + n2] = sum_k1 w_W^(-n1 k1) v_k1[n2]; window t in [len-1, len-1+m)
// -> output bit g0 + t - (len - 1).  Lanes take consecutive j (consecutive t).
struct FinishArgs {
    const uint32_t *recv;
    uint64_t len, m;           // product length (n) and outputs per block
    uint32_t N2, W, rank;
    uint32_t icM[8][8];        // w_W^(-n1 k1) * 2^32 mod p (Montgomery form)
    OutStream out;
    uint64_t g0;               // global output bit of y_0
};
__global__ void dist_finish_kernel(FinishArgs a) {
    constexpr uint32_t Pp = Fld<1>::P;
    const uint32_t C = a.N2 / a.W;
    const int lane = threadIdx.x & 31;
    for (uint32_t j0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; j0 < C; j0 += gridDim.x * blockDim.x) {
        const uint32_t j = j0 + lane;  // C % 32 == 0
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < (int)a.W ? __ldg(a.recv + (size_t)k * C + j) : 0u;
        for (uint32_t n1 = 0; n1 < a.W; ++n1) {
            uint32_t z = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < (int)a.W) z = red2<1>(z + mont<1>(v[k], a.icM[n1][k]));
            z = z >= Pp ? z - Pp : z;
            const uint64_t t = (uint64_t)a.N2 * n1 + (uint64_t)a.rank * C + j;
            const int64_t i = (int64_t)t - (int64_t)(a.len - 1);
            const bool valid = i >= 0 && i < (int64_t)a.m;
            const uint32_t bal = __ballot_sync(0xffffffffu, valid && (z & 1u));
            if (lane == 0 && bal) {
                const int64_t G = (int64_t)a.g0 + ((int64_t)((uint64_t)a.N2 * n1 + (uint64_t)a.rank * C + j0) -
                                                   (int64_t)(a.len - 1));
                const uint32_t V = __brev(bal);  // lane L (output G + L) -> logical bit 31 - L
                const int64_t W0 = G >= 0 ? (G >> 5) : -((31 - G) >> 5);
                const int o = (int)(G - W0 * 32);
                const uint32_t hi = V >> o, lo = o ? (V << (32 - o)) : 0u;
                if (hi) emit_word(a.out, (uint64_t)W0, hi, false);
                if (lo) emit_word(a.out, (uint64_t)(W0 + 1), lo, false);
            }
        }
    }
}

static unsigned grid_of(uint64_t items, unsigned block = 256) {
    const uint64_t g = (items + block - 1) / block;
    return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

// The local length-N2 transform chain on one buffer (in place): forward; then
// either the scaled spectrum (seed: SEGFWD, written to shat) or the pointwise
// product with shat and the inverse (data: SEG + inverse passes).
static qrng_status dist_local_ntt(const DistPlan &pl, uint32_t *ws, bool seed, uint32_t scaleM, cudaStream_t s) {
    const int logN2 = pl.logN2;
    FusedArgs fa{};
    fa.shat = pl.shat;
    fa.tw = pl.tw;
    fa.itw = pl.itw;
    fa.scaleM = scaleM;
    if (logN2 <= kSegLog) {
        fa.tw_shift = 0;
        switch (logN2) {
#define X(LS)                                                                                               \
    case LS:                                                                                                \
        return seed ? launch_segments<SEGFWD, 1, LS>(fa, ws, LS, 1, s, false)                                \
                    : launch_segments<SEG, 1, LS>(fa, ws, LS, 1, s, true);
            X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)
#undef X
            default: set_error("distributed NTT: unsupported N2 = 2^%d", logN2); return QRNG_E_UNSUPPORTED;
        }
    }
    int r[2];
    const int np = global_radices(logN2, r);
    PassArgs pa{};
    pa.ws = ws;
    pa.tw = pl.tw;
    pa.itw = pl.itw;
    pa.logP = (uint32_t)logN2;
    pa.S = 0;
    qrng_status st = launch_pass<PASS_FWD, 1>(r[0], pa, 1, s, !seed);
    if (st == QRNG_OK && np == 2) {
        pa.S = (uint32_t)r[0];
        st = launch_pass<PASS_FWD, 1>(r[1], pa, 1, s, !seed);
    }
    fa.tw_shift = (uint32_t)(logN2 - kSegLog);
    if (st == QRNG_OK) st = seed ? launch_segments<SEGFWD, 1>(fa, ws, logN2, 1, s, false)
                                 : launch_segments<SEG, 1>(fa, ws, logN2, 1, s, true);
    if (seed || st != QRNG_OK) return st;
    if (np == 2) {
        pa.S = (uint32_t)r[0];
        st = launch_pass<PASS_INV, 1>(r[1], pa, 1, s, true);
    }
    if (st == QRNG_OK) {
        pa.S = 0;
        st = launch_pass<PASS_INV, 1>(r[0], pa, 1, s, true);
    }
    return st;
}

static qrng_status dist_col(const DistPlan &pl, const uint8_t *bits, uint64_t len, uint32_t *u, cudaStream_t s) {
    ColArgs c{};
    c.bits = bits;
    c.len = len;
    c.N2 = pl.N2;
    c.W = pl.world;
    for (uint32_t i = 0; i < 8; ++i) c.c[i] = i < pl.world ? pl.colw[i] : 0u;
    c.twM = pl.twr;
    c.u = u;
    count_launch();
    dist_col_dft_kernel<<<grid_of(pl.N2), 256, 0, s>>>(c);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

qrng_status dist_plan_init(DistPlan &pl, uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t world,
                           uint32_t rank, cudaStream_t s) {
    if (world == 0 || world > 8 || (world & (world - 1)) || rank >= world) {
        set_error("distributed NTT: world must be 1, 2, 4 or 8 and rank < world (got %u, %u)", world, rank);
        return QRNG_E_INVALID;
    }
    const uint64_t L = n + m - 1;
    int logP = 5;
    while ((1ull << logP) < L) ++logP;
    int logW = 0;
    while ((1u << logW) < world) ++logW;
    if (logP - logW < 10) logP = 10 + logW;  // N2 / W >= 32 columns per peer (warp-wide finish)
    if (logP > kMaxLogP2) {
        set_error("distributed NTT: L = %llu exceeds 2^26", (unsigned long long)L);
        return QRNG_E_UNSUPPORTED;
    }
    constexpr uint64_t Pp = Fld<1>::P;
    pl.n = n;
    pl.m = m;
    pl.world = world;
    pl.rank = rank;
    pl.logP = logP;
    pl.logN2 = logP - logW;
    pl.N2 = 1u << pl.logN2;
    const uint64_t wP = powmod_p(3, (Pp - 1) >> logP, Pp);        // w_P
    const uint64_t wN2 = powmod_p(wP, world, Pp);                  // w_N2 = w_P^W
    const uint64_t wW = powmod_p(wP, 1ull << pl.logN2, Pp);        // w_W = w_P^N2
    const uint64_t iwW = powmod_p(wW, Pp - 2, Pp);
    const uint64_t R32 = (1ull << 32) % Pp;
    for (uint32_t i = 0; i < 8; ++i) {
        pl.colw[i] = (uint32_t)powmod_p(wW, (uint64_t)i * rank, Pp);
        for (uint32_t k = 0; k < 8; ++k)
            pl.icolM[i][k] = (uint32_t)(powmod_p(iwW, (uint64_t)i * k % world, Pp) * R32 % Pp);
    }
    const size_t bytes = (size_t)pl.N2 * 4;
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.shat, bytes, s));
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.tw, bytes, s));
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.itw, bytes, s));
    count_launch();
    twiddle_table_kernel<1><<<(unsigned)(((pl.N2 + kTwChain - 1) / kTwChain + 127) / 128), 128, 0, s>>>(
        pl.tw, pl.itw, pl.N2, (uint32_t)wN2, (uint32_t)powmod_p(wN2, Pp - 2, Pp));
    QRNG_CUDA_TRY(cudaGetLastError());
    if (rank != 0) {  // twist tables w_P^(+-n2 r), Montgomery form
        QRNG_CUDA_TRY(cudaMallocAsync(&pl.twr, bytes, s));
        QRNG_CUDA_TRY(cudaMallocAsync(&pl.itwr, bytes, s));
        const uint64_t wr = powmod_p(wP, rank, Pp);
        count_launch();
        twiddle_table_kernel<1><<<(unsigned)(((pl.N2 + kTwChain - 1) / kTwChain + 127) / 128), 128, 0, s>>>(
            pl.twr, pl.itwr, pl.N2, (uint32_t)wr, (uint32_t)powmod_p(wr, Pp - 2, Pp));
        QRNG_CUDA_TRY(cudaGetLastError());
    }
    // seed spectrum slice k1 = rank, scaled by P^-1 (and 2^32: Montgomery form
    // for the pointwise product): scaleM = P^-1 * 2^64 mod p
    uint32_t *u = nullptr;
    QRNG_CUDA_TRY(cudaMallocAsync(&u, bytes, s));
    qrng_status st = dist_col(pl, d_seed, L, u, s);
    const uint64_t pinvP = powmod_p((1ull << logP) % Pp, Pp - 2, Pp);
    const uint32_t scaleM = (uint32_t)((unsigned __int128)pinvP * (((unsigned __int128)1 << 64) % Pp) % Pp);
    if (st == QRNG_OK) st = dist_local_ntt(pl, u, true, scaleM, s);
    cudaFreeAsync(u, s);
    return st;
}

void dist_plan_free(DistPlan &pl, cudaStream_t s, bool async) {
    for (uint32_t *p : {pl.shat, pl.tw, pl.itw, pl.twr, pl.itwr})
        if (p) { if (async) cudaFreeAsync(p, s); else cudaFree(p); }
    pl = DistPlan{};
}

qrng_status dist_local(const DistPlan &pl, const uint8_t *d_block_bits, uint32_t *d_buf, cudaStream_t s) {
    qrng_status st = dist_col(pl, d_block_bits, pl.n, d_buf, s);
    if (st == QRNG_OK) st = dist_local_ntt(pl, d_buf, false, 0, s);
    if (st == QRNG_OK && pl.itwr) {
        count_launch();
        dist_twist_kernel<<<grid_of(pl.N2), 256, 0, s>>>(d_buf, pl.itwr, pl.N2);
        QRNG_CUDA_TRY(cudaGetLastError());
    }
    return st;
}

qrng_status dist_finish(const DistPlan &pl, const uint32_t *d_recv, const OutStream &out, uint64_t g0,
                        cudaStream_t s) {
    FinishArgs f{};
    f.recv = d_recv;
    f.len = pl.n;
    f.m = pl.m;
    f.N2 = pl.N2;
    f.W = pl.world;
    f.rank = pl.rank;
    memcpy(f.icM, pl.icolM, sizeof f.icM);
    f.out = out;
    f.g0 = g0;
    KernelTimer t(s, true);
    dist_finish_kernel<<<grid_of(pl.N2 / pl.world), 256, 0, s>>>(f);
    t.stop();
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

}  // namespace ntt
}  // namespace qrng
