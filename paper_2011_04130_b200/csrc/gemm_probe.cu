// gemm_probe.cu -- test and profiling instruments around the tcgen05 path
// (not on the extraction path): the live MMA-rate microbenchmark the bench's
// roofline divides by (qrng_debug_mma_rate), the int8 and E2M1 layout /
// exactness probes the GPU tests use (qrng_debug_umma_probe,
// qrng_debug_mxf4_probe).  Product kernels live in gemm_tc.cu.
#include "qrng_internal.cuh"
#include "tc_ptx.cuh"

namespace qrng {
namespace gemm {
using namespace tc;

namespace {
// kind::i8 (probes / microbenchmark only): S32 accumulate, S8 x S8 (or U8 x U8), K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool is_signed = true) {
    return (2u << 4) | ((is_signed ? 1u : 0u) << 7) | ((is_signed ? 1u : 0u) << 10) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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
}  // namespace

// ---- MMA-rate microbenchmark (profiling only) ---------------------------------------
// One elected thread per CTA issues `iters` back-to-back int8 MMAs on fixed
// operands (no data movement): form 0 = cta_group::1, A in TMEM, M128 N=n;
// form 1 = cta_group::1, A in SMEM, M128 N=n; form 2 (cta_group::2) was removed
// with the 2-SM kernel.  Time it with CUDA events; MACs = CTAs x iters x
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
        *reinterpret_cast<volatile uint32_t *>(smem + 64 * 1024 + 32) = 0u;  // form 5 writer stop flag
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
    __syncthreads();
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
                            mma_mxf4_ss(tmem + 224, ad, desc_kmajor(cb + ((it & 3) * 16 + kk * 8 + n0 / 8) * 128, 512, 128),
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
    if (FORM == 5 && warp == 1 && commit_every > 0) {
        // shared-memory contention (form 5 + 16k): this warp stores k bytes per
        // clock on average (one 512-byte st.shared.v4 per 512/k clocks) into a
        // region the MMAs do not read, until the MMAs have completed
        const long long period = 512 / commit_every;
        volatile uint32_t *stop = reinterpret_cast<volatile uint32_t *>(smem + 64 * 1024 + 32);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + 65 * 1024);
        const int lane = threadIdx.x & 31;
        uint32_t i = 0;
        long long t = clock64();
        while (!*stop) {
            dst[(i & 63) * 32 + lane] = make_uint4(i, i + 1, i + 2, i + 3);
            ++i;
            t += period;
            while (clock64() < t) {}
        }
    }
    if (FORM == 2 || rank == 0) {
        if (threadIdx.x == 0) {
            mbar_wait(&bar, 0);
            *reinterpret_cast<volatile uint32_t *>(smem + 64 * 1024 + 32) = 1u;
        }
    }
    tc_fence_before();
    __syncthreads();
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
    const size_t smem = 65 * 1024 + 32 * 1024;  // operands, barriers, form-5 writer region
    const unsigned grid = (unsigned)sms;
    count_launch();
    switch (form) {
        case 0: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<0>)); mma_rate_kernel<0><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 1: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<1>)); mma_rate_kernel<1><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 3: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<3>)); mma_rate_kernel<3><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 4: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<4>)); mma_rate_kernel<4><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
        case 5: allow_max_smem(reinterpret_cast<const void *>(mma_rate_kernel<5>)); mma_rate_kernel<5><<<grid, 128, smem, s>>>(iters, n, nullptr, commit_every); break;
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
    const int warp = threadIdx.x >> 5, tid = threadIdx.x;
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

qrng_status trace(uint64_t *h_out, int reset) { return timeline(h_out, reset); }

}  // namespace gemm
}  // namespace qrng
