// hist.cu -- exact 256-bin histogram of 8-bit ADC samples (HBM-bound).
//
// Feeds the empirical distribution P'(x) of PAPER.md:141-155 (Sec. II.C) and
// the max-probability H_min of PAPER.md:59.  B200 design: grid-stride over
// 16-byte vectors (one LDG.128 per thread per iteration), per-warp private
// sub-histograms in shared memory (Gaussian ADC data concentrates on a few
// bins, so a single CTA histogram would serialise on the hot bins), then one
// 64-bit global atomic per bin per CTA.  Counts are exact (uint32 in smem per
// CTA chunk, uint64 in HBM).  d_samples may have any alignment (head bytes up
// to the first 16-byte boundary are counted with scalar loads).
#include "qrng_internal.cuh"

namespace qrng {

namespace {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
#ifndef QRNG_HIST_COPIES
#define QRNG_HIST_COPIES 1  // sub-histograms per warp (lane % copies picks one): fewer same-bin atomic collisions
#endif
constexpr int kCopies = QRNG_HIST_COPIES;
constexpr int kSub = kWarps * kCopies;

__device__ __forceinline__ void add4(uint32_t *h, uint32_t w) {
    atomicAdd(&h[w & 0xFF], 1u);
    atomicAdd(&h[(w >> 8) & 0xFF], 1u);
    atomicAdd(&h[(w >> 16) & 0xFF], 1u);
    atomicAdd(&h[w >> 24], 1u);
}

__global__ void __launch_bounds__(kThreads) hist256_kernel(const uint8_t *__restrict__ x, uint64_t n,
                                                           unsigned long long *__restrict__ counts) {
    extern __shared__ uint32_t hs[];  // [kSub][256]
    for (int i = threadIdx.x; i < kSub * 256; i += kThreads) hs[i] = 0;
    __syncthreads();
    uint32_t *mine = hs + ((threadIdx.x >> 5) * kCopies + (threadIdx.x & (kCopies - 1))) * 256;
    const uint64_t tid = blockIdx.x * (uint64_t)kThreads + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * kThreads;
    // any alignment: the bytes before the first 16-byte boundary are counted
    // one by one (a shard slice samples[lo:hi] starts anywhere), then vectors
    uint64_t head = (16u - ((uintptr_t)x & 15u)) & 15u;
    if (head > n) head = n;
    if (tid < head) atomicAdd(&mine[x[tid]], 1u);
    x += head;
    n -= head;
    const uint64_t nvec = n / 16;
    const uint4 *v = reinterpret_cast<const uint4 *>(x);
    for (uint64_t i = tid; i < nvec; i += nthr) {
        uint4 q = __ldcs(v + i);  // streamed once
        add4(mine, q.x);
        add4(mine, q.y);
        add4(mine, q.z);
        add4(mine, q.w);
    }
    for (uint64_t i = nvec * 16 + tid; i < n; i += nthr) atomicAdd(&mine[x[i]], 1u);
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += kThreads) {
        uint32_t s = 0;
        for (int w = 0; w < kSub; ++w) s += hs[w * 256 + b];
        if (s) atomicAdd(counts + b, (unsigned long long)s);
    }
}
}  // namespace

qrng_status hist256_launch(const uint8_t *d_samples, uint64_t n, unsigned long long *d_counts,
                           cudaStream_t s) {
    int dev = 0, sms = 148;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // <= 2^31 samples per CTA keeps every per-CTA smem count below 2^32
    uint64_t want = (n / 16 + kThreads - 1) / kThreads;
    uint64_t grid = want < (uint64_t)sms * 4 ? want : (uint64_t)sms * 4;
    uint64_t min_grid = n / (1ull << 31) + 1;
    if (grid < min_grid) grid = min_grid;
    if (grid == 0) grid = 1;
    count_launch();
    const size_t smem = (size_t)kSub * 256 * 4;
    if (smem > 48 * 1024) {
        const qrng_status st = allow_max_smem(reinterpret_cast<const void *>(hist256_kernel));
        if (st != QRNG_OK) return st;
    }
    hist256_kernel<<<(unsigned)grid, kThreads, smem, s>>>(d_samples, n, d_counts);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

}  // namespace qrng
