// api.cu -- the C ABI of libqrng.so (include/qrng.h): argument validation,
// plans and the block scheduler that picks the extraction path, and the
// host-side finalisation of the min-entropy chain.
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <set>
#include <algorithm>
#include <vector>
#include "qrng_internal.cuh"

namespace qrng {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

// ---- instrumentation (qrng_debug_*) ----
static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_timing{0};
static std::mutex g_tmu;
struct TimedLaunch {
    cudaEvent_t a, b;
    int channel;
};
static std::vector<TimedLaunch> g_events;

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static thread_local SideStream g_side;

qrng_status side_stream(cudaStream_t *s2, cudaEvent_t *fork, cudaEvent_t *join) {
    int dev = 0;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    if (g_side.dev != dev) {
        if (g_side.s) {
            cudaStreamDestroy(g_side.s);
            cudaEventDestroy(g_side.fork);
            cudaEventDestroy(g_side.join);
        }
        g_side = SideStream{};
        QRNG_CUDA_TRY(cudaStreamCreateWithFlags(&g_side.s, cudaStreamNonBlocking));
        QRNG_CUDA_TRY(cudaEventCreateWithFlags(&g_side.fork, cudaEventDisableTiming));
        QRNG_CUDA_TRY(cudaEventCreateWithFlags(&g_side.join, cudaEventDisableTiming));
        g_side.dev = dev;
    }
    *s2 = g_side.s;
    *fork = g_side.fork;
    *join = g_side.join;
    return QRNG_OK;
}

qrng_status allow_max_smem(const void *func) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({func, dev})) return QRNG_OK;
    QRNG_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    done.insert({func, dev});
    return QRNG_OK;
}

// Timing events are recycled (bench mode records two per timed launch; creating
// them on every launch would put host work inside the timed region).
static std::vector<cudaEvent_t> g_event_pool;
static cudaEvent_t pooled_event() {
    {
        std::lock_guard<std::mutex> lk(g_tmu);
        if (!g_event_pool.empty()) {
            cudaEvent_t e = g_event_pool.back();
            g_event_pool.pop_back();
            return e;
        }
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}

KernelTimer::KernelTimer(cudaStream_t st, bool timed, int ch) : s(st), channel(ch) {
    count_launch();
    // level 1: the main extraction kernel(s) (channel 0) only; level 2: also the
    // auxiliary kernels (each timed launch adds two event records to the stream)
    const int lvl = g_timing.load();
    if (!timed || lvl < 1 || (ch != 0 && lvl < 2)) return;
    a = pooled_event();
    b = pooled_event();
    if (!a || !b) { a = b = nullptr; return; }
    cudaEventRecord(a, s);
}
void KernelTimer::stop() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_tmu);
    g_events.push_back(TimedLaunch{a, b, channel});
}

// Measured GEMM/NTT crossover in n; GEMM for n <= this.
static uint64_t g_gemm_max_n = 1ull << 18;  // profiles/sweep_r1u.jsonl (E2M1 operands): Karatsuba GEMM 68.5 vs NTT 48.5 Gbit/s at 2^18, 40.6 vs 47.5 at 2^19
static std::atomic<int> g_debug_path{QRNG_PATH_AUTO};
static std::atomic<int> g_last_path{-1};  // product path of the most recent extraction (bench labels)
// Small batches on the CUDA cores (bits.cu) instead of the dense tcgen05 kernel
// when an AUTO plan's batch has at most bits_max_macs(n) bit-MACs (n m n_blocks).
// Measured (tools/bits_crossover.py, one-shot device time, L2 flushed): the
// CUDA-core kernel takes ~8 us + 8.4 ns per 1e6 bit-MACs whatever n; the
// tcgen05 kernel's small-batch floor grows with n (13.3 / 15.4 / 17.4 us at
// n = 1024 / 2048 / 4096), so the crossover is 6e8 / 8.8e8 / 1.1e9 bit-MACs:
// 6e8 + 2.7e8 log2(n / 1024), at least 6e8.  QRNG_BITS_MAX_MACS overrides.
static double bits_max_macs(uint64_t n) {
    static const double v = [] {
        const char *e = getenv("QRNG_BITS_MAX_MACS");
        return (e && *e) ? atof(e) : -1.0;
    }();
    if (v >= 0) return v;
    return n <= 1024 ? 6.0e8 : 6.0e8 + 2.7e8 * std::log2((double)n / 1024.0);
}
// Karatsuba depth over the GEMM path: -1 = the planner's cost model, 0 = plain
// GEMM kernel, d > 0 = split whenever allowed down to depth d (tests).
static std::atomic<int> g_kara_depth{-1};

// One-time device check: sm_100 required (no CPU fallback), stream-ordered
// pool kept warm so per-call workspace allocation is cheap.
static qrng_status device_ready() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        set_error("no CUDA device: %s", cudaGetErrorString(e));
        return QRNG_E_CUDA;
    }
    static std::mutex mu;
    static bool ready[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 64 && ready[dev]) return QRNG_OK;
    int major = 0, minor = 0;
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    QRNG_CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    if (major != 10 || minor != 0) {
        set_error("libqrng is built for sm_100a (B200); device %d is sm_%d%d", dev, major, minor);
        return QRNG_E_CUDA;
    }
    cudaMemPool_t pool;
    QRNG_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thresh = UINT64_MAX;
    QRNG_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    if (dev < 64) ready[dev] = true;
    return QRNG_OK;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static bool overlap(const void *a, uint64_t na, const void *b, uint64_t nb) {
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

static qrng_status check_nm(uint64_t n, uint64_t m) {
    if (n == 0 || m == 0 || m >= n) {
        set_error("need 0 < m < n (got n=%llu, m=%llu)", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_INVALID;
    }
    if (n % 32 != 0) {
        set_error("n must be a multiple of 32 (got %llu)", (unsigned long long)n);
        return QRNG_E_UNSUPPORTED;
    }
    if (n + m - 1 > (1ull << ntt::kMaxLogP2)) {
        set_error("seed length n+m-1 = %llu exceeds 2^26", (unsigned long long)(n + m - 1));
        return QRNG_E_UNSUPPORTED;
    }
    return QRNG_OK;
}

}  // namespace qrng

using namespace qrng;

struct qrng_plan {
    uint64_t n = 0, m = 0;
    int path = QRNG_PATH_NTT;
    bool auto_path = false;  // chosen by the scheduler (not forced): small batches may run on the CUDA cores
    bool kara_on = false;  // GEMM path through the Karatsuba decomposition
    bool modified = false;  // modified Toeplitz [T | I_m] (n-bit seed)
    const uint8_t *direct_seed = nullptr;  // one-shot dense GEMM: the caller's seed, read by the kernel itself
    ntt::Plan ntt;
    gemm::Plan gemm;
    kara::Plan kara;
};

static void plan_release(qrng_plan *p, cudaStream_t s, bool async) {
    if (!p) return;
    auto fr = [&](void *ptr) {
        if (!ptr) return;
        if (async) cudaFreeAsync(ptr, s);
        else cudaFree(ptr);
    };
    fr(p->ntt.shat); fr(p->ntt.tw); fr(p->ntt.itw); fr(p->ntt.l1tw); fr(p->ntt.work);
    for (int f = 0; f < 3; ++f) { fr(p->ntt.shat3[f]); fr(p->ntt.tw3[f]); fr(p->ntt.itw3[f]); fr(p->ntt.l1tw3[f]); }
    fr(p->gemm.seed_words);
    fr(p->kara.seeds);
    delete p;
}

extern "C" {

const char *qrng_last_error(void) { return g_err; }
const char *qrng_version(void) { return "qrng-b200 0.1 sm_100a"; }
void qrng_debug_set_path(int path) { g_debug_path.store(path); }
uint64_t qrng_debug_launch_count(void) { return g_launches.load(); }
qrng_status qrng_debug_butterfly_rate(int iters, uint64_t *butterflies, cudaStream_t stream) {
    if (!butterflies || iters <= 0) { set_error("bad arguments"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return ntt::butterfly_rate(iters, butterflies, stream, false);
}
qrng_status qrng_debug_pass_rate(int iters, uint64_t *butterflies, cudaStream_t stream) {
    if (!butterflies || iters <= 0) { set_error("bad arguments"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return ntt::butterfly_rate(iters, butterflies, stream, true);
}
qrng_status qrng_debug_umma_probe(const uint8_t *d_A, const uint8_t *d_h, int32_t *d_D, int N, int K,
                                  cudaStream_t stream) {
    if (!d_A || !d_h || !d_D) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return gemm::probe(d_A, d_h, d_D, N, K, stream);
}
int qrng_debug_gemm_operand_bits(void) { return gemm::operand_bits(); }
qrng_status qrng_debug_mxf4_probe(const uint8_t *d_A, const uint8_t *d_h, float *d_D, int N, int K, int hi_first,
                                  cudaStream_t stream) {
    if (!d_A || !d_h || !d_D) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return gemm::mxf4_probe(d_A, d_h, d_D, N, K, hi_first, stream);
}
qrng_status qrng_debug_mma_rate(int form, int iters, int n, uint64_t *macs, cudaStream_t stream) {
    const int n0 = n & 511, n1 = n >> 9;  // form 3: two N tiles (n1 = 0: same as n0)
    if (!macs || iters <= 0 || n0 < 16 || n0 > 256 || n0 % 16 || n1 > 224 || n1 % 16 ||
        ((form % 16) != 3 && (form % 16) != 5 && n1) || ((form % 16) == 5 && n0 > 224)) {
        set_error("bad arguments");
        return QRNG_E_INVALID;
    }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return gemm::mma_rate(form, iters, n, macs, stream);
}
qrng_status qrng_debug_gemm_trace(uint64_t *h_counters32, int reset) {
    if (!h_counters32) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    return gemm::trace(h_counters32, reset);
}
void qrng_debug_kernel_timing(int enable) { g_timing.store(enable < 0 ? 0 : (enable > 2 ? 2 : enable)); }
double qrng_debug_kernel_time_split(double *aux_ms, uint64_t *launches, uint64_t *aux_launches) {
    std::lock_guard<std::mutex> lk(g_tmu);
    double tot[2] = {0, 0};
    uint64_t cnt[2] = {0, 0};
    for (auto &e : g_events) {
        float ms = 0;
        if (cudaEventSynchronize(e.b) == cudaSuccess && cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess)
            tot[e.channel ? 1 : 0] += ms;
        ++cnt[e.channel ? 1 : 0];
        g_event_pool.push_back(e.a);
        g_event_pool.push_back(e.b);
    }
    g_events.clear();
    if (aux_ms) *aux_ms = tot[1];
    if (launches) *launches = cnt[0];
    if (aux_launches) *aux_launches = cnt[1];
    return tot[0];
}
double qrng_debug_kernel_time_ms(uint64_t *launches) { return qrng_debug_kernel_time_split(nullptr, launches, nullptr); }

int qrng_plan_path(const qrng_plan *plan) { return plan ? plan->path : -1; }
int qrng_debug_last_path(void) { return g_last_path.load(); }

void qrng_debug_set_karatsuba(int max_depth) { g_kara_depth.store(max_depth < -1 ? -1 : max_depth); }

qrng_status qrng_plan_info(const qrng_plan *plan, qrng_plan_info_t *info) {
    if (!plan || !info) { set_error("NULL argument"); return QRNG_E_INVALID; }
    memset(info, 0, sizeof *info);
    info->path = plan->path;
    if (plan->path == QRNG_PATH_NTT) {
        info->log2_transform = plan->ntt.logP;
        info->blocks_per_transform = plan->ntt.crt ? plan->ntt.crt : plan->ntt.pack_shift ? 2 : 1;
        info->primes = plan->ntt.crt ? 3 : 1;
    } else if (plan->kara_on) {
        int d = 0, l = 0;
        uint64_t macs = 0;
        kara::describe(plan->kara, &d, &l, &macs, &info->x_words, &info->y_words);
        info->karatsuba_depth = d;
        info->leaves = l;
        info->macs_per_block = macs;
    } else {
        info->leaves = 1;
        info->macs_per_block = plan->modified ? (plan->n - plan->m + 127) / 128 * 128 * plan->m : plan->n * plan->m;
    }
    return QRNG_OK;
}

// The block scheduler's path choice (row a2): the tensor-core path for n a
// multiple of 128 up to the measured crossover (Karatsuba tree if the planner
// decomposes (n, m)), the NTT path above it and for every shape the dense
// kernel cannot take.
static qrng_status resolve_path(uint64_t n, uint64_t m, int *path, bool *kara_on) {
    int want = g_debug_path.load();
    const bool automatic = want == QRNG_PATH_AUTO;
    *kara_on = false;
    if (want == QRNG_PATH_BITS) {
        if (!bits::supported(n, m)) {
            set_error("CUDA-core path does not support n=%llu, m=%llu", (unsigned long long)n, (unsigned long long)m);
            return QRNG_E_UNSUPPORTED;
        }
        *path = want;
        return QRNG_OK;
    }
    if (automatic) want = (n % 128 == 0 && n <= g_gemm_max_n) ? QRNG_PATH_GEMM : QRNG_PATH_NTT;
    if (want == QRNG_PATH_GEMM) *kara_on = kara::choose(n, m, g_kara_depth.load());
    // AUTO: a shape the planner leaves undecomposed (small m at large n) that the
    // dense kernel cannot take runs on the NTT path, which accepts every valid (n, m)
    if (automatic && want == QRNG_PATH_GEMM && !*kara_on && !gemm::supported(n, m)) want = QRNG_PATH_NTT;
    if (want == QRNG_PATH_GEMM && !*kara_on && !gemm::supported(n, m)) {
        set_error("GEMM path does not support n=%llu, m=%llu", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    *path = want;
    return QRNG_OK;
}

static qrng_status plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t stream,
                               qrng_plan **plan, bool oneshot);

qrng_status qrng_plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t stream,
                             qrng_plan **plan) {
    return plan_create(n, m, d_seed, stream, plan, false);
}

// oneshot: the plan is extracted exactly once, on `stream`, by the caller
// (qrng_toeplitz_extract_async): work that can ride on the extraction's own
// launches (the Karatsuba leaf seeds) is deferred to them.
static qrng_status plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t stream,
                               qrng_plan **plan, bool oneshot) {
    if (!plan) { set_error("plan is NULL"); return QRNG_E_INVALID; }
    *plan = nullptr;
    qrng_status st = check_nm(n, m);
    if (st != QRNG_OK) return st;
    if (!d_seed || !aligned16(d_seed)) { set_error("d_seed is NULL or not 16-byte aligned"); return QRNG_E_INVALID; }
    if ((st = device_ready()) != QRNG_OK) return st;
    int want = 0;
    bool kara_on = false;
    if ((st = resolve_path(n, m, &want, &kara_on)) != QRNG_OK) return st;
    qrng_plan *p = new (std::nothrow) qrng_plan;
    if (!p) { set_error("host allocation failed"); return QRNG_E_NOMEM; }
    p->n = n;
    p->m = m;
    p->kara_on = kara_on;
    p->path = want;
    p->auto_path = g_debug_path.load() == QRNG_PATH_AUTO;
    const int kd = g_kara_depth.load();
    st = (want == QRNG_PATH_NTT)    ? ntt::plan_init(p->ntt, n, m, d_seed, 0, false, stream)
         : (want == QRNG_PATH_BITS) ? bits::plan_init(p->gemm, n, m, d_seed, stream)
         : p->kara_on            ? kara::plan_init(p->kara, n, m, kd, d_seed, stream, oneshot)
                                 : gemm::plan_init(p->gemm, n, m, d_seed, stream);
    if (st != QRNG_OK) { plan_release(p, stream, true); return st; }
    *plan = p;
    return QRNG_OK;
}

// Modified Toeplitz [T_{m x (n-m)} | I_m]: the product of the
// first n-m raw bits of each block with T (seed bits a_2..a_n, C1 form with
// n' = n-m) XOR the block's last m raw bits; always the NTT path.
qrng_status qrng_plan_create_modified(uint64_t n, uint64_t m, const uint8_t *d_seed, cudaStream_t stream,
                                      qrng_plan **plan) {
    if (!plan) { set_error("plan is NULL"); return QRNG_E_INVALID; }
    *plan = nullptr;
    if (n == 0 || m == 0 || m >= n) {
        set_error("need 0 < m < n (got n=%llu, m=%llu)", (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_INVALID;
    }
    if (n % 32 != 0) { set_error("n must be a multiple of 32"); return QRNG_E_UNSUPPORTED; }
    if (n - 1 > (1ull << ntt::kMaxLogP)) { set_error("n - 1 exceeds 2^23"); return QRNG_E_UNSUPPORTED; }
    if (!d_seed || !aligned16(d_seed)) { set_error("d_seed is NULL or not 16-byte aligned"); return QRNG_E_INVALID; }
    int want = g_debug_path.load();
    if (want == QRNG_PATH_BITS) {
        set_error("modified Toeplitz: no CUDA-core path (QRNG_PATH_BITS)");
        return QRNG_E_UNSUPPORTED;
    }
    const uint64_t kprod = (n - m + 127) / 128 * 128;  // GEMM product length (n - m rounded up to 128)
    if (want == QRNG_PATH_AUTO) want = (gemm::modified_supported(n, m) && kprod <= g_gemm_max_n) ? QRNG_PATH_GEMM : QRNG_PATH_NTT;
    if (want == QRNG_PATH_GEMM && !gemm::modified_supported(n, m)) {
        set_error("GEMM path: the modified Toeplitz needs n %% 32 == 0 and n - m <= 2^16 (n=%llu, m=%llu)",
                  (unsigned long long)n, (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    qrng_plan *p = new (std::nothrow) qrng_plan;
    if (!p) { set_error("host allocation failed"); return QRNG_E_NOMEM; }
    p->n = n;
    p->m = m;
    p->path = want;
    p->modified = true;
    st = want == QRNG_PATH_GEMM ? gemm::plan_init_modified(p->gemm, n, m, d_seed, stream)
                                : ntt::plan_init(p->ntt, n - m, m, d_seed, 1, true, stream);
    if (st != QRNG_OK) { plan_release(p, stream, true); return st; }
    *plan = p;
    return QRNG_OK;
}

qrng_status qrng_modified_toeplitz_extract_async(const uint8_t *d_raw_bits, uint64_t n_blocks, uint64_t n,
                                                 uint64_t m, const uint8_t *d_seed, uint8_t *d_out,
                                                 cudaStream_t stream) {
    if (!d_raw_bits || !d_seed || !d_out) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    if (n_blocks == 0) { set_error("n_blocks must be > 0"); return QRNG_E_INVALID; }
    if (n != 0 && m != 0 && n_blocks <= UINT64_MAX / m &&
        overlap(d_seed, (n + 7) / 8, d_out, (n_blocks * m + 7) / 8)) {
        set_error("d_out overlaps d_seed");
        return QRNG_E_INVALID;
    }
    qrng_plan *p = nullptr;
    qrng_status st = qrng_plan_create_modified(n, m, d_seed, stream, &p);
    if (st != QRNG_OK) return st;
    st = qrng_plan_extract(p, d_raw_bits, n_blocks, d_out, stream);
    plan_release(p, stream, true);
    return st;
}

void qrng_plan_destroy(qrng_plan *plan) { plan_release(plan, 0, false); }

qrng_status qrng_plan_extract(const qrng_plan *plan, const uint8_t *d_raw_bits, uint64_t n_blocks,
                              uint8_t *d_out, cudaStream_t stream) {
    if (!plan) { set_error("plan is NULL"); return QRNG_E_INVALID; }
    const uint64_t n = plan->n, m = plan->m;
    if (n_blocks == 0) { set_error("n_blocks must be > 0"); return QRNG_E_INVALID; }
    if (!d_raw_bits || !d_out) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    if (!aligned16(d_raw_bits)) { set_error("d_raw_bits must be 16-byte aligned"); return QRNG_E_INVALID; }
    if (((uintptr_t)d_out & 3u) != 0) { set_error("d_out must be 4-byte aligned"); return QRNG_E_INVALID; }
    if (n_blocks > (UINT64_MAX / n)) { set_error("n_blocks * n overflows"); return QRNG_E_INVALID; }
    const uint64_t raw_bytes = n_blocks * n / 8, out_bits = n_blocks * m, out_bytes = (out_bits + 7) / 8;
    if (overlap(d_raw_bits, raw_bytes, d_out, out_bytes)) { set_error("d_out overlaps d_raw_bits"); return QRNG_E_INVALID; }
    OutStream o;
    o.words = reinterpret_cast<uint32_t *>(d_out);
    o.total_bits = out_bits;
    o.full_words = out_bytes / 4;
    o.tail = nullptr;
    // A final partial 32-bit word (out_bytes % 4 != 0) is assembled in a 4-byte
    // scratch owned by this call (so concurrent calls on one plan never share
    // it) and its valid bytes copied back: nothing past out_bytes is touched.
    if (out_bytes % 4) {
        cudaError_t e = cudaMallocAsync(&o.tail, 4, stream);
        if (e != cudaSuccess) { set_error("cudaMallocAsync: %s", cudaGetErrorString(e)); return QRNG_E_NOMEM; }
        QRNG_CUDA_TRY(cudaMemsetAsync(o.tail, 0, 4, stream));
    }
    // small batches of a dense AUTO plan run on the CUDA cores (latency-bound on
    // the tensor cores; bits.cu)
    const bool use_bits = plan->path == QRNG_PATH_BITS ||
                          (plan->auto_path && plan->path == QRNG_PATH_GEMM && !plan->kara_on && !plan->modified &&
                           bits::supported(n, m) && (double)n * (double)m * (double)n_blocks <= bits_max_macs(n));
    g_last_path.store(use_bits ? QRNG_PATH_BITS : plan->path);
    // the Karatsuba pack and CUDA-core kernels write every output word once; the
    // other epilogues OR the words they share with a neighbouring tile / CTA
    if (!use_bits && !(plan->path == QRNG_PATH_GEMM && plan->kara_on))
        QRNG_CUDA_TRY(cudaMemsetAsync(d_out, 0, out_bytes, stream));
    qrng_status st = use_bits ? bits::extract(plan->direct_seed ? nullptr : plan->gemm.seed_words, plan->direct_seed,
                                              d_raw_bits, n_blocks, n, m, o, stream)
                     : (plan->path == QRNG_PATH_NTT) ? ntt::extract(plan->ntt, d_raw_bits, n_blocks, n, m, o, stream)
                     : plan->kara_on ? kara::extract(plan->kara, d_raw_bits, n_blocks, n, m, o, stream)
                     : plan->modified ? gemm::extract_modified(plan->gemm, d_raw_bits, n_blocks, n, m, o, stream)
                     : plan->direct_seed ? gemm::extract_direct(plan->direct_seed, d_raw_bits, n_blocks, n, m, o, stream)
                                      : gemm::extract(plan->gemm, d_raw_bits, n_blocks, n, m, o, stream);
    if (st == QRNG_OK && o.tail) {
        cudaError_t e = cudaMemcpyAsync(d_out + (out_bytes / 4) * 4, o.tail, out_bytes % 4,
                                        cudaMemcpyDeviceToDevice, stream);
        if (e != cudaSuccess) { set_error("tail copy: %s", cudaGetErrorString(e)); st = QRNG_E_CUDA; }
    }
    if (o.tail) cudaFreeAsync(o.tail, stream);
    return st;
}

qrng_status qrng_toeplitz_extract_async(const uint8_t *d_raw_bits, uint64_t n_blocks, uint64_t n, uint64_t m,
                                        const uint8_t *d_seed, uint8_t *d_out, cudaStream_t stream) {
    qrng_status st = check_nm(n, m);
    if (st != QRNG_OK) return st;
    if (!d_raw_bits || !d_seed || !d_out) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    if (n_blocks == 0) { set_error("n_blocks must be > 0"); return QRNG_E_INVALID; }
    if (d_out && d_seed && n_blocks <= UINT64_MAX / m &&
        overlap(d_seed, (n + m - 1 + 7) / 8, d_out, (n_blocks * m + 7) / 8)) {
        set_error("d_out overlaps d_seed");
        return QRNG_E_INVALID;
    }
    if (!aligned16(d_seed)) { set_error("d_seed must be 16-byte aligned"); return QRNG_E_INVALID; }
    if ((st = device_ready()) != QRNG_OK) return st;
    int path = 0;
    bool kara_on = false;
    if ((st = resolve_path(n, m, &path, &kara_on)) != QRNG_OK) return st;
    if ((path == QRNG_PATH_GEMM && !kara_on) || path == QRNG_PATH_BITS) {
        // dense product (tensor cores, or the CUDA cores for a small batch): no
        // plan buffers or seed kernel; the kernel forms the seed words from d_seed
        // in its prologue (small batches are latency-bound: this removes an
        // allocation, a launch and a free)
        qrng_plan direct;
        direct.n = n;
        direct.m = m;
        direct.path = path;
        direct.auto_path = g_debug_path.load() == QRNG_PATH_AUTO;
        direct.direct_seed = d_seed;
        return qrng_plan_extract(&direct, d_raw_bits, n_blocks, d_out, stream);
    }
    qrng_plan *p = nullptr;
    if ((st = plan_create(n, m, d_seed, stream, &p, true)) != QRNG_OK) return st;
    st = qrng_plan_extract(p, d_raw_bits, n_blocks, d_out, stream);
    plan_release(p, stream, true);
    return st;
}

qrng_status qrng_toeplitz_extract(const uint8_t *d_raw_bits, uint64_t n_blocks, uint64_t n, uint64_t m,
                                  const uint8_t *d_seed, uint8_t *d_out) {
    qrng_status st = qrng_toeplitz_extract_async(d_raw_bits, n_blocks, n, m, d_seed, d_out, 0);
    if (st != QRNG_OK) return st;
    QRNG_CUDA_TRY(cudaStreamSynchronize(0));
    return QRNG_OK;
}

// Copy streams of the calling thread (host-buffer path): H2D and D2H run on
// their own streams so both PCIe directions overlap the kernels.
struct CopyStreams {
    int dev = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr, comp2 = nullptr;
};
static thread_local CopyStreams g_cs;

static qrng_status copy_streams(int dev, cudaStream_t *h2d, cudaStream_t *d2h, cudaStream_t *comp2) {
    if (g_cs.dev != dev) {
        if (g_cs.h2d) { cudaStreamDestroy(g_cs.h2d); cudaStreamDestroy(g_cs.d2h); cudaStreamDestroy(g_cs.comp2); }
        g_cs = CopyStreams{};
        QRNG_CUDA_TRY(cudaStreamCreateWithFlags(&g_cs.h2d, cudaStreamNonBlocking));
        QRNG_CUDA_TRY(cudaStreamCreateWithFlags(&g_cs.d2h, cudaStreamNonBlocking));
        QRNG_CUDA_TRY(cudaStreamCreateWithFlags(&g_cs.comp2, cudaStreamNonBlocking));
        g_cs.dev = dev;
    }
    *h2d = g_cs.h2d;
    *d2h = g_cs.d2h;
    *comp2 = g_cs.comp2;
    return QRNG_OK;
}

qrng_status qrng_toeplitz_extract_host(const uint8_t *h_raw_bits, uint64_t n_blocks, uint64_t n, uint64_t m,
                                       const uint8_t *h_seed, uint8_t *h_out, cudaStream_t stream) {
    qrng_status st = check_nm(n, m);
    if (st != QRNG_OK) return st;
    if (!h_raw_bits || !h_seed || !h_out) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    if (n_blocks == 0 || n_blocks > UINT64_MAX / n) { set_error("bad n_blocks"); return QRNG_E_INVALID; }
    if ((st = device_ready()) != QRNG_OK) return st;
    int dev = 0;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    cudaStream_t s_in, s_out, s_c2;
    if ((st = copy_streams(dev, &s_in, &s_out, &s_c2)) != QRNG_OK) return st;
    const uint64_t raw_bytes = n_blocks * n / 8, seed_bytes = (n + m - 1 + 7) / 8,
                   out_bytes = (n_blocks * m + 7) / 8;
    uint8_t *d_raw = nullptr, *d_seed = nullptr, *d_out = nullptr;
    {  // on any failure here, free what was already allocated (no early return past an allocation)
        cudaError_t e = cudaMallocAsync(&d_raw, raw_bytes, stream);
        if (e == cudaSuccess) e = cudaMallocAsync(&d_seed, seed_bytes, stream);
        if (e == cudaSuccess) e = cudaMallocAsync(&d_out, out_bytes, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_seed, h_seed, seed_bytes, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) {
            set_error("host path setup: %s", cudaGetErrorString(e));
            for (uint8_t *ptr : {d_raw, d_seed, d_out})
                if (ptr) cudaFreeAsync(ptr, stream);
            return e == cudaErrorMemoryAllocation ? QRNG_E_NOMEM : QRNG_E_CUDA;
        }
    }
    qrng_plan *plan = nullptr;
    st = qrng_plan_create(n, m, d_seed, stream, &plan);
    // Pipeline over chunks of whole 32-block granules: every chunk's key starts
    // on a 32-bit word boundary (32 m % 32 == 0) and its raw bytes on a 16-byte
    // boundary, so chunks are independent self-contained extractions.  Chunk kernels
    // alternate between two compute streams so a chunk's CTAs fill the SMs the
    // previous chunk's tail leaves idle.
    static const uint64_t kChunks = [] {  // QRNG_HOST_CHUNKS: pipeline depth override (experiments)
        const char *e = getenv("QRNG_HOST_CHUNKS");
        const long v = e ? atol(e) : 0;
        return (uint64_t)(v > 0 ? v : 8);
    }();
    const uint64_t G = (n_blocks + 31) / 32, K = G < kChunks ? G : kChunks;
    std::vector<cudaEvent_t> ev(3 * K + 1, nullptr);
    for (auto &e : ev)
        if (st == QRNG_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            set_error("cudaEventCreate failed");
            st = QRNG_E_CUDA;
        }
    if (st == QRNG_OK) {
        cudaEventRecord(ev[3 * K], stream);  // buffers allocated, plan enqueued
        cudaStreamWaitEvent(s_in, ev[3 * K], 0);
        cudaStreamWaitEvent(s_out, ev[3 * K], 0);
        cudaStreamWaitEvent(s_c2, ev[3 * K], 0);
    }
    for (uint64_t c = 0; c < K && st == QRNG_OK; ++c) {
        const uint64_t b0 = 32 * (c * G / K), b1 = std::min(n_blocks, 32 * ((c + 1) * G / K));
        const uint64_t r0 = b0 * n / 8, r1 = b1 * n / 8;
        const uint64_t o0 = b0 * m / 8, o1 = (c + 1 == K) ? out_bytes : b1 * m / 8;
        if (cudaMemcpyAsync(d_raw + r0, h_raw_bits + r0, r1 - r0, cudaMemcpyHostToDevice, s_in) != cudaSuccess) {
            set_error("H2D copy failed");
            st = QRNG_E_CUDA;
            break;
        }
        cudaEventRecord(ev[3 * c], s_in);
        cudaStream_t sc = (c & 1) ? s_c2 : stream;
        cudaStreamWaitEvent(sc, ev[3 * c], 0);
        st = qrng_plan_extract(plan, d_raw + r0, b1 - b0, d_out + o0, sc);
        if (st != QRNG_OK) break;
        cudaEventRecord(ev[3 * c + 1], sc);
        cudaStreamWaitEvent(s_out, ev[3 * c + 1], 0);
        if (cudaMemcpyAsync(h_out + o0, d_out + o0, o1 - o0, cudaMemcpyDeviceToHost, s_out) != cudaSuccess) {
            set_error("D2H copy failed");
            st = QRNG_E_CUDA;
            break;
        }
        cudaEventRecord(ev[3 * c + 2], s_out);
    }
    if (ev[3 * K]) {  // join the side streams back into `stream`
        cudaEventRecord(ev[3 * K], s_in);
        cudaStreamWaitEvent(stream, ev[3 * K], 0);
        cudaEventRecord(ev[3 * K], s_c2);
        cudaStreamWaitEvent(stream, ev[3 * K], 0);
        cudaEventRecord(ev[3 * K], s_out);
        cudaStreamWaitEvent(stream, ev[3 * K], 0);
    }
    if (plan) plan_release(plan, stream, true);
    cudaFreeAsync(d_raw, stream);
    cudaFreeAsync(d_seed, stream);
    cudaFreeAsync(d_out, stream);
    cudaError_t e = cudaStreamSynchronize(stream);
    for (auto &x : ev)
        if (x) cudaEventDestroy(x);
    if (e != cudaSuccess && st == QRNG_OK) {
        set_error("cudaStreamSynchronize: %s", cudaGetErrorString(e));
        st = QRNG_E_CUDA;
    }
    return st;
}

// ---- streaming ingest (NEXT-3) ------------------------------------------------
// Three-stage pipeline: host->device copies on s_in, extraction on s_comp (one
// batch at a time gets the whole GPU), device->host copies on s_out; `depth`
// device buffer pairs rotate, a slot being reused once its key copy is done.
struct qrng_stream {
    const qrng_plan *plan = nullptr;
    uint64_t max_blocks = 0;
    uint32_t depth = 0, flags = 0, next = 0;
    int dev = 0;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    struct Slot {
        cudaEvent_t in_done = nullptr, comp_done = nullptr, out_done = nullptr;
        uint8_t *d_raw = nullptr, *d_out = nullptr;
        bool busy = false;
    } slot[8];
    uint64_t *d_counts = nullptr;
    qrng_status err = QRNG_OK;
    char errmsg[512] = "";
};

static void stream_release(qrng_stream *st) {
    if (!st) return;
    for (cudaStream_t s : {st->s_in, st->s_comp, st->s_out})
        if (s) cudaStreamSynchronize(s);
    for (auto &sl : st->slot) {
        if (sl.d_raw) cudaFree(sl.d_raw);
        if (sl.d_out) cudaFree(sl.d_out);
        for (cudaEvent_t e : {sl.in_done, sl.comp_done, sl.out_done})
            if (e) cudaEventDestroy(e);
    }
    for (cudaStream_t s : {st->s_in, st->s_comp, st->s_out})
        if (s) cudaStreamDestroy(s);
    if (st->d_counts) cudaFree(st->d_counts);
    delete st;
}

qrng_status qrng_stream_create(const qrng_plan *plan, uint64_t max_blocks, uint32_t depth, uint32_t flags,
                               qrng_stream **out) {
    if (!plan || !out) { set_error("NULL argument"); return QRNG_E_INVALID; }
    *out = nullptr;
    if (max_blocks == 0 || depth < 2 || depth > 8) { set_error("need max_blocks > 0 and depth in [2, 8]"); return QRNG_E_INVALID; }
    if (max_blocks > UINT64_MAX / plan->n) { set_error("max_blocks * n overflows"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    qrng_stream *q = new (std::nothrow) qrng_stream;
    if (!q) { set_error("host allocation failed"); return QRNG_E_NOMEM; }
    q->plan = plan;
    q->max_blocks = max_blocks;
    q->depth = depth;
    q->flags = flags;
    cudaGetDevice(&q->dev);
    bool ok = cudaStreamCreateWithFlags(&q->s_in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&q->s_comp, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&q->s_out, cudaStreamNonBlocking) == cudaSuccess;
    const size_t raw_bytes = max_blocks * plan->n / 8, out_bytes = (max_blocks * plan->m + 7) / 8;
    for (uint32_t i = 0; i < depth && ok; ++i) {
        auto &sl = q->slot[i];
        ok = cudaEventCreateWithFlags(&sl.in_done, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&sl.comp_done, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&sl.out_done, cudaEventDisableTiming) == cudaSuccess &&
             cudaMalloc(&sl.d_raw, raw_bytes) == cudaSuccess && cudaMalloc(&sl.d_out, out_bytes) == cudaSuccess;
    }
    if (ok && (flags & QRNG_STREAM_HIST))
        ok = cudaMalloc(&q->d_counts, 256 * sizeof(uint64_t)) == cudaSuccess &&
             cudaMemset(q->d_counts, 0, 256 * sizeof(uint64_t)) == cudaSuccess;
    if (!ok) {
        set_error("stream allocation failed");
        stream_release(q);
        return QRNG_E_NOMEM;
    }
    *out = q;
    return QRNG_OK;
}

qrng_status qrng_stream_submit(qrng_stream *q, const uint8_t *h_raw_bits, uint64_t n_blocks, uint8_t *h_out) {
    if (!q || !h_raw_bits || !h_out) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (n_blocks == 0 || n_blocks > q->max_blocks) { set_error("n_blocks must be in [1, max_blocks]"); return QRNG_E_INVALID; }
    QRNG_CUDA_TRY(cudaSetDevice(q->dev));
    auto &sl = q->slot[q->next];
    q->next = (q->next + 1) % q->depth;
    if (sl.busy) QRNG_CUDA_TRY(cudaEventSynchronize(sl.out_done));  // the slot's previous batch is finished
    const uint64_t n = q->plan->n, m = q->plan->m;
    const size_t raw_bytes = n_blocks * n / 8, out_bytes = (n_blocks * m + 7) / 8;
    QRNG_CUDA_TRY(cudaMemcpyAsync(sl.d_raw, h_raw_bits, raw_bytes, cudaMemcpyHostToDevice, q->s_in));
    QRNG_CUDA_TRY(cudaEventRecord(sl.in_done, q->s_in));
    QRNG_CUDA_TRY(cudaStreamWaitEvent(q->s_comp, sl.in_done, 0));
    qrng_status st = QRNG_OK;
    if (q->d_counts)
        st = hist256_launch(sl.d_raw, raw_bytes, reinterpret_cast<unsigned long long *>(q->d_counts), q->s_comp);
    if (st == QRNG_OK) st = qrng_plan_extract(q->plan, sl.d_raw, n_blocks, sl.d_out, q->s_comp);
    if (st == QRNG_OK) {
        cudaError_t e = cudaEventRecord(sl.comp_done, q->s_comp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(q->s_out, sl.comp_done, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, sl.d_out, out_bytes, cudaMemcpyDeviceToHost, q->s_out);
        if (e == cudaSuccess) e = cudaEventRecord(sl.out_done, q->s_out);
        if (e != cudaSuccess) { set_error("stream copy: %s", cudaGetErrorString(e)); st = QRNG_E_CUDA; }
    }
    sl.busy = true;
    if (st != QRNG_OK && q->err == QRNG_OK) {
        q->err = st;
        snprintf(q->errmsg, sizeof q->errmsg, "%s", g_err);
    }
    return st;
}

qrng_status qrng_stream_synchronize(qrng_stream *q) {
    if (!q) { set_error("NULL argument"); return QRNG_E_INVALID; }
    for (uint32_t i = 0; i < q->depth; ++i) {
        auto &sl = q->slot[i];
        if (sl.busy) {
            cudaError_t e = cudaEventSynchronize(sl.out_done);
            sl.busy = false;
            if (e != cudaSuccess && q->err == QRNG_OK) {
                q->err = QRNG_E_CUDA;
                snprintf(q->errmsg, sizeof q->errmsg, "stream batch: %s", cudaGetErrorString(e));
            }
        }
    }
    const qrng_status st = q->err;
    if (st != QRNG_OK) set_error("%s", q->errmsg);
    q->err = QRNG_OK;
    return st;
}

qrng_status qrng_stream_counts(qrng_stream *q, uint64_t *h_counts256) {
    if (!q || !h_counts256) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (!q->d_counts) { set_error("stream created without QRNG_STREAM_HIST"); return QRNG_E_INVALID; }
    const qrng_status st = qrng_stream_synchronize(q);
    if (st != QRNG_OK) return st;
    QRNG_CUDA_TRY(cudaMemcpy(h_counts256, q->d_counts, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return QRNG_OK;
}

void qrng_stream_destroy(qrng_stream *q) { stream_release(q); }

// ---- NEXT-4: one block across GPUs ----------------------------------------------
struct qrng_dist_plan {
    ntt::DistPlan d;
};

qrng_status qrng_dist_plan_create(uint64_t n, uint64_t m, const uint8_t *d_seed, uint32_t world, uint32_t rank,
                                  cudaStream_t stream, qrng_dist_plan **plan) {
    if (!plan) { set_error("plan is NULL"); return QRNG_E_INVALID; }
    *plan = nullptr;
    qrng_status st = check_nm(n, m);
    if (st != QRNG_OK) return st;
    if (!d_seed || !aligned16(d_seed)) { set_error("d_seed is NULL or not 16-byte aligned"); return QRNG_E_INVALID; }
    if (world == 0 || world > 8 || (world & (world - 1)) || rank >= world) {
        set_error("world must be 1, 2, 4 or 8 and rank < world (got %u, %u)", world, rank);
        return QRNG_E_INVALID;
    }
    if ((st = device_ready()) != QRNG_OK) return st;
    qrng_dist_plan *p = new (std::nothrow) qrng_dist_plan;
    if (!p) { set_error("host allocation failed"); return QRNG_E_NOMEM; }
    st = ntt::dist_plan_init(p->d, n, m, d_seed, world, rank, stream);
    if (st != QRNG_OK) {
        ntt::dist_plan_free(p->d, stream, true);
        delete p;
        return st;
    }
    *plan = p;
    return QRNG_OK;
}

uint64_t qrng_dist_exchange_words(const qrng_dist_plan *plan) { return plan ? plan->d.N2 : 0; }

qrng_status qrng_dist_local(const qrng_dist_plan *plan, const uint8_t *d_block_bits, uint32_t *d_buf,
                            cudaStream_t stream) {
    if (!plan || !d_block_bits || !d_buf) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (!aligned16(d_buf)) { set_error("d_buf must be 16-byte aligned"); return QRNG_E_INVALID; }
    if (overlap(d_block_bits, (plan->d.n + 7) / 8, d_buf, (uint64_t)plan->d.N2 * 4)) {
        set_error("d_buf overlaps d_block_bits");
        return QRNG_E_INVALID;
    }
    return ntt::dist_local(plan->d, d_block_bits, d_buf, stream);
}

qrng_status qrng_dist_finish(const qrng_dist_plan *plan, const uint32_t *d_recv, uint8_t *d_key,
                             cudaStream_t stream) {
    if (!plan || !d_recv || !d_key) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (((uintptr_t)d_key & 3u) != 0) { set_error("d_key must be 4-byte aligned"); return QRNG_E_INVALID; }
    const uint64_t m = plan->d.m, key_bytes = (m + 7) / 8;
    if (overlap(d_recv, (uint64_t)plan->d.N2 * 4, d_key, key_bytes)) {
        set_error("d_key overlaps d_recv");
        return QRNG_E_INVALID;
    }
    OutStream o;
    o.words = reinterpret_cast<uint32_t *>(d_key);
    o.total_bits = m;
    o.full_words = key_bytes / 4;
    o.tail = nullptr;
    if (key_bytes % 4) {  // the final partial word goes through a scratch word (nothing past key_bytes is touched)
        cudaError_t e = cudaMallocAsync(&o.tail, 4, stream);
        if (e != cudaSuccess) { set_error("cudaMallocAsync: %s", cudaGetErrorString(e)); return QRNG_E_NOMEM; }
        QRNG_CUDA_TRY(cudaMemcpyAsync(o.tail, d_key + (key_bytes / 4) * 4, key_bytes % 4, cudaMemcpyDeviceToDevice,
                                      stream));
    }
    qrng_status st = ntt::dist_finish(plan->d, d_recv, o, 0, stream);
    if (st == QRNG_OK && o.tail) {
        cudaError_t e = cudaMemcpyAsync(d_key + (key_bytes / 4) * 4, o.tail, key_bytes % 4, cudaMemcpyDeviceToDevice,
                                        stream);
        if (e != cudaSuccess) { set_error("tail copy: %s", cudaGetErrorString(e)); st = QRNG_E_CUDA; }
    }
    if (o.tail) cudaFreeAsync(o.tail, stream);
    return st;
}

void qrng_dist_plan_destroy(qrng_dist_plan *plan) {
    if (!plan) return;
    ntt::dist_plan_free(plan->d, 0, false);
    delete plan;
}

// ---- min-entropy ------------------------

qrng_status qrng_hist256_async(const uint8_t *d_samples, uint64_t n_samples, uint64_t *d_counts,
                               cudaStream_t stream) {
    if (!d_samples || !d_counts) { set_error("NULL buffer"); return QRNG_E_INVALID; }
    if (n_samples == 0) { set_error("n_samples must be > 0"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    return hist256_launch(d_samples, n_samples, reinterpret_cast<unsigned long long *>(d_counts), stream);
}

static double std_normal_cdf(double z) { return 0.5 * (1.0 + erf(z / sqrt(2.0))); }

qrng_status qrng_entropy_from_counts(const uint64_t *h_counts, uint32_t bit_depth, const qrng_gauss *model,
                                     uint64_t n, uint32_t s, qrng_entropy_report *rep) {
    if (!h_counts || !rep) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (bit_depth < 1 || bit_depth > 8) { set_error("bit_depth must be in [1, 8]"); return QRNG_E_INVALID; }
    memset(rep, 0, sizeof *rep);
    const int K = 1 << bit_depth;
    uint64_t total = 0, cmax = 0;
    for (int k = 0; k < 256; ++k) {
        rep->counts[k] = h_counts[k];
        total += h_counts[k];
        if (k >= K && h_counts[k]) {
            set_error("sample value %d >= 2^bit_depth", k);
            return QRNG_E_INVALID;
        }
        if (h_counts[k] > cmax) cmax = h_counts[k];
    }
    rep->n_samples = total;
    rep->bit_depth = bit_depth;
    if (total == 0) { set_error("empty histogram"); return QRNG_E_INVALID; }
    const double T = (double)total;
    // H_min of the empirical distribution P'(x) = counts / T
    rep->h_min_hist = -log2((double)cmax / T);
    double mu, sigma;
    if (model) {
        mu = model->mu;
        sigma = model->sigma;
    } else {  // reading A10: moments of the histogram, population sigma
        double s1 = 0, s2 = 0;
        for (int k = 0; k < K; ++k) {
            s1 += (double)k * (double)h_counts[k];
            s2 += (double)k * (double)k * (double)h_counts[k];
        }
        mu = s1 / T;
        double var = s2 / T - mu * mu;
        sigma = sqrt(var > 0 ? var : 0);
    }
    rep->mu = mu;
    rep->sigma = sigma;
    if (!(sigma > 0)) { set_error("model sigma must be > 0"); return QRNG_E_INVALID; }
    // ideal model P: N(mu, sigma^2) on bins [k-1/2, k+1/2), tails in the edge bins
    double pmax = 0, d = 0, prev = 0;
    for (int k = 0; k < K; ++k) {
        double cdf = (k == K - 1) ? 1.0 : std_normal_cdf(((double)k + 0.5 - mu) / sigma);
        double pk = cdf - prev;
        prev = cdf;
        if (pk > pmax) pmax = pk;
        d += fabs((double)h_counts[k] / T - pk);
    }
    d *= 0.5;                                                     // d_U
    rep->h_min_ideal = -log2(pmax);
    rep->stat_dist = d;
    rep->delta_h_m = log2(d / pow(2.0, -(double)bit_depth - 1.0) + 1.0);
    double hm = rep->h_min_ideal - rep->delta_h_m;
    rep->h_min_mod = hm > 0 ? hm : 0.0;
    rep->m = (int64_t)floor((double)n * rep->h_min_mod / (double)bit_depth) - (int64_t)s;
    if (rep->m <= 0) {
        set_error("derived m = %lld <= 0", (long long)rep->m);
        return QRNG_E_NO_OUTPUT;
    }
    return QRNG_OK;
}

qrng_status qrng_minentropy(const uint8_t *d_samples, uint64_t n_samples, uint32_t bit_depth,
                            const qrng_gauss *model, uint64_t n, uint32_t s, qrng_entropy_report *rep,
                            cudaStream_t stream) {
    if (!d_samples || !rep) { set_error("NULL argument"); return QRNG_E_INVALID; }
    if (n_samples == 0) { set_error("n_samples must be > 0"); return QRNG_E_INVALID; }
    if (bit_depth < 1 || bit_depth > 8) { set_error("bit_depth must be in [1, 8]"); return QRNG_E_INVALID; }
    if (model && !(model->sigma > 0)) { set_error("model sigma must be > 0"); return QRNG_E_INVALID; }
    qrng_status st = device_ready();
    if (st != QRNG_OK) return st;
    uint64_t *d_counts = nullptr;
    uint64_t h[256];
    QRNG_CUDA_TRY(cudaMallocAsync(&d_counts, 256 * sizeof(uint64_t), stream));
    QRNG_CUDA_TRY(cudaMemsetAsync(d_counts, 0, 256 * sizeof(uint64_t), stream));
    st = hist256_launch(d_samples, n_samples, reinterpret_cast<unsigned long long *>(d_counts), stream);
    if (st == QRNG_OK) {
        cudaError_t e = cudaMemcpyAsync(h, d_counts, sizeof h, cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) { set_error("histogram copy: %s", cudaGetErrorString(e)); st = QRNG_E_CUDA; }
    }
    cudaFreeAsync(d_counts, stream);
    if (st != QRNG_OK) return st;
    return qrng_entropy_from_counts(h, bit_depth, model, n, s, rep);
}

}  // extern "C"
