// karatsuba.cu -- sub-quadratic Toeplitz products on the tcgen05 GEMM path.
//
// Method: y = T x mod 2 with T[i][j] = s[i - j + n - 1] (PAPER.md:189-197,
// reading C1).  The paper lowers the O(mn) cost with an FFT;
// here the work stays on the int8 tensor cores but the product is split
// Karatsuba-style over GF(2) (SURVEY.md 8(f) NEXT-2 "carry-less Karatsuba"),
// so the tensor cores run a quarter less work per level.
//
// For an r x w Toeplitz product with h = w/2 and r > h, split x = (x0, x1)
// and the rows at h.  The four h x h blocks are Toeplitz with seeds
//     A = T00 = T11 : d[h, 3h-1)     B = T01 : d[0, 2h-1)     C = T10 : d[2h, ...)
// (T00 and T11 share their diagonals), so over GF(2)
//     Q  = A (x0 ^ x1)              (h x h)
//     P2 = (A ^ B) x1               (h x h)
//     P3 = (A ^ C)[:r-h] x0         ((r-h) x h)
//     y[0, h) = Q ^ P2,   y[h, r) = Q[0, r-h) ^ P3
// -- three half-size Toeplitz products instead of four, each again of the
// form "seed window times block", because A ^ B is the Toeplitz matrix of the
// XOR of the two seed windows.  If r <= h the columns are split instead
// (y = T[:, :h] x0 ^ T[:, h:] x1, two r x h products) so that the halves can be
// split again.  Applied recursively, every leaf is a Toeplitz product whose
// seed is an XOR of windows of s (prepared once per plan) and whose input is
// an XOR of windows of the block (formed per batch); all leaves run in ONE
// grouped launch of the tcgen05 kernel (gemm_tc.cu), which writes word-aligned
// leaf parities; a combine kernel XORs them back up the tree and packs the key
// (C4).  Exactness: every step is a GF(2) identity and each leaf is exact
// int32 accumulation followed by & 1.
#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include "qrng_internal.cuh"

namespace qrng {
namespace kara {

constexpr uint32_t kMinLeafW = 128;   // narrowest leaf the planner creates (one K stage)
constexpr int kMaxLeaves = 1024;
constexpr int kMaxDepth = 10;

// ---- planner (host only; no CUDA calls) ------------------------------------
// Cost model in units of (output row x K) for one M tile of 128 blocks on the
// tensor cores; per-tile pipeline overhead and the workspace traffic of the
// input / parity combinations are expressed in the same unit (calibrated on
// B200).
constexpr double kTileOverhead = 150e3;  // per work tile (pipeline fill, accumulator drain)
constexpr double kPrepPerBit = 100.0;    // forming x0 ^ x1 in the workspace, per input bit
constexpr double kCombPerRow = 50.0;     // leaf parities written + combined, per output row

static double leaf_cost(uint32_t r, uint32_t w) {
    double c = 0;
    for (uint32_t n0 = 0; n0 < r; n0 += gemm::kTileRows) {
        const uint32_t left = std::min<uint32_t>(gemm::kTileRows, r - n0);
        const uint32_t rows = std::max<uint32_t>((left + 15) & ~15u, 128);  // A expansion floor
        c += (double)rows * w + kTileOverhead;
    }
    return c;
}

enum { LEAF = 0, KARA = 1, COLS = 2 };

struct Node {
    int kind;
    uint32_t r, w, h;
    int child[3];
};

static bool can_split(uint32_t w) { return w % 256 == 0 && w / 2 >= kMinLeafW; }

struct Planner {
    std::map<std::tuple<uint32_t, uint32_t, int>, std::pair<double, int>> memo;
    bool forced;  // forced depth: split whenever allowed

    std::pair<double, int> best(uint32_t r, uint32_t w, int depth) {
        auto key = std::make_tuple(r, w, depth);
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
        std::pair<double, int> res{leaf_cost(r, w), LEAF};
        if (depth > 0 && can_split(w)) {
            const uint32_t h = w / 2;
            if (r > h) {
                const double c = 2 * best(h, h, depth - 1).first + best(r - h, h, depth - 1).first +
                                 kPrepPerBit * h + kCombPerRow * r;
                if (forced || c < res.first) res = {c, KARA};
            } else {
                const double c = 2 * best(r, h, depth - 1).first + kCombPerRow * r;
                if (forced || c < res.first) res = {c, COLS};
            }
        }
        memo[key] = res;
        return res;
    }

    int build(uint32_t r, uint32_t w, int depth, std::vector<Node> &nodes) {
        const int kind = best(r, w, depth).second;
        const int id = (int)nodes.size();
        nodes.push_back(Node{kind, r, w, w / 2, {-1, -1, -1}});
        if (kind == KARA) {
            const uint32_t h = w / 2;
            const int a = build(h, h, depth - 1, nodes);
            const int b = build(h, h, depth - 1, nodes);
            const int c = build(r - h, h, depth - 1, nodes);
            nodes[id].child[0] = a; nodes[id].child[1] = b; nodes[id].child[2] = c;
        } else if (kind == COLS) {
            const int a = build(r, w / 2, depth - 1, nodes);
            const int b = build(r, w / 2, depth - 1, nodes);
            nodes[id].child[0] = a; nodes[id].child[1] = b;
        }
        return id;
    }
};

// Host form of the decomposition.
struct HostLeaf {
    uint32_t r, w;
    std::vector<uint32_t> sterms, iterms;  // bit offsets into the root seed / the raw block
    uint32_t out_off = 0;                  // word offset in a block's Y row
    int src = -1;                          // input buffer: -1 raw block, else Q buffer index
    uint32_t src_off = 0;                  // bit offset of the input window in that buffer
};
// Q = x0 ^ x1 of a Karatsuba node, materialised once per block in the X
// workspace; its children read windows of it.  gen = nesting depth of Q buffers.
struct QBuf {
    uint32_t gen, h;                       // generation (1 = from the raw block); bits
    int src;                               // parent buffer (-1 raw)
    uint32_t src_off;                      // bit offset of x0 in the parent (x1 = x0 + h)
    uint32_t dst = 0;                      // word offset in a block's X row
};
struct HostTables {
    int depth = 0;
    std::vector<HostLeaf> leaves;          // sorted by w (descending) = tile order
    std::vector<QBuf> qbufs;               // sorted by generation
    uint32_t max_gen = 0;
    // internal nodes for the bottom-up combine, sorted by height: {kind, words,
    // h/32, dst word in a block's Z row, child locations (word offset | 1<<31 if in Z)}
    std::vector<std::array<uint32_t, 8>> inner;
    std::vector<uint32_t> height_end;      // inner[height_end[h-1] .. height_end[h]) have height h
    uint32_t z_stride = 0, root_z = 0;
    std::vector<uint32_t> comb_ptr, comb_idx;  // CSR per root output word -> Y-row word offsets
    uint32_t y_stride = 0, x_stride = 0, total_npairs = 0, root_words = 0, seed_total = 0;
    uint64_t macs = 0;                     // leaf multiply-accumulates per block
};

static void collect(const std::vector<Node> &nodes, int id, std::vector<uint32_t> so, std::vector<uint32_t> io,
                    int src, uint32_t src_off, uint32_t gen, std::vector<int> &leaf_of_node,
                    std::vector<HostLeaf> &leaves, std::vector<QBuf> &qbufs) {
    const Node &nd = nodes[id];
    if (nd.kind == LEAF) {
        leaf_of_node[id] = (int)leaves.size();
        HostLeaf L{nd.r, nd.w, so, io, 0, src, src_off};
        leaves.push_back(L);
        return;
    }
    const uint32_t h = nd.h;
    auto plus = [](const std::vector<uint32_t> &v, uint32_t d) {
        std::vector<uint32_t> o(v);
        for (auto &x : o) x += d;
        return o;
    };
    auto cat = [](std::vector<uint32_t> a, const std::vector<uint32_t> &b) {
        a.insert(a.end(), b.begin(), b.end());
        return a;
    };
    if (nd.kind == KARA) {
        const int q = (int)qbufs.size();
        qbufs.push_back(QBuf{gen + 1, h, src, src_off, 0});
        collect(nodes, nd.child[0], plus(so, h), cat(io, plus(io, h)), q, 0, gen + 1, leaf_of_node, leaves, qbufs);  // Q
        collect(nodes, nd.child[1], cat(plus(so, h), so), plus(io, h), src, src_off + h, gen, leaf_of_node, leaves,
                qbufs);                                                                                   // P2
        collect(nodes, nd.child[2], cat(plus(so, h), plus(so, 2 * h)), io, src, src_off, gen, leaf_of_node, leaves,
                qbufs);                                                                                   // P3
    } else {
        collect(nodes, nd.child[0], plus(so, h), io, src, src_off, gen, leaf_of_node, leaves, qbufs);      // T[:, :h] x0
        collect(nodes, nd.child[1], so, plus(io, h), src, src_off + h, gen, leaf_of_node, leaves, qbufs);  // T[:, h:] x1
    }
}

// Y-row words whose XOR is word j of node id's output.
static void contrib(const std::vector<Node> &nodes, const std::vector<int> &leaf_of_node,
                    const std::vector<HostLeaf> &leaves, int id, uint32_t j, std::vector<uint32_t> &out) {
    const Node &nd = nodes[id];
    if (nd.kind == LEAF) {
        out.push_back(leaves[leaf_of_node[id]].out_off + j);
        return;
    }
    if (nd.kind == KARA) {
        const uint32_t hw = nd.h / 32;
        if (j < hw) {
            contrib(nodes, leaf_of_node, leaves, nd.child[0], j, out);
            contrib(nodes, leaf_of_node, leaves, nd.child[1], j, out);
        } else {
            contrib(nodes, leaf_of_node, leaves, nd.child[0], j - hw, out);
            contrib(nodes, leaf_of_node, leaves, nd.child[2], j - hw, out);
        }
    } else {
        contrib(nodes, leaf_of_node, leaves, nd.child[0], j, out);
        contrib(nodes, leaf_of_node, leaves, nd.child[1], j, out);
    }
}

static bool plan_host_depth(uint64_t n, uint64_t m, int depth, bool forced, HostTables &T);

static bool plan_host(uint64_t n, uint64_t m, int max_depth, HostTables &T) {
    if (n % 128 || m == 0 || m >= n || n > (1u << 22)) return false;
    // auto: the cost model's best tree with at most kMaxLeaves leaves
    for (int depth = max_depth >= 0 ? std::min(max_depth, kMaxDepth) : kMaxDepth; depth >= 0; --depth)
        if (plan_host_depth(n, m, depth, max_depth >= 0, T)) return true;
    return false;
}

static bool plan_host_depth(uint64_t n, uint64_t m, int depth, bool forced, HostTables &T) {
    Planner pl;
    pl.forced = forced;
    std::vector<Node> nodes;
    pl.build((uint32_t)m, (uint32_t)n, depth, nodes);
    std::vector<int> leaf_of_node(nodes.size(), -1);
    std::vector<HostLeaf> leaves;
    std::vector<QBuf> qbufs;
    collect(nodes, 0, {0}, {0}, -1, 0, 0, leaf_of_node, leaves, qbufs);
    if ((int)leaves.size() > kMaxLeaves) return false;
    // depth of the tree
    std::vector<int> dep(nodes.size(), 0);
    int maxd = 0;
    for (size_t i = 0; i < nodes.size(); ++i)
        for (int c : nodes[i].child)
            if (c >= 0) { dep[c] = dep[i] + 1; maxd = std::max(maxd, dep[c]); }
    T = HostTables{};
    T.depth = maxd;
    // Y rows: leaves in tree order; tile order: widest leaves first (longest tiles first)
    uint32_t yo = 0;
    for (auto &L : leaves) {
        L.out_off = yo;
        yo += (L.r + 31) / 32;
        T.macs += (uint64_t)L.r * L.w;
    }
    T.y_stride = (yo + 3) & ~3u;
    const uint32_t ywords = (uint32_t)((m + 31) / 32);
    T.comb_ptr.push_back(0);
    for (uint32_t j = 0; j < ywords; ++j) {
        contrib(nodes, leaf_of_node, leaves, 0, j, T.comb_idx);
        T.comb_ptr.push_back((uint32_t)T.comb_idx.size());
    }
    // internal nodes: heights, Z rows, child locations
    std::vector<int> height(nodes.size(), 0);
    for (int i = (int)nodes.size() - 1; i >= 0; --i)  // children have larger ids than parents
        for (int c : nodes[i].child)
            if (c >= 0) height[i] = std::max(height[i], height[c] + 1);
    std::vector<int> inner_ids;
    for (size_t i = 0; i < nodes.size(); ++i)
        if (nodes[i].kind != LEAF) inner_ids.push_back((int)i);
    std::stable_sort(inner_ids.begin(), inner_ids.end(), [&](int a, int b) { return height[a] < height[b]; });
    std::vector<uint32_t> zoff(nodes.size(), 0);
    uint32_t zo = 0;
    for (int i : inner_ids) { zoff[i] = zo; zo += (nodes[i].r + 31) / 32; }
    T.z_stride = (zo + 3) & ~3u;
    T.root_z = zoff[0];
    auto loc = [&](int c) -> uint32_t {
        if (c < 0) return 0;
        return nodes[c].kind == LEAF ? leaves[leaf_of_node[c]].out_off : (zoff[c] | 0x80000000u);
    };
    T.height_end.assign(maxd + 1, 0);
    for (int i : inner_ids) {
        const Node &nd = nodes[i];
        T.inner.push_back({(uint32_t)nd.kind, (nd.r + 31) / 32, nd.h / 32, zoff[i], loc(nd.child[0]),
                           loc(nd.child[1]), loc(nd.child[2]), 0u});
        for (int h = height[i]; h <= maxd; ++h) T.height_end[h] = (uint32_t)T.inner.size();
    }
    std::stable_sort(leaves.begin(), leaves.end(), [](const HostLeaf &a, const HostLeaf &b) { return a.w > b.w; });
    T.leaves = leaves;
    // X row: Q buffers in generation order (a buffer's parent is always earlier)
    std::vector<int> order(qbufs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return qbufs[a].gen < qbufs[b].gen; });
    uint32_t xo = 0;
    for (int i : order) {
        qbufs[i].dst = xo;
        xo += qbufs[i].h / 32;
        T.max_gen = std::max(T.max_gen, qbufs[i].gen);
    }
    for (int i : order) T.qbufs.push_back(qbufs[i]);
    std::vector<int> pos(qbufs.size());
    for (size_t j = 0; j < order.size(); ++j) pos[order[j]] = (int)j;
    for (auto &Q : T.qbufs)
        if (Q.src >= 0) Q.src = pos[Q.src];
    for (auto &L : T.leaves)
        if (L.src >= 0) L.src = pos[L.src];
    uint32_t np = 0, so = 0, rw = 0;
    for (auto &L : T.leaves) {
        np += (L.r + gemm::kTileRows - 1) / gemm::kTileRows;
        const uint32_t sw = gemm::seed_words_needed(L.w, L.r);
        so += (sw + 3) & ~3u;
        for (uint32_t t : L.sterms) rw = std::max(rw, t / 32 + sw + 2);
    }
    T.x_stride = xo;
    T.total_npairs = np;
    T.seed_total = so;
    T.root_words = rw;
    return true;
}

// ---- device tables (cached per device and (n, m, depth)) ------------------
struct Tables {
    HostTables host;
    gemm::Leaf *leaves = nullptr;  // device
    uint32_t *terms = nullptr;     // device: seed and input terms
    uint4 *qbufs = nullptr;        // device: {src word offset (raw: in block; X: in row), words, dst, src is X}
    uint32_t *inner = nullptr;     // device: internal-node table (8 words per node)
    std::vector<gemm::Leaf> hleaves;
};

static qrng_status get_tables(uint64_t n, uint64_t m, int max_depth, const Tables **out) {
    static std::mutex mu;
    static std::map<std::tuple<int, uint64_t, uint64_t, int>, Tables *> cache;
    int dev = 0;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, n, m, max_depth);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return QRNG_OK; }
    Tables *t = new Tables;
    if (!plan_host(n, m, max_depth, t->host)) {
        delete t;
        set_error("Karatsuba planner: no decomposition for n=%llu m=%llu", (unsigned long long)n,
                  (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    const HostTables &H = t->host;
    std::vector<uint32_t> terms;
    uint32_t npb = 0, so = 0;
    std::vector<uint4> hq;
    for (const auto &Q : H.qbufs) {
        const uint32_t off = Q.src < 0 ? Q.src_off / 32 : H.qbufs[Q.src].dst + Q.src_off / 32;
        hq.push_back(make_uint4(off, Q.h / 32, Q.dst, Q.src < 0 ? 0u : 1u));
    }
    for (const auto &L : H.leaves) {
        gemm::Leaf g{};
        g.w = L.w;
        g.r = L.r;
        g.npairs = (L.r + gemm::kTileRows - 1) / gemm::kTileRows;
        g.npair_base = npb;
        npb += g.npairs;
        g.seed_off = so;
        g.seed_n = gemm::seed_words_needed(L.w, L.r);
        so += (g.seed_n + 3) & ~3u;
        if (L.src < 0) { g.x_src = 0; g.x_off = L.src_off / 32; }
        else { g.x_src = 1; g.x_off = H.qbufs[L.src].dst + L.src_off / 32; }
        g.out_off = L.out_off;
        g.sterm_base = (uint32_t)terms.size();
        g.sterm_n = (uint32_t)L.sterms.size();
        terms.insert(terms.end(), L.sterms.begin(), L.sterms.end());
        g.iterm_base = 0;  // inputs come from the Q buffers; the expanded terms are host-only
        g.iterm_n = 0;
        t->hleaves.push_back(g);
    }
    cudaError_t e = cudaMalloc(&t->leaves, t->hleaves.size() * sizeof(gemm::Leaf));
    if (e == cudaSuccess) e = cudaMalloc(&t->terms, terms.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&t->inner, H.inner.size() * 32 + 32);
    if (e == cudaSuccess && !hq.empty()) e = cudaMalloc(&t->qbufs, hq.size() * sizeof(uint4));
    if (e == cudaSuccess && !hq.empty()) e = cudaMemcpy(t->qbufs, hq.data(), hq.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(t->leaves, t->hleaves.data(), t->hleaves.size() * sizeof(gemm::Leaf), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(t->terms, terms.data(), terms.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !H.inner.empty())
        e = cudaMemcpy(t->inner, H.inner.data(), H.inner.size() * 32, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        set_error("Karatsuba tables: %s", cudaGetErrorString(e));
        cudaFree(t->leaves); cudaFree(t->terms); cudaFree(t->inner); cudaFree(t->qbufs);
        delete t;
        return QRNG_E_CUDA;
    }
    cache[key] = t;
    *out = t;
    return QRNG_OK;
}

bool choose(uint64_t n, uint64_t m, int max_depth) {
    if (max_depth == 0) return false;
    HostTables T;
    if (!plan_host(n, m, max_depth, T)) return false;
    return T.depth > 0;
}

// ---- kernels ---------------------------------------------------------------
__device__ __forceinline__ uint32_t bswap(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// seed bytes (MSB-first) -> logical big-endian words, zero past L
__global__ void root_words_kernel(const uint8_t *seed, uint64_t L, uint32_t *words, uint32_t nwords) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const uint64_t byte = (uint64_t)w * 4 + k;
            v |= (byte * 8 < L ? (uint32_t)seed[byte] : 0u) << (24 - 8 * k);
        }
        const uint64_t lo = (uint64_t)w * 32;
        if (lo + 32 > L) v &= (L > lo) ? (0xFFFFFFFFu << (32 - (L - lo))) : 0u;
        words[w] = v;
    }
}

// Leaf seeds: word q of leaf l = XOR over its terms t of root bits [t + 32q, t + 32q + 32),
// zero at and past the leaf seed length r + w - 1.
__global__ void leaf_seed_kernel(const gemm::Leaf *leaves, const uint32_t *terms, const uint32_t *root,
                                 uint32_t *seeds) {
    const gemm::Leaf L = leaves[blockIdx.y];
    const uint32_t nw = L.seed_n;
    const uint32_t len = L.r + L.w - 1;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nw; q += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (uint32_t k = 0; k < L.sterm_n; ++k) {
            const uint32_t pos = terms[L.sterm_base + k] + 32 * q;
            v ^= __funnelshift_l(root[(pos >> 5) + 1], root[pos >> 5], pos & 31);
        }
        const uint32_t lo = 32 * q;
        if (lo + 32 > len) v &= (len > lo) ? (0xFFFFFFFFu << (32 - (len - lo))) : 0u;
        seeds[L.seed_off + q] = v;
    }
}

// Q buffers of one generation: X[b][dst + g] = S[b][off + g] ^ S[b][off + h/32 + g]
// (x0 ^ x1 of a Karatsuba node; S = raw block or an earlier Q buffer; 16-byte
// granules).  blockIdx.y = buffer; each CTA covers `per` blocks per pass.
__global__ void __launch_bounds__(256) qbuf_kernel(const uint4 *qb, uint32_t q0, const uint4 *raw, uint64_t n_blocks,
                                                   uint32_t n, uint4 *xws, uint32_t x_stride) {
    const uint4 Q = qb[q0 + blockIdx.y];  // {src word offset, words, dst word offset, src is X}
    const uint32_t gper = Q.y / 4;
    const uint32_t per = gper >= blockDim.x ? 1u : blockDim.x / gper;
    const uint32_t bl = gper >= blockDim.x ? 0u : threadIdx.x / gper;
    const uint32_t g0 = gper >= blockDim.x ? threadIdx.x : threadIdx.x - bl * gper;
    const uint32_t gstep = gper >= blockDim.x ? blockDim.x : gper;
    if (bl >= per) return;
    for (uint64_t b = (uint64_t)blockIdx.x * per + bl; b < n_blocks; b += (uint64_t)gridDim.x * per) {
        const uint4 *src = Q.w ? xws + b * (x_stride / 4) : raw + b * (n / 128);
        uint4 *dst = xws + b * (x_stride / 4) + Q.z / 4;
        for (uint32_t g = g0; g < gper; g += gstep) {
            const uint4 u = src[Q.x / 4 + g], v = src[(Q.x + Q.y) / 4 + g];
            dst[g] = make_uint4(u.x ^ v.x, u.y ^ v.y, u.z ^ v.z, u.w ^ v.w);
        }
    }
}

// Combine, one launch per height: node output word j of block b (Z row) =
//   KARA: j < h/32 ? Q[j] ^ P2[j] : Q[j - h/32] ^ P3[j - h/32]      (y0 = Q^P2, y1 = Q^P3)
//   COLS: L[j] ^ R[j]
// children read from the leaf parities (Y) or lower nodes (Z); coalesced words.
__global__ void __launch_bounds__(256) combine_kernel(const uint32_t *inner, uint32_t i0, const uint32_t *yws,
                                                      uint32_t y_stride, uint32_t *zws, uint32_t z_stride,
                                                      uint64_t n_blocks) {
    const uint32_t *nd = inner + 8 * (i0 + blockIdx.y);
    const uint32_t kind = nd[0], words = nd[1], hw = nd[2], dst = nd[3];
    const uint32_t c0 = nd[4], c1 = nd[5], c2 = nd[6];
    const uint32_t per = words >= blockDim.x ? 1u : blockDim.x / words;
    const uint32_t bl = words >= blockDim.x ? 0u : threadIdx.x / words;
    const uint32_t j0 = words >= blockDim.x ? threadIdx.x : threadIdx.x - bl * words;
    const uint32_t jstep = words >= blockDim.x ? blockDim.x : words;
    if (bl >= per) return;
    for (uint64_t b = (uint64_t)blockIdx.x * per + bl; b < n_blocks; b += (uint64_t)gridDim.x * per) {
        const uint32_t *Y = yws + b * y_stride;
        uint32_t *Z = zws + b * z_stride;
        auto at = [&](uint32_t c, uint32_t w) { return (c >> 31) ? Z[(c & 0x7FFFFFFFu) + w] : Y[c + w]; };
        for (uint32_t j = j0; j < words; j += jstep) {
            uint32_t v;
            if (kind == 1) v = j < hw ? (at(c0, j) ^ at(c1, j)) : (at(c0, j - hw) ^ at(c2, j - hw));
            else v = at(c0, j) ^ at(c1, j);
            Z[dst + j] = v;
        }
    }
}

// Key stream (C4): CTA c owns blocks [32c, 32c+32), whose keys fill exactly
// the output words [c*m, (c+1)*m) (32 m bits).  Word w of the group holds bits
// [32w, 32w+32) of the group; block b's key is the first m bits of its root
// row.  Every word has one writer (no pre-zeroing); a final partial word goes
// to the tail scratch.
__global__ void __launch_bounds__(256) pack_kernel(const uint32_t *rows, uint32_t stride, uint32_t off,
                                                   uint64_t n_blocks, uint32_t m, OutStream out) {
    const uint64_t b0 = (uint64_t)blockIdx.x * 32;
    const uint32_t nb = (uint32_t)min((uint64_t)32, n_blocks - b0);
    const uint32_t gbits = nb * m, gwords = (gbits + 31) / 32, rw = (m + 31) / 32;
    for (uint32_t w = threadIdx.x; w < gwords; w += blockDim.x) {
        const uint32_t G = w * 32, end = min(G + 32, gbits);
        uint32_t b = G / m, i = G - b * m, pos = G, word = 0;
        while (pos < end) {
            const uint32_t len = min(m - i, end - pos);  // 1..32 bits of block b
            const uint32_t *row = rows + (b0 + b) * stride + off;
            const uint32_t q = i >> 5, s = i & 31;
            const uint32_t w0 = row[q], w1 = (s && q + 1 < rw) ? row[q + 1] : 0u;
            const uint32_t bits = s ? ((w0 << s) | (w1 >> (32 - s))) : w0;  // rows i.. at the MSB
            word |= (bits >> (32 - len)) << (32 - len - (pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, (uint64_t)blockIdx.x * m + w, word, true);
    }
}

// ---- host entry points -----------------------------------------------------
qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, int max_depth, const uint8_t *d_seed, cudaStream_t s) {
    const Tables *t = nullptr;
    qrng_status st = get_tables(n, m, max_depth, &t);
    if (st != QRNG_OK) return st;
    pl.tab = t;
    const HostTables &H = t->host;
    uint32_t *root = nullptr;
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.seeds, (size_t)H.seed_total * 4, s));
    QRNG_CUDA_TRY(cudaMallocAsync(&root, (size_t)H.root_words * 4, s));
    count_launch();
    root_words_kernel<<<(H.root_words + 255) / 256, 256, 0, s>>>(d_seed, n + m - 1, root, H.root_words);
    QRNG_CUDA_TRY(cudaGetLastError());
    uint32_t maxw = 0;
    for (const auto &g : t->hleaves) maxw = std::max(maxw, g.seed_n);
    count_launch();
    leaf_seed_kernel<<<dim3((maxw + 127) / 128, (unsigned)t->hleaves.size()), 128, 0, s>>>(t->leaves, t->terms, root,
                                                                                           pl.seeds);
    QRNG_CUDA_TRY(cudaGetLastError());
    cudaFreeAsync(root, s);
    return QRNG_OK;
}

void plan_free(Plan &pl) {
    if (pl.seeds) cudaFree(pl.seeds);
    pl = Plan{};
}

void describe(const Plan &pl, int *depth, int *n_leaves, uint64_t *macs_per_block) {
    if (!pl.tab) { *depth = 0; *n_leaves = 0; *macs_per_block = 0; return; }
    *depth = pl.tab->host.depth;
    *n_leaves = (int)pl.tab->host.leaves.size();
    *macs_per_block = pl.tab->host.macs;
}

qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                    const OutStream &out, cudaStream_t s) {
    const Tables *t = pl.tab;
    const HostTables &H = t->host;
    uint32_t *xws = nullptr, *yws = nullptr;
    if (H.x_stride) QRNG_CUDA_TRY(cudaMallocAsync(&xws, (size_t)n_blocks * H.x_stride * 4, s));
    QRNG_CUDA_TRY(cudaMallocAsync(&yws, (size_t)n_blocks * H.y_stride * 4, s));
    qrng_status st = QRNG_OK;
    // Q buffers generation by generation (each reads its parent generation)
    for (uint32_t gen = 1, q0 = 0; gen <= H.max_gen && st == QRNG_OK; ++gen) {
        uint32_t q1 = q0, maxw = 0;
        while (q1 < H.qbufs.size() && H.qbufs[q1].gen == gen) maxw = std::max(maxw, H.qbufs[q1++].h / 32);
        const uint32_t per = std::max<uint32_t>(1, 256 / std::max<uint32_t>(1, maxw / 4));
        const unsigned gx = (unsigned)std::min<uint64_t>((n_blocks + per - 1) / per, 4096);
        count_launch();
        qbuf_kernel<<<dim3(gx, q1 - q0), 256, 0, s>>>(t->qbufs, q0, reinterpret_cast<const uint4 *>(d_raw), n_blocks,
                                                      (uint32_t)n, reinterpret_cast<uint4 *>(xws), H.x_stride);
        if (cudaGetLastError() != cudaSuccess) { set_error("qbuf_kernel launch failed"); st = QRNG_E_CUDA; }
        q0 = q1;
    }
    if (st == QRNG_OK)
        st = gemm::extract_grouped(t->leaves, (uint32_t)t->hleaves.size(), H.total_npairs, pl.seeds, d_raw, n_blocks,
                                   n, xws, H.x_stride, yws, H.y_stride, s);
    uint32_t *zws = nullptr;
    if (st == QRNG_OK && cudaMallocAsync(&zws, (size_t)n_blocks * H.z_stride * 4, s) != cudaSuccess) {
        set_error("cudaMallocAsync failed");
        st = QRNG_E_NOMEM;
    }
    for (size_t h = 1; h < H.height_end.size() && st == QRNG_OK; ++h) {
        const uint32_t i0 = H.height_end[h - 1], i1 = H.height_end[h];
        if (i1 == i0) continue;
        uint32_t maxw = 0;
        for (uint32_t i = i0; i < i1; ++i) maxw = std::max(maxw, H.inner[i][1]);
        const uint32_t per = std::max<uint32_t>(1, 256 / std::max<uint32_t>(1, maxw));
        const unsigned gx = (unsigned)std::min<uint64_t>((n_blocks + per - 1) / per, 8192);
        count_launch();
        combine_kernel<<<dim3(gx, i1 - i0), 256, 0, s>>>(t->inner, i0, yws, H.y_stride, zws, H.z_stride, n_blocks);
        if (cudaGetLastError() != cudaSuccess) { set_error("combine_kernel launch failed"); st = QRNG_E_CUDA; }
    }
    if (st == QRNG_OK) {
        count_launch();
        pack_kernel<<<(unsigned)((n_blocks + 31) / 32), 256, 0, s>>>(
            zws, H.z_stride, H.root_z, n_blocks, (uint32_t)m, out);
        if (cudaGetLastError() != cudaSuccess) { set_error("pack_kernel launch failed"); st = QRNG_E_CUDA; }
    }
    if (zws) cudaFreeAsync(zws, s);
    if (xws) cudaFreeAsync(xws, s);
    cudaFreeAsync(yws, s);
    return st;
}

}  // namespace kara
}  // namespace qrng

// ---- TEST ONLY: the host planner's decomposition (no GPU needed) ------------
// See include/qrng.h (qrng_debug_karatsuba_plan).
extern "C" qrng_status qrng_debug_karatsuba_plan(uint64_t n, uint64_t m, int max_depth, uint32_t *leaf_rw,
                                                 uint32_t leaf_cap, uint32_t *terms, uint32_t term_cap,
                                                 uint32_t *comb, uint32_t comb_cap, uint32_t *counts) {
    using namespace qrng;
    using namespace qrng::kara;
    HostTables T;
    if (!counts) { set_error("counts is NULL"); return QRNG_E_INVALID; }
    if (!plan_host(n, m, max_depth, T)) { set_error("no decomposition"); return QRNG_E_UNSUPPORTED; }
    uint32_t nterms = 0;
    for (const auto &L : T.leaves) nterms += (uint32_t)(L.sterms.size() + L.iterms.size());
    counts[0] = (uint32_t)T.leaves.size();
    counts[1] = nterms;
    counts[2] = (uint32_t)T.comb_idx.size();
    counts[3] = (uint32_t)T.depth;
    if (!leaf_rw || !terms || !comb || leaf_cap < T.leaves.size() || term_cap < nterms ||
        comb_cap < T.comb_idx.size() + T.comb_ptr.size())
        return QRNG_OK;  // sizes only
    uint32_t tp = 0;
    for (size_t l = 0; l < T.leaves.size(); ++l) {
        const auto &L = T.leaves[l];
        uint32_t *e = leaf_rw + 6 * l;
        e[0] = L.r; e[1] = L.w; e[2] = L.out_off;
        e[3] = tp; e[4] = (uint32_t)L.sterms.size(); e[5] = (uint32_t)L.iterms.size();
        for (uint32_t v : L.sterms) terms[tp++] = v;
        for (uint32_t v : L.iterms) terms[tp++] = v;
    }
    for (size_t j = 0; j < T.comb_ptr.size(); ++j) comb[j] = T.comb_ptr[j];
    for (size_t j = 0; j < T.comb_idx.size(); ++j) comb[T.comb_ptr.size() + j] = T.comb_idx[j];
    return QRNG_OK;
}
