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
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <array>
#include <list>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include "qrng_internal.cuh"

namespace qrng {
namespace kara {

#ifndef QRNG_CSR_THREADS
#define QRNG_CSR_THREADS 512  // threads of the combine+pack kernel
#endif
constexpr uint32_t kMinLeafW = 128;   // narrowest leaf the planner creates (one K stage)
#ifndef QRNG_KARA_MAXLEAVES
// the leaf table is staged in the GEMM kernel's shared memory (32 B per leaf):
// 2,187 leaves (3^7) = 70 KB next to the B ring and A stages (~200 KB in all)
#define QRNG_KARA_MAXLEAVES 2187
#endif
constexpr int kMaxLeaves = QRNG_KARA_MAXLEAVES;
constexpr int kMaxDepth = 10;
// auto mode: deeper trees spill the leaf parities out of L2 (measured: depth 6
// loses at n = 2^16, wins at 2^17).  At n >= 2^18 depth 7 (the
// 2048-wide packed leaves, with B reuse across tile runs): 2^18 69.8 -> 77.3
// Gbit/s (tools/kara_d7_ab.sh)
static int auto_max_depth(uint64_t n) { return n >= (1u << 18) ? 7 : n >= (1u << 17) ? 6 : 5; }

// ---- planner (host only; no CUDA calls) ------------------------------------
// Cost model in units of (output row x K) for one M tile of 128 blocks on the
// tensor cores; per-tile pipeline overhead and the workspace traffic of the
// input / parity combinations are expressed in the same unit (calibrated on
// B200).
// Fitted on the int8 kernel.  Re-checked on the E2M1 kernel (which does the
// row x K work in about half the tensor time) with a full depth scan,
// profiles/kara_depths_r1j.jsonl: the same constants pick the measured best
// depth at 2^12, 2^13, 2^14, 2^16, 2^17, 2^18 and one level too deep at 2^15
// (223 vs 232 Gbit/s); halving the MAC weight would pick d0 at 2^13 (-6%) and
// d4 at 2^16 (-3.5%).  QRNG_KARA_MAC_WEIGHT overrides it for calibration.
constexpr double kTileOverhead = 186e3;  // per work tile (pipeline fill, accumulator drain; ~3.6k SM clocks)
constexpr double kPrepPerBit = 180.0;    // forming x0 ^ x1 in the workspace, per input bit
constexpr double kLeafRow = 250.0;       // leaf parities written by the GEMM and read by the combine, per row
constexpr double kCombPerRow = 0.0;      // internal node row written and read back, per row
static double mac_weight() {
    static const double w = [] {
        const char *e = getenv("QRNG_KARA_MAC_WEIGHT");  // calibration override
        return e ? atof(e) : 1.0;
    }();
    return w;
}

static double leaf_cost(uint32_t r, uint32_t w) {
    double c = kLeafRow * r;
    for (uint32_t n0 = 0; n0 < r; n0 += gemm::kTileRows) {
        const uint32_t left = std::min<uint32_t>(gemm::kTileRows, r - n0);
        const uint32_t rows = std::max<uint32_t>((left + 15) & ~15u, 128);  // A expansion floor
        c += mac_weight() * (double)rows * w + kTileOverhead;
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
    // inside a tree (w below the root's), split leaves wider than the E2M1
    // kernel's packed-accumulator limit so that the whole launch can use it
    uint32_t root_w = 0, pack_w = 0;

    std::pair<double, int> best(uint32_t r, uint32_t w, int depth) {
        auto key = std::make_tuple(r, w, depth);
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
        std::pair<double, int> res{leaf_cost(r, w), LEAF};
        if (depth > 0 && can_split(w)) {
            const uint32_t h = w / 2;
            const bool pack_split = pack_w && w < root_w && w > pack_w;
            if (r > h) {
                const double c = 2 * best(h, h, depth - 1).first + best(r - h, h, depth - 1).first +
                                 kPrepPerBit * h + kCombPerRow * r;
                if (forced || pack_split || c < res.first) res = {c, KARA};
            } else {
                const double c = 2 * best(r, h, depth - 1).first + kCombPerRow * r;
                if (forced || pack_split || c < res.first) res = {c, COLS};
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
    std::vector<std::array<uint32_t, 4>> levels;  // {first node, end node, units per block, unit_node offset}; root last
    std::vector<uint32_t> unit_node;       // per level: 16-byte unit -> node index
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
    // auto: the cost model's best tree with at most kMaxLeaves leaves picks the
    // depth; the tree itself is then the uniform one (every node split down to
    // that depth), measured at least as fast as the cost model's mixed trees
    // (profiles/kara_depths_r1q.jsonl: 2^14 d3 484 vs 443 Gbit/s, 2^15 d4 273
    // vs 259, equal elsewhere)
    for (int depth = max_depth >= 0 ? std::min(max_depth, kMaxDepth) : auto_max_depth(n); depth >= 0; --depth)
        if (plan_host_depth(n, m, depth, max_depth >= 0, T)) {
            if (max_depth < 0 && T.depth > 0) {
                HostTables U;
                if (plan_host_depth(n, m, T.depth, true, U)) T = std::move(U);
            }
            return true;
        }
    return false;
}

static bool plan_host_depth(uint64_t n, uint64_t m, int depth, bool forced, HostTables &T) {
    Planner pl;
    pl.forced = forced;
    pl.root_w = (uint32_t)n;
    static const bool pack_split = [] {
        const char *e = getenv("QRNG_KARA_PACK_SPLIT");  // calibration override
        return e ? atoi(e) != 0 : true;
    }();
    // measured (profiles/sweep_r1n.jsonl, tools/ab_pack.sh): splitting for the
    // packed accumulators pays at config 2 (2^13, 16384 blocks: 510 -> 528
    // Gbit/s) and from 2^16 (2048-wide leaves: 156 -> 166), loses at 2^14 /
    // 2^15 (398 -> 391, 226 -> 204)
    const bool pack_here = n <= 8192 || n >= 65536;
    if (pack_split && pack_here) pl.pack_w = 2048;  // gemm_tc.cu kMaxPackedK
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
        yo += ((L.r + 31) / 32 + 3) & ~3u;  // 16-byte aligned rows: the combine moves uint4
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
    for (int i : inner_ids)
        if (i != 0) { zoff[i] = zo; zo += ((nodes[i].r + 31) / 32 + 3) & ~3u; }  // the root is packed directly
    T.z_stride = (zo + 3) & ~3u;
    T.root_z = zoff[0];
    auto loc = [&](int c) -> uint32_t {
        if (c < 0) return 0;
        return nodes[c].kind == LEAF ? leaves[leaf_of_node[c]].out_off : (zoff[c] | 0x80000000u);
    };
    T.height_end.assign(maxd + 1, 0);
    uint32_t pre = 0;
    int cur_h = 0;
    for (int i : inner_ids) {
        const Node &nd = nodes[i];
        if (height[i] != cur_h) { cur_h = height[i]; pre = 0; }
        const uint32_t words = (nd.r + 31) / 32;
        // nd[7]: first 16-byte unit of this node within its level (item numbering)
        T.inner.push_back({(uint32_t)nd.kind, words, nd.h / 32, zoff[i], loc(nd.child[0]), loc(nd.child[1]),
                           loc(nd.child[2]), pre});
        pre += (words + 3) / 4;
        for (int h = height[i]; h <= maxd; ++h) T.height_end[h] = (uint32_t)T.inner.size();
    }
    // levels {first node, end node, 16-byte units per block}; the root level (last)
    // counts the root row plus one zero unit (the pack reads one word past a row)
    for (int h = 1; h <= maxd; ++h) {
        const uint32_t i0 = T.height_end[h - 1], i1 = T.height_end[h];
        if (i1 == i0) continue;
        const auto &last = T.inner[i1 - 1];
        uint32_t u = last[7] + (last[1] + 3) / 4;
        if (h == maxd) u += 1;
        T.levels.push_back({i0, i1, u, (uint32_t)T.unit_node.size()});
        for (uint32_t i = i0; i < i1; ++i)  // unit -> node of this level
            for (uint32_t v = 0; v < (T.inner[i][1] + 3) / 4; ++v) T.unit_node.push_back(i);
        if (h == maxd) T.unit_node.push_back(i1 - 1);  // the root's zero unit
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

// One-pass Q-buffer form (qslice_kernel): each Q buffer as the XOR of raw
// windows x[o, o + h) (symmetric difference of the parent's expansion shifted
// to x0 and x1), cut into chunks of the narrowest Q width s; chunk = {mask of
// the block's n / s aligned s-bit slices, destination 16-byte unit in the X
// row}.  Returns n / s, or 0 when the tree has no Q buffers or needs more than
// 16 slices / 80 chunks (the generation kernel then forms them).
struct QSliceHost {
    uint32_t n_ent = 0, lsu = 0;  // chunks; log2 of 16-byte units per slice
    uint32_t ent[80] = {};        // slice mask (bits 0..15) | destination unit (bits 16..31)
};
static int qslice_host(const HostTables &H, uint64_t n, QSliceHost &qs) {
    qs = QSliceHost{};
    if (H.qbufs.empty()) return 0;
    uint32_t s = UINT32_MAX;
    for (const auto &Q : H.qbufs) s = std::min(s, Q.h);
    if (s % 128 || n % s || n / s > 16) return 0;
    const uint64_t ns = n / s;
    std::vector<std::vector<uint32_t>> ex(H.qbufs.size());  // sorted raw offsets (bits)
    std::vector<std::array<uint32_t, 2>> ent;
    for (size_t qi = 0; qi < H.qbufs.size(); ++qi) {
        const QBuf &Q = H.qbufs[qi];
        const std::vector<uint32_t> par = Q.src < 0 ? std::vector<uint32_t>{0} : ex[Q.src];
        std::map<uint32_t, int> cnt;
        for (uint32_t o : par) { cnt[o + Q.src_off] ^= 1; cnt[o + Q.src_off + Q.h] ^= 1; }
        for (const auto &kv : cnt)
            if (kv.second) ex[qi].push_back(kv.first);
        for (uint32_t c = 0; c < Q.h / s; ++c) {
            uint32_t mask = 0;
            for (uint32_t o : ex[qi]) {
                const uint64_t bit = o + (uint64_t)c * s;
                if (bit % s || bit / s >= ns) return 0;
                mask ^= 1u << (bit / s);
            }
            const uint32_t dw = Q.dst + c * s / 32;  // destination word in the X row
            if (dw % 4 || dw / 4 >= 65536) return 0;
            ent.push_back({mask, dw / 4});
        }
    }
    if (ent.size() > 80) return 0;
    uint32_t lsu = 0;
    while ((1u << lsu) < s / 128) ++lsu;
    if ((1u << lsu) != s / 128) return 0;
    qs.n_ent = (uint32_t)ent.size();
    qs.lsu = lsu;
    for (size_t i = 0; i < ent.size(); ++i) qs.ent[i] = ent[i][0] | (ent[i][1] << 16);
    return (int)ns;
}

// ---- device tables (cached per device and (n, m, depth)) ------------------
struct Tables {
    HostTables host;
    gemm::Leaf *leaves = nullptr;  // device
    uint32_t *terms = nullptr;     // device: seed and input terms
    uint4 *qbufs = nullptr;        // device: per 16-byte unit of the Q buffers (see get_tables)
    std::vector<uint32_t> qgen;    // first unit of each generation (+ end)
    uint32_t *qgen_dev = nullptr;
    uint32_t *inner = nullptr;     // device: internal-node table (8 words per node)
    uint4 *levels = nullptr;       // device: level table
    uint32_t *unit_node = nullptr; // device: unit -> node per level
    uint32_t *csr = nullptr;       // device: root word -> Y-row words (counts, then column-major entries)
    uint32_t csr_words = 0;
    uint32_t csr_kmax = 0;         // most entries of one key word
    // the same flattened tree as runs Z[dst, dst + len) ^= Y[src, src + len),
    // in batches of runs with disjoint dst ranges (see csr_run_key_kernel)
    uint4 *runs = nullptr;         // device: {dst, src, len, 0}, batch-major
    uint32_t *run_ptr = nullptr;   // device: first run of each batch (+ end)
    uint32_t n_batches = 0, n_runs = 0;
    std::vector<gemm::Leaf> hleaves;
    uint32_t max_leaf_w = 0;       // widest leaf (K) -- the packed-accumulator kernel takes w <= 2048
    int qs_ns = 0;                 // slices of the one-pass Q-buffer form (0: trees it does not cover)
    QSliceHost qs;                 // its chunk list (= QSlice, defined with the kernels)
    ~Tables() {
        // the last owner is the cache or a plan; cudaFree waits for the work that reads them
        for (void *ptr : {(void *)leaves, (void *)terms, (void *)qbufs, (void *)qgen_dev, (void *)inner,
                          (void *)levels, (void *)unit_node, (void *)csr, (void *)runs, (void *)run_ptr})
            if (ptr) cudaFree(ptr);
    }
};

// Device tables are shared by every plan of the same (device, n, m, depth) and
// cached so that one-shot calls do not re-plan.  The cache is bounded (LRU,
// kTableCacheCap entries): a long-running process that re-derives m from live
// min-entropy creates a new (n, m) per re-plan, and evicted tables are freed
// once the last plan holding them is destroyed (shared ownership).
constexpr size_t kTableCacheCap = 16;

static qrng_status get_tables(uint64_t n, uint64_t m, int max_depth, std::shared_ptr<const Tables> *out) {
    using Key = std::tuple<int, uint64_t, uint64_t, int>;
    static std::mutex mu;
    static std::list<std::pair<Key, std::shared_ptr<const Tables>>> lru;  // front = most recent
    int dev = 0;
    QRNG_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const Key key = std::make_tuple(dev, n, m, max_depth);
    for (auto it = lru.begin(); it != lru.end(); ++it)
        if (it->first == key) {
            lru.splice(lru.begin(), lru, it);
            *out = lru.front().second;
            return QRNG_OK;
        }
    auto t = std::make_shared<Tables>();
    if (!plan_host(n, m, max_depth, t->host)) {
        set_error("Karatsuba planner: no decomposition for n=%llu m=%llu", (unsigned long long)n,
                  (unsigned long long)m);
        return QRNG_E_UNSUPPORTED;
    }
    const HostTables &H = t->host;
    std::vector<uint32_t> terms;
    uint32_t npb = 0, so = 0;
    std::vector<uint4> hq;
    // one entry per 16-byte unit of every Q buffer, generation by generation:
    // {x0 word offset in the source row, h/32, destination word in the X row, source is X}
    for (uint32_t gen = 1; gen <= H.max_gen; ++gen) {
        t->qgen.push_back((uint32_t)hq.size());
        for (const auto &Q : H.qbufs) {
            if (Q.gen != gen) continue;
            const uint32_t off = Q.src < 0 ? Q.src_off / 32 : H.qbufs[Q.src].dst + Q.src_off / 32;
            for (uint32_t g = 0; g < Q.h / 128; ++g)
                hq.push_back(make_uint4(off + 4 * g, Q.h / 32, Q.dst + 4 * g, Q.src < 0 ? 0u : 1u));
        }
    }
    t->qgen.push_back((uint32_t)hq.size());
    t->qs_ns = qslice_host(H, n, t->qs);  // one-pass Q-buffer form (qslice_kernel)
    for (const auto &L : H.leaves) {
        gemm::Leaf g{};
        g.w = L.w;
        g.r = L.r;
        t->max_leaf_w = std::max(t->max_leaf_w, L.w);
        g.npairs = (L.r + gemm::kTileRows - 1) / gemm::kTileRows;
        // equal tiles (no narrow N = 64 tail MMA, which runs at ~60% of the pipe rate)
        g.pair_rows = ((L.r + g.npairs - 1) / g.npairs + 31) & ~31u;
        if (g.pair_rows > gemm::kTileRows) g.pair_rows = gemm::kTileRows;
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
    if (e == cudaSuccess) e = cudaMalloc(&t->qgen_dev, t->qgen.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(t->qgen_dev, t->qgen.data(), t->qgen.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(t->leaves, t->hleaves.data(), t->hleaves.size() * sizeof(gemm::Leaf), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(t->terms, terms.data(), terms.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !H.inner.empty())
        e = cudaMemcpy(t->inner, H.inner.data(), H.inner.size() * 32, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&t->levels, H.levels.size() * 16 + 16);
    if (e == cudaSuccess) e = cudaMalloc(&t->unit_node, H.unit_node.size() * 4 + 4);
    // the flattened tree for the combine kernel, column-major so that threads
    // taking consecutive key words read consecutive shared-memory words:
    // [count per word (ywords)] [entry k of word j at ywords + k*ywords + j]
    {
        const uint32_t yw = (uint32_t)H.comb_ptr.size() - 1;
        uint32_t kmax = 0;
        for (uint32_t j = 0; j < yw; ++j) kmax = std::max(kmax, H.comb_ptr[j + 1] - H.comb_ptr[j]);
        std::vector<uint32_t> cm(yw + (size_t)kmax * yw, 0);
        for (uint32_t j = 0; j < yw; ++j) {
            cm[j] = H.comb_ptr[j + 1] - H.comb_ptr[j];
            for (uint32_t q = 0; q < cm[j]; ++q) cm[yw + (size_t)q * yw + j] = H.comb_idx[H.comb_ptr[j] + q];
        }
        t->csr_words = (uint32_t)cm.size();
        t->csr_kmax = kmax;
        if (e == cudaSuccess) e = cudaMalloc(&t->csr, cm.size() * 4);
        if (e == cudaSuccess) e = cudaMemcpy(t->csr, cm.data(), cm.size() * 4, cudaMemcpyHostToDevice);
        // runs: key word j takes Y word j + d for the entries of each offset d;
        // maximal stretches of consecutive j with the same d are one run.
        // Batches: interval partitioning by dst (runs sorted by dst, each into
        // the first batch that ended before it starts), so runs of one batch
        // never write the same key word; the batch count is the deepest overlap
        // (kmax).
        std::map<int64_t, std::vector<uint32_t>> by_d;
        for (uint32_t j = 0; j < yw; ++j)
            for (uint32_t q = H.comb_ptr[j]; q < H.comb_ptr[j + 1]; ++q) by_d[(int64_t)H.comb_idx[q] - j].push_back(j);
        std::vector<std::array<uint32_t, 3>> rr;  // {dst, src, len}
        for (const auto &kv : by_d) {
            const std::vector<uint32_t> &js = kv.second;
            for (size_t i = 0; i < js.size();) {
                size_t k = i + 1;
                while (k < js.size() && js[k] == js[k - 1] + 1) ++k;
                rr.push_back({js[i], (uint32_t)((int64_t)js[i] + kv.first), (uint32_t)(k - i)});
                i = k;
            }
        }
        std::sort(rr.begin(), rr.end());
        std::vector<uint32_t> bend;                      // end of each batch's last run
        std::vector<std::vector<std::array<uint32_t, 3>>> bat;
        for (const auto &r : rr) {
            size_t bi = 0;
            while (bi < bend.size() && bend[bi] > r[0]) ++bi;
            if (bi == bend.size()) { bend.push_back(0); bat.emplace_back(); }
            bend[bi] = r[0] + r[2];
            bat[bi].push_back(r);
        }
        std::vector<uint4> hr;
        std::vector<uint32_t> hp{0};
        for (const auto &b : bat) {
            for (const auto &r : b) hr.push_back(make_uint4(r[0], r[1], r[2], 0));
            hp.push_back((uint32_t)hr.size());
        }
        t->n_batches = (uint32_t)bat.size();
        t->n_runs = (uint32_t)hr.size();
        if (e == cudaSuccess) e = cudaMalloc(&t->runs, hr.size() * sizeof(uint4) + 16);
        if (e == cudaSuccess) e = cudaMalloc(&t->run_ptr, hp.size() * 4);
        if (e == cudaSuccess && !hr.empty()) e = cudaMemcpy(t->runs, hr.data(), hr.size() * sizeof(uint4), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(t->run_ptr, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess && !H.unit_node.empty())
        e = cudaMemcpy(t->unit_node, H.unit_node.data(), H.unit_node.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !H.levels.empty())
        e = cudaMemcpy(t->levels, H.levels.data(), H.levels.size() * 16, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        set_error("Karatsuba tables: %s", cudaGetErrorString(e));
        return QRNG_E_CUDA;  // t's destructor frees what was allocated
    }
    lru.emplace_front(key, t);
    while (lru.size() > kTableCacheCap) lru.pop_back();
    *out = lru.front().second;
    return QRNG_OK;
}

// Planner decision, cached on the host per (n, m, depth) (plan creation sits
// inside the one-shot call; re-planning would stall the launch sequence).
bool choose(uint64_t n, uint64_t m, int max_depth) {
    if (max_depth == 0) return false;
    static std::mutex mu;
    static std::map<std::tuple<uint64_t, uint64_t, int>, bool> cache;
    const auto key = std::make_tuple(n, m, max_depth);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    HostTables T;
    const bool use = plan_host(n, m, max_depth, T) && T.depth > 0;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = use;
    return use;
}

// ---- kernels ---------------------------------------------------------------
__device__ __forceinline__ uint32_t bswap(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// 32 seed bits [pos, pos+32) of an MSB-first byte buffer as a logical
// big-endian word, zero at and past bit L.
__device__ __forceinline__ uint32_t seed_window32(const uint8_t *seed, uint64_t L, uint64_t pos) {
    if (pos >= L) return 0u;
    const uint64_t b = pos >> 3, nbytes = (L + 7) / 8;
    uint32_t r;
    const uint64_t w = pos >> 5;  // two aligned words hold bits [32w, 32w + 64) (the seed is 16-byte aligned)
    if ((w + 2) * 4 <= nbytes) {
        const uint32_t *s32 = reinterpret_cast<const uint32_t *>(seed);
        const uint32_t hi = __byte_perm(__ldg(s32 + w), 0, 0x0123), lo = __byte_perm(__ldg(s32 + w + 1), 0, 0x0123);
        r = __funnelshift_l(lo, hi, (uint32_t)(pos & 31));
    } else {
        uint64_t v = 0;
        for (int i = 0; i < 5; ++i) v = (v << 8) | (b + i < nbytes ? seed[b + i] : 0u);
        r = (uint32_t)(v >> (8 - (pos & 7)));
    }
    if (pos + 32 > L) r &= 0xFFFFFFFFu << (32 - (uint32_t)(L - pos));
    return r;
}

// Leaf seeds: word q of leaf l = XOR over its terms t of seed bits [t + 32q, t + 32q + 32)
// (zero past n+m-1), zero at and past the leaf seed length r + w - 1.
__device__ __forceinline__ void leaf_seed_words(const gemm::Leaf &Lf, const uint32_t *terms, const uint8_t *seed,
                                                uint64_t L, uint32_t *seeds, uint32_t q0, uint32_t stride) {
    const uint32_t len = Lf.r + Lf.w - 1;
    for (uint32_t q = q0; q < Lf.seed_n; q += stride) {
        uint32_t v = 0;
#pragma unroll 8
        for (uint32_t k = 0; k < Lf.sterm_n; ++k) v ^= seed_window32(seed, L, __ldg(terms + Lf.sterm_base + k) + 32ull * q);
        const uint32_t lo = 32 * q;
        if (lo + 32 > len) v &= (len > lo) ? (0xFFFFFFFFu << (32 - (len - lo))) : 0u;
        seeds[Lf.seed_off + q] = v;
    }
}

__global__ void leaf_seed_kernel(const gemm::Leaf *leaves, const uint32_t *terms, const uint8_t *seed, uint64_t L,
                                 uint32_t *seeds) {
    leaf_seed_words(leaves[blockIdx.y], terms, seed, L, seeds, blockIdx.x * blockDim.x + threadIdx.x,
                    gridDim.x * blockDim.x);
}

// One-shot calls: the leaf seeds of a fresh plan are formed by extra CTAs of
// the Q-buffer launch (the two are independent), so plan preparation costs no
// launch of its own; the grouped GEMM's programmatic wait covers both.
struct SeedJob {
    const gemm::Leaf *leaves;
    const uint32_t *terms;
    const uint8_t *seed;       // null: no seed work in this launch
    uint64_t L;
    uint32_t *seeds;
    uint32_t n_leaves, q_ctas;  // CTAs [q_ctas, gridDim.x) do seed work
};

// All Q buffers of a few blocks, generation by generation (one launch):
// X[b][dst] = S[b][x0] ^ S[b][x0 + h/32] per 16-byte unit (x0 ^ x1 of a
// Karatsuba node; S = the raw block or an earlier Q buffer of the same block,
// written by this CTA before the __syncthreads that separates generations).
// Every (block, unit) of a generation is an independent item; U per thread
// with their loads in flight together.
template <int U>
__global__ void __launch_bounds__(512) qbuf_kernel(const uint4 *units, const uint32_t *gen_start, uint32_t n_gen,
                                                   const uint4 *raw, uint64_t n_blocks, uint32_t n, uint4 *xws,
                                                   uint32_t x_stride, uint32_t bpc, SeedJob sj) {
    pdl_release();  // the grouped GEMM may be scheduled as CTAs finish
    if (blockIdx.x >= sj.q_ctas) {  // leaf-seed CTAs (one-shot calls)
        for (uint32_t l = blockIdx.x - sj.q_ctas; l < sj.n_leaves; l += gridDim.x - sj.q_ctas)
            leaf_seed_words(sj.leaves[l], sj.terms, sj.seed, sj.L, sj.seeds, threadIdx.x, blockDim.x);
        return;
    }
    const uint64_t b0 = (uint64_t)blockIdx.x * bpc;
    const uint32_t nb = (uint32_t)min((uint64_t)bpc, n_blocks - b0);
    const uint32_t xs4 = x_stride / 4, rs4 = n / 128;
    for (uint32_t gi = 0; gi < n_gen; ++gi) {
        if (gi) __syncthreads();  // this generation reads the previous one
        const uint32_t u0 = gen_start[gi], per = gen_start[gi + 1] - u0, total = nb * per;
        for (uint32_t base = threadIdx.x; base < total; base += U * blockDim.x) {
            uint4 a[U], c[U];
            uint4 *dst[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t idx = base + u * blockDim.x;
                dst[u] = nullptr;
                if (idx < total) {
                    const uint32_t bl = idx / per, r = idx - bl * per;
                    const uint4 e = __ldg(units + u0 + r);
                    const uint64_t b = b0 + bl;
                    const uint4 *src = e.w ? xws + b * xs4 : raw + b * rs4;
                    a[u] = src[e.x / 4];
                    c[u] = src[(e.x + e.y) / 4];
                    dst[u] = xws + b * xs4 + e.z / 4;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (dst[u]) *dst[u] = make_uint4(a[u].x ^ c[u].x, a[u].y ^ c[u].y, a[u].z ^ c[u].z, a[u].w ^ c[u].w);
        }
    }
}

// All Q buffers of shallow trees in one pass, no generation barrier (round 2).
// Every Q buffer of width h is an XOR of windows x[o, o + h) of the raw block
// with o a multiple of h (the node inputs sit at multiples of their width), so
// with s = the narrowest Q width each s-bit chunk of a Q buffer is the XOR of
// a fixed set of the block's NS = n / s aligned s-bit slices.  Thread (block,
// unit j of a slice) loads unit j of every slice once (NS 16-byte loads, all in
// flight) and writes unit j of every Q chunk from registers; the host lists
// each chunk as {slice mask, destination unit in the X row}.
constexpr int kQSliceMaxEnt = 80;  // Q chunks at NS = 16: (3^4 - 2^4) = 65
struct QSlice {
    uint32_t n_ent, lsu;           // chunks; log2 of 16-byte units per slice
    uint32_t ent[kQSliceMaxEnt];   // slice mask (bits 0..15) | destination unit (bits 16..31)
};

template <int NS>
__global__ void __launch_bounds__(256) qslice_kernel(const __grid_constant__ QSlice qs, const uint4 *raw,
                                                     uint64_t n_blocks, uint4 *xws, uint32_t x_stride, SeedJob sj) {
    pdl_release();  // the grouped GEMM may be scheduled as CTAs finish
    if (blockIdx.x >= sj.q_ctas) {  // leaf-seed CTAs (one-shot calls)
        for (uint32_t l = blockIdx.x - sj.q_ctas; l < sj.n_leaves; l += gridDim.x - sj.q_ctas)
            leaf_seed_words(sj.leaves[l], sj.terms, sj.seed, sj.L, sj.seeds, threadIdx.x, blockDim.x);
        return;
    }
    const uint64_t item = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t b = item >> qs.lsu;
    if (b >= n_blocks) return;
    const uint32_t su = 1u << qs.lsu, j = (uint32_t)item & (su - 1);
    const uint4 *src = raw + b * (NS * su) + j;
    uint4 v[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) v[i] = __ldcs(src + i * su);  // read once: streaming
    uint4 *dst = xws + b * (x_stride / 4) + j;
    for (uint32_t e = 0; e < qs.n_ent; ++e) {
        const uint32_t en = qs.ent[e];
        uint4 a = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int i = 0; i < NS; ++i)
            if ((en >> i) & 1u) a = make_uint4(a.x ^ v[i].x, a.y ^ v[i].y, a.z ^ v[i].z, a.w ^ v[i].w);
        dst[en >> 16] = a;
    }
}

// Combine, one launch per height: node output words [4q, 4q+4) of block b (Z row) =
//   KARA: 4q < h/32 ? Q ^ P2 : Q[. - h/32] ^ P3[. - h/32]          (y0 = Q^P2, y1 = Q^P3)
//   COLS: L ^ R
// children read from the leaf parities (Y) or lower nodes (Z).  Every row and
// h/32 are multiples of 4 words, so each thread moves 16-byte vectors; words
// past a child's rows are don't-care (they only reach rows >= the node's r).
__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }
__device__ __forceinline__ uint4 node_word4(const uint32_t *nd, const uint4 *Y, const uint4 *Z, uint32_t q) {
    const uint32_t kind = nd[0], hq = nd[2] / 4;
    auto at = [&](uint32_t c, uint32_t i) { return (c >> 31) ? Z[(c & 0x7FFFFFFFu) / 4 + i] : Y[c / 4 + i]; };
    if (kind == 1) return q < hq ? xor4(at(nd[4], q), at(nd[5], q)) : xor4(at(nd[4], q - hq), at(nd[6], q - hq));
    return xor4(at(nd[4], q), at(nd[5], q));
}

// One combine level for the nb blocks of a CTA: every (block, node, 16-byte
// unit) of the level is an independent item; each thread takes U items at a
// time with all their loads in flight before the stores.  Y: leaf parities of
// block b0 (row stride ys4 units); Z: node rows (stride zs4); the root level
// writes R (stride rs4; units past the root row are zero).
template <int U>
__device__ __forceinline__ void combine_level(const uint32_t *inner, const uint32_t *unit_node, uint4 lv, uint32_t nb,
                                              const uint4 *Y, uint32_t ys4, uint4 *Z, uint32_t zs4, uint4 *R,
                                              uint32_t rs4) {
    const uint32_t total = nb * lv.z;
    for (uint32_t base = threadIdx.x; base < total; base += U * blockDim.x) {
        uint4 va[U], vb[U];
        uint4 *dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t idx = base + u * blockDim.x;
            dst[u] = nullptr;
            va[u] = vb[u] = make_uint4(0, 0, 0, 0);
            if (idx < total) {
                const uint32_t bl = idx / lv.z, r = idx - bl * lv.z;
                const uint32_t *nd = inner + 8 * __ldg(unit_node + lv.w + r);
                const uint32_t q = r - nd[7], hq = nd[2] / 4;
                const uint4 *Yb = Y + bl * ys4;
                uint4 *Zb = Z + bl * zs4;
                dst[u] = R ? R + bl * rs4 + q : Zb + nd[3] / 4 + q;
                if (q < (nd[1] + 3) / 4) {
                    uint32_t c0 = nd[4], c1 = nd[5], qq = q;
                    if (nd[0] == 1 && q >= hq) { c1 = nd[6]; qq = q - hq; }  // y1 = Q ^ P3
                    const uint4 *p0 = (c0 >> 31) ? Zb + (c0 & 0x7FFFFFFFu) / 4 : Yb + c0 / 4;
                    const uint4 *p1 = (c1 >> 31) ? Zb + (c1 & 0x7FFFFFFFu) / 4 : Yb + c1 / 4;
                    va[u] = p0[qq];
                    vb[u] = p1[qq];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (dst[u]) *dst[u] = xor4(va[u], vb[u]);
    }
}

// Every level below the root for bpc blocks per CTA (node rows in global Z).
__global__ void __launch_bounds__(512) combine_kernel(const uint32_t *inner, const uint32_t *unit_node,
                                                      const uint4 *levels, uint32_t n_levels,
                                                      const uint32_t *yws, uint32_t y_stride, uint32_t *zws,
                                                      uint32_t z_stride, uint64_t n_blocks, uint32_t bpc) {
    const uint64_t b0 = (uint64_t)blockIdx.x * bpc;
    const uint32_t nb = (uint32_t)min((uint64_t)bpc, n_blocks - b0);
    for (uint32_t l = 0; l < n_levels; ++l) {
        if (l) __syncthreads();  // the next level reads this one
        combine_level<8>(inner, unit_node, levels[l], nb, reinterpret_cast<const uint4 *>(yws + b0 * y_stride),
                         y_stride / 4, reinterpret_cast<uint4 *>(zws + b0 * z_stride), z_stride / 4, nullptr, 0);
    }
}

// Key stream (C4): CTA c owns blocks [32c, 32c+32), whose keys fill exactly
// the output words [c*m, (c+1)*m) (32 m bits).  The root node (the last
// combine level) is evaluated here: STAGED = into shared memory first (rows of
// up to ~1600 words), else word by word from the children.  Word w of the group
// = bits [32w, 32w+32) of the concatenated keys (block b's key = the first m
// bits of its root row).  Every output word has one writer (no pre-zeroing); a
// final partial word goes to the tail scratch.
template <bool STAGED>
__global__ void __launch_bounds__(256) pack_kernel(const uint32_t *root, const uint32_t *yws, uint32_t y_stride,
                                                   const uint32_t *zws, uint32_t z_stride, uint64_t n_blocks,
                                                   uint32_t m, OutStream out) {
    extern __shared__ uint4 rs4[];  // STAGED: 32 rows of rw4 uint4 (last one zero)
    const uint32_t *rs = reinterpret_cast<const uint32_t *>(rs4);
    const uint64_t b0 = (uint64_t)blockIdx.x * 32;
    const uint32_t nb = (uint32_t)min((uint64_t)32, n_blocks - b0);
    const uint32_t rw4 = ((m + 31) / 32 + 3) / 4 + 1, rwords = 4 * rw4;
    if (STAGED) {
        for (uint32_t i = threadIdx.x; i < nb * rw4; i += blockDim.x) {
            const uint32_t bl = i / rw4, q = i - bl * rw4;
            const uint64_t b = b0 + bl;
            rs4[i] = q + 1 < rw4 ? node_word4(root, reinterpret_cast<const uint4 *>(yws + b * y_stride),
                                              reinterpret_cast<const uint4 *>(zws + b * z_stride), q)
                                 : make_uint4(0, 0, 0, 0);
        }
        __syncthreads();
    }
    auto rword = [&](uint32_t bl, uint32_t q) -> uint32_t {  // word q of block b0+bl's root row
        if (STAGED) return rs[bl * rwords + q];
        const uint64_t b = b0 + bl;
        const uint4 v = node_word4(root, reinterpret_cast<const uint4 *>(yws + b * y_stride),
                                   reinterpret_cast<const uint4 *>(zws + b * z_stride), q / 4);
        const uint32_t r = q & 3;
        return r == 0 ? v.x : r == 1 ? v.y : r == 2 ? v.z : v.w;
    };
    const uint32_t gbits = nb * m, gwords = (gbits + 31) / 32;
    for (uint32_t w = threadIdx.x; w < gwords; w += blockDim.x) {
        const uint32_t G = w * 32, end = min(G + 32, gbits);
        uint32_t b = G / m, i = G - b * m, pos = G, word = 0;
        while (pos < end) {
            const uint32_t len = min(m - i, end - pos);  // 1..32 bits of block b
            const uint32_t q = i >> 5, s = i & 31;
            const uint32_t w0 = rword(b, q);
            const uint32_t bits = s ? ((w0 << s) | (rword(b, q + 1) >> (32 - s))) : w0;  // rows i.. at the MSB
            word |= (bits >> (32 - len)) << (32 - len - (pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, b0 * m / 32 + w, word, true);
    }
}

// Fused tree combine + pack for 32 blocks whose internal node rows and root
// rows fit in shared memory: leaf parities are read from Y (L2), every combine
// level stays in shared memory, then the key words [c*m, (c+1)*m) of the
// group are written (one writer each, no pre-zeroing).
__global__ void __launch_bounds__(512) tree_pack_kernel(const uint32_t *inner, const uint32_t *unit_node,
                                                        const uint4 *levels, uint32_t n_levels,
                                                        const uint32_t *yws, uint32_t y_stride, uint32_t z_stride,
                                                        uint64_t n_blocks, uint32_t m, OutStream out) {
    extern __shared__ uint4 sm4[];
    const uint64_t b0 = (uint64_t)blockIdx.x * 32;
    const uint32_t nb = (uint32_t)min((uint64_t)32, n_blocks - b0);
    const uint32_t zs4 = z_stride / 4, rw4 = levels[n_levels - 1].z, rwords = 4 * rw4;
    uint4 *Zs = sm4, *Rs = Zs + 32 * zs4;
    const uint4 *Ys = reinterpret_cast<const uint4 *>(yws + b0 * y_stride);
    for (uint32_t l = 0; l < n_levels; ++l) {
        if (l) __syncthreads();
        combine_level<8>(inner, unit_node, levels[l], nb, Ys, y_stride / 4, Zs, zs4, l + 1 == n_levels ? Rs : nullptr,
                         rw4);
    }
    __syncthreads();
    const uint32_t *rs = reinterpret_cast<const uint32_t *>(Rs);
    const uint32_t gbits = nb * m, gwords = (gbits + 31) / 32;
    for (uint32_t w = threadIdx.x; w < gwords; w += blockDim.x) {
        const uint32_t G = w * 32, end = min(G + 32, gbits);
        uint32_t b = G / m, i = G - b * m, pos = G, word = 0;
        while (pos < end) {
            const uint32_t len = min(m - i, end - pos);  // 1..32 bits of block b
            const uint32_t *row = rs + b * rwords;
            const uint32_t q = i >> 5, s = i & 31;
            const uint32_t bits = s ? ((row[q] << s) | (row[q + 1] >> (32 - s))) : row[q];
            word |= (bits >> (32 - len)) << (32 - len - (pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, b0 * m / 32 + w, word, true);
    }
}

// Combine + pack for bpc blocks whose leaf parities fit in shared memory
// (bpc m % 32 == 0, so the group's key is whole output words): the bpc Y rows
// (contiguous in the workspace) are copied in with coalesced 16-byte loads,
// each root word is the XOR of its leaf words (the flattened tree: the CSR of
// qrng_debug_karatsuba_plan, also staged in shared memory), then the key words
// [c bpc m/32, (c+1) bpc m/32) of the group are written (one writer each).
__global__ void __launch_bounds__(QRNG_CSR_THREADS) csr_pack_kernel(const uint32_t *csr, uint32_t csr_words, const uint32_t *yws,
                                                       uint32_t y_stride, uint64_t n_blocks, uint32_t m, uint32_t bpc,
                                                       OutStream out) {
    extern __shared__ uint4 sm4[];
    const uint64_t b0 = (uint64_t)blockIdx.x * bpc;
    const uint32_t nb = (uint32_t)min((uint64_t)bpc, n_blocks - b0);
    const uint32_t ywords = (m + 31) / 32, rwords = ywords + 1;
    uint32_t *Ys = reinterpret_cast<uint32_t *>(sm4);
    uint32_t *Rs = Ys + bpc * y_stride;
    uint32_t *Cs = Rs + bpc * rwords;
    const uint4 *src = reinterpret_cast<const uint4 *>(yws + b0 * y_stride);
    {  // coalesced copy with 8 independent 16-byte loads in flight per thread
        const uint32_t n4 = nb * (y_stride / 4);
        for (uint32_t base = threadIdx.x; base < n4; base += 8 * blockDim.x) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (base + u * blockDim.x < n4) v[u] = __ldg(src + base + u * blockDim.x);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (base + u * blockDim.x < n4) sm4[base + u * blockDim.x] = v[u];
        }
    }
    for (uint32_t i = threadIdx.x; i < csr_words; i += blockDim.x) Cs[i] = __ldg(csr + i);
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < nb * rwords; idx += blockDim.x) {
        const uint32_t bl = idx / rwords, j = idx - bl * rwords;
        uint32_t v = 0;
        if (j < ywords) {
            const uint32_t *yr = Ys + bl * y_stride;
            for (uint32_t e = 0, c = Cs[j]; e < c; ++e) v ^= yr[Cs[ywords + e * ywords + j]];
        }
        Rs[idx] = v;
    }
    __syncthreads();
    const uint32_t gbits = nb * m, gwords = (gbits + 31) / 32;
    for (uint32_t w = threadIdx.x; w < gwords; w += blockDim.x) {
        const uint32_t G = w * 32, end = min(G + 32, gbits);
        uint32_t b = G / m, i = G - b * m, pos = G, word = 0;
        while (pos < end) {
            const uint32_t len = min(m - i, end - pos);  // 1..32 bits of block b
            const uint32_t *row = Rs + b * rwords;
            const uint32_t q = i >> 5, s = i & 31;
            const uint32_t bits = s ? ((row[q] << s) | (row[q + 1] >> (32 - s))) : row[q];
            word |= (bits >> (32 - len)) << (32 - len - (pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, b0 * m / 32 + w, word, true);
    }
}

// Streaming form of the staged combine + pack: a persistent grid, each CTA
// walks groups of bpc blocks; a group's leaf-parity rows are one contiguous
// range of the workspace and arrive by a single TMA bulk copy
// (cp.async.bulk, mbarrier completion) into one of two shared buffers, so the
// next group's rows are in flight while this group is combined and packed.
__device__ __forceinline__ uint32_t ksmem(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// 32-bit shared-window accesses from precomputed addresses (the generic
// pointer form re-derived the window base for every load: ~6 instructions per
// combined word instead of an add, a load and a fused and-xor)
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// KU: CSR entries per key word handled branch-free (the table's maximum when
// it is <= 8; padded entries are masked); entries past KU take a loop.
// FUSED (m >= 64): combine and pack in one pass -- lane l of a warp combines
// key word 31w + l of a block and takes word + 1 from lane l + 1 by a shuffle
// (lane 31 only feeds lane 30), so the shifted output word is formed in
// registers; only each block's word 0 (the low part of the word straddling
// into it) goes through shared memory.
#ifndef QRNG_CSR_NBUF
#define QRNG_CSR_NBUF 2  // leaf-parity group buffers in flight per CTA
#endif
template <int KU, bool FUSED>
__global__ void __launch_bounds__(QRNG_CSR_THREADS) csr_stream_pack_kernel(const uint32_t *csr, uint32_t csr_words,
                                                                           const uint32_t *yws, uint32_t y_stride,
                                                                           uint64_t n_blocks, uint32_t m, uint32_t bpc,
                                                                           uint64_t m_magic, OutStream out) {
    extern __shared__ uint4 sm4[];
    const uint32_t ywords = (m + 31) / 32, rwords = ywords + 1;
    const uint32_t ybuf_words = bpc * y_stride;
    uint32_t *Y0 = reinterpret_cast<uint32_t *>(sm4);
    uint32_t *Rs = Y0 + QRNG_CSR_NBUF * ybuf_words;
    // fused form: Rs holds only each block's word 0 (the straddle heads)
    const uint32_t rs_words = (FUSED && m >= 64) ? bpc : bpc * rwords;
    uint32_t *Cs = Rs + rs_words;
    const uint32_t bar_off = (QRNG_CSR_NBUF * ybuf_words + rs_words + csr_words + 1) & ~1u;  // 8-byte aligned
    uint64_t *bar = reinterpret_cast<uint64_t *>(Y0 + bar_off);
    const uint64_t n_groups = (n_blocks + bpc - 1) / bpc;
    auto issue = [&](uint64_t g, uint32_t buf) {  // one thread
        const uint32_t nb = (uint32_t)min((uint64_t)bpc, n_blocks - g * bpc);
        const uint32_t bytes = nb * y_stride * 4;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ksmem(bar + buf)), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ksmem(Y0 + buf * ybuf_words)),
            "l"(yws + g * bpc * y_stride), "r"(bytes), "r"(ksmem(bar + buf))
            : "memory");
    };
    for (uint32_t i = threadIdx.x; i < csr_words; i += blockDim.x) Cs[i] = __ldg(csr + i);
    pdl_wait();  // the leaf parities (previous kernel) are complete
    if (threadIdx.x == 0) {
        for (int i = 0; i < QRNG_CSR_NBUF; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ksmem(bar + i)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (uint32_t i = 0; i < QRNG_CSR_NBUF; ++i)
            if (blockIdx.x + (uint64_t)i * gridDim.x < n_groups) issue(blockIdx.x + (uint64_t)i * gridDim.x, i);
    }
    __syncthreads();
    uint32_t k = 0;
    for (uint64_t g = blockIdx.x; g < n_groups; g += gridDim.x, ++k) {
        const uint32_t buf = k % QRNG_CSR_NBUF, ph = (k / QRNG_CSR_NBUF) & 1;
        {
            uint32_t done = 0;
            do {
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done) : "r"(ksmem(bar + buf)), "r"(ph) : "memory");
            } while (!done);
        }
        const uint64_t b0 = g * bpc;
        const uint32_t nb = (uint32_t)min((uint64_t)bpc, n_blocks - b0);
        const uint32_t *Ys = Y0 + buf * ybuf_words;
        const uint32_t ys_sa = ksmem(Ys), rs_sa = ksmem(Rs);
        if (FUSED && m >= 64) {
            const uint32_t c0 = Cs[0];
            for (uint32_t bl = threadIdx.x; bl < nb; bl += blockDim.x) {  // heads: key word 0 of each block
                const uint32_t row = ys_sa + bl * y_stride * 4;
                uint32_t v = 0;
                for (uint32_t e = 0; e < c0; ++e) v ^= lds32(row + 4 * Cs[ywords + e * ywords]);
                sts32(rs_sa + bl * 4, v);
            }
            __syncthreads();
            const uint32_t lane = threadIdx.x & 31, wpb = ywords + 1;  // >= words starting in one block
            const uint32_t tps = 32 * ((wpb + 30) / 31);                // threads per block set (whole warps)
            const uint32_t sets = max(1u, blockDim.x / tps);
            const uint64_t wbase = b0 * m / 32;
            for (uint32_t u = threadIdx.x; u < sets * tps; u += blockDim.x) {  // warp-uniform bounds
                const uint32_t set = u / tps, kk = 31 * ((u - set * tps) >> 5) + lane;
                const uint32_t c = kk < ywords ? Cs[kk] : 0u;
                uint32_t off[KU], msk[KU];
#pragma unroll
                for (int e = 0; e < KU; ++e) {
                    off[e] = (uint32_t)e < c ? 4 * Cs[ywords + e * ywords + kk] : 0u;
                    msk[e] = (uint32_t)e < c ? ~0u : 0u;
                }
                const uint32_t rstep = sets * y_stride * 4, sstep = sets * m, kk32 = 32 * kk;
                const bool active = lane != 31 && kk < wpb;  // lane 31 only feeds lane 30
                // whole group inside the buffer's full words: plain stores, no per-word check
                const bool fast = (b0 * m + (uint64_t)nb * m + 31) / 32 <= out.full_words;
                uint32_t *const ow = out.words + wbase;
                uint32_t row = ys_sa + set * y_stride * 4, s0 = set * m;  // s0: first bit of block bl in the group
                for (uint32_t bl = set; bl < nb; bl += sets, row += rstep, s0 += sstep) {
                    uint32_t r0 = 0;
#pragma unroll
                    for (int e = 0; e < KU; ++e) r0 ^= lds32(row + off[e]) & msk[e];
                    for (uint32_t e = KU; e < c; ++e) r0 ^= lds32(row + 4 * Cs[ywords + e * ywords + kk]);
                    const uint32_t r1 = __shfl_down_sync(0xFFFFFFFFu, r0, 1);  // key word kk + 1
                    if (!active) continue;
                    // the kk-th output word starting inside block bl begins at key bit i0
                    const uint32_t sh = (0u - s0) & 31u, i0 = sh + kk32;
                    if (i0 >= m) continue;  // block bl has fewer words (other blocks may not)
                    uint32_t word = __funnelshift_l(r1, r0, sh);
                    if (i0 + 32 > m) {  // tail of block bl, then the head of block bl + 1
                        const uint32_t len1 = m - i0;
                        word &= ~(0xFFFFFFFFu >> len1);
                        if (bl + 1 < nb) word |= lds32(rs_sa + (bl + 1) * 4) >> len1;
                    }
                    const uint32_t W = ((s0 + 31) >> 5) + kk;
                    if (fast) ow[W] = bswap32(word);
                    else emit_word(out, wbase + W, word, true);
                }
            }
            __syncthreads();  // this buffer's rows and the heads are no longer read
            if (threadIdx.x == 0 && g + QRNG_CSR_NBUF * (uint64_t)gridDim.x < n_groups) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(g + QRNG_CSR_NBUF * (uint64_t)gridDim.x, buf);
            }
            continue;
        }
        {
            // thread (set, j): key word j of blocks set, set + sets, ...; the word's
            // CSR entries are read once and reused for every block of the group
            const uint32_t sets = max(1u, blockDim.x / rwords);
            for (uint32_t u = threadIdx.x; u < sets * rwords; u += blockDim.x) {
                const uint32_t set = u / rwords, j = u - set * rwords;
                const uint32_t rstep = sets * y_stride * 4, dstep = sets * rwords * 4;
                uint32_t row = ys_sa + set * y_stride * 4, dst = rs_sa + (set * rwords + j) * 4;
                if (j < ywords) {
                    const uint32_t c = Cs[j];
                    uint32_t off[KU], msk[KU];
#pragma unroll
                    for (int e = 0; e < KU; ++e) {
                        off[e] = (uint32_t)e < c ? 4 * Cs[ywords + e * ywords + j] : 0u;
                        msk[e] = (uint32_t)e < c ? ~0u : 0u;
                    }
                    for (uint32_t bl = set; bl < nb; bl += sets, row += rstep, dst += dstep) {
                        uint32_t v = 0;
#pragma unroll
                        for (int e = 0; e < KU; ++e) v ^= lds32(row + off[e]) & msk[e];
                        for (uint32_t e = KU; e < c; ++e) v ^= lds32(row + 4 * Cs[ywords + e * ywords + j]);
                        sts32(dst, v);
                    }
                } else {
                    for (uint32_t bl = set; bl < nb; bl += sets, dst += dstep) sts32(dst, 0);
                }
            }
        }
        __syncthreads();  // Rs complete; this buffer's rows are no longer read
        if (threadIdx.x == 0 && g + QRNG_CSR_NBUF * (uint64_t)gridDim.x < n_groups) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(g + QRNG_CSR_NBUF * (uint64_t)gridDim.x, buf);
        }
        const uint32_t gbits = nb * m, gwords = (gbits + 31) / 32;
        const uint64_t wbase = b0 * m / 32;
        if (m >= 64) {
            // per block row: the words inside block bl are its key row shifted by
            // a constant (bl m mod 32); the one word straddling bl and bl + 1 is
            // assembled by the thread that owns it.  No division per word.
            const uint32_t wpb = (m + 31) / 32 + 1;  // >= words starting in one block
            const uint32_t sets = max(1u, blockDim.x / wpb);
            for (uint32_t u = threadIdx.x; u < sets * wpb; u += blockDim.x) {
                const uint32_t set = u / wpb, k = u - set * wpb;
                for (uint32_t bl = set; bl < nb; bl += sets) {
                    const uint32_t s0 = bl * m, s1 = s0 + m;  // bit range of block bl in the group
                    const uint32_t W = (s0 + 31) / 32 + k;    // k-th word starting inside block bl
                    if (32 * W >= s1) continue;  // block bl has fewer words (other blocks may not)
                    const uint32_t i0 = 32 * W - s0, sft = i0 & 31;
                    const uint32_t ra = rs_sa + (bl * rwords + (i0 >> 5)) * 4;
                    // row[q + 1] exists (rwords = ywords + 1, the pad word is 0)
                    uint32_t word = __funnelshift_l(lds32(ra + 4), lds32(ra), sft);
                    if (32 * W + 32 > s1) {
                        // tail of block bl (len1 bits), then the head of block bl + 1
                        const uint32_t len1 = s1 - 32 * W;
                        word &= ~(0xFFFFFFFFu >> len1);
                        if (bl + 1 < nb) word |= lds32(rs_sa + (bl + 1) * rwords * 4) >> len1;
                    }
                    emit_word(out, wbase + W, word, true);
                }
            }
            __syncthreads();
            continue;
        }
        for (uint32_t w = threadIdx.x; w < gwords; w += blockDim.x) {
            const uint32_t G = w * 32, end = min(G + 32, gbits);
            uint32_t b = m_magic ? (uint32_t)__umul64hi((uint64_t)G, m_magic) : G;  // G / m
            uint32_t i = G - b * m, pos = G, word = 0;
            while (pos < end) {
                const uint32_t len = min(m - i, end - pos);  // 1..32 bits of block b
                const uint32_t *row = Rs + b * rwords;
                const uint32_t q = i >> 5, sft = i & 31;
                const uint32_t bits = sft ? ((row[q] << sft) | (row[q + 1] >> (32 - sft))) : row[q];
                word |= (bits >> (32 - len)) << (32 - len - (pos - G));
                pos += len;
                ++b;
                i = 0;
            }
            emit_word(out, wbase + w, word, true);
        }
        __syncthreads();  // Rs is rewritten by the next group
    }
}

// Gather form of the same combine + pack: one thread per output word, no
// shared memory.  Output word w covers key bits [32w, 32w + 32): at most two
// blocks; for each, the (one or two) key-row words the bits come from are
// XORed straight from the leaf-parity rows in L2 as the CSR lists them
// (neighbouring threads read neighbouring words, so the gathers coalesce).
// Every output word has exactly one writer.
__device__ __forceinline__ uint32_t csr_word(const uint32_t *__restrict__ csr, uint32_t ywords,
                                             const uint32_t *__restrict__ yr, uint32_t q) {
    // the first 8 terms with independent (predicated) loads, so the gathers of
    // one word are in flight together; deeper trees loop over the rest
    const uint32_t c = __ldg(csr + q);
    uint32_t idx[8];
#pragma unroll
    for (uint32_t e = 0; e < 8; ++e) idx[e] = e < c ? __ldg(csr + ywords + e * ywords + q) : 0u;
    uint32_t v = 0;
#pragma unroll
    for (uint32_t e = 0; e < 8; ++e)
        if (e < c) v ^= __ldg(yr + idx[e]);
    for (uint32_t e = 8; e < c; ++e) v ^= __ldg(yr + __ldg(csr + ywords + e * ywords + q));
    return v;
}
__global__ void __launch_bounds__(256) csr_gather_pack_kernel(const uint32_t *__restrict__ csr,
                                                              const uint32_t *__restrict__ yws, uint32_t y_stride,
                                                              uint64_t n_blocks, uint32_t m, uint64_t m_magic,
                                                              OutStream out) {
    const uint32_t ywords = (m + 31) / 32;
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
            const uint32_t *yr = yws + b * y_stride;
            const uint32_t q = i >> 5, sft = i & 31;
            const uint32_t c0 = csr_word(csr, ywords, yr, q);
            const uint32_t c1 = (sft && q + 1 < ywords) ? csr_word(csr, ywords, yr, q + 1) : 0u;
            const uint32_t bits = sft ? ((c0 << sft) | (c1 >> (32 - sft))) : c0;
            word |= (bits >> (32 - len)) << (32 - len - (uint32_t)(pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, w, word, true);
    }
}

// Long key rows, two phases.  (1) every key word once: Z[b][j] = XOR of its
// CSR entries (one thread per (block, word), consecutive threads on
// consecutive words: coalesced gathers); (2) the packed stream from the Z rows
// (one thread per output word, <= 4 Z words each, L2 hits).  The one-phase
// gather form forms most output words from two key words (m % 32 != 0), i.e.
// computes every key word twice.
__global__ void __launch_bounds__(256) csr_key_kernel(const uint32_t *__restrict__ csr, const uint32_t *__restrict__ yws,
                                                      uint32_t y_stride, uint64_t n_blocks, uint32_t ywords,
                                                      uint32_t *__restrict__ zws, uint32_t z_stride) {
    const uint64_t total = n_blocks * ywords;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = t / ywords;
        const uint32_t j = (uint32_t)(t - b * ywords);
        zws[b * z_stride + j] = csr_word(csr, ywords, yws + b * y_stride, j);
    }
}

// Phase (1), staged: one CTA per block copies the block's whole leaf-parity
// row (y_stride words, coalesced 16-byte loads at streaming bandwidth) into
// shared memory and forms every key word from there; the CSR table (shared by
// all blocks) is read through L1 / L2.  The gather form above is bound by the
// latency of its dependent index -> parity loads from DRAM.
__global__ void __launch_bounds__(512) csr_stage_key_kernel(const uint32_t *__restrict__ csr,
                                                            const uint32_t *__restrict__ yws, uint32_t y_stride,
                                                            uint32_t ywords, uint32_t *__restrict__ zws,
                                                            uint32_t z_stride) {
    extern __shared__ uint4 ys4[];
    const uint32_t *ys = reinterpret_cast<const uint32_t *>(ys4);
    const uint64_t b = blockIdx.x;
    const uint4 *src = reinterpret_cast<const uint4 *>(yws + b * y_stride);  // y_stride % 4 == 0
    for (uint32_t i = threadIdx.x; i < y_stride / 4; i += blockDim.x) ys4[i] = __ldcs(src + i);
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < ywords; j += blockDim.x) {
        const uint32_t c = __ldg(csr + j);
        uint32_t v = 0;
        for (uint32_t e = 0; e < c; ++e) v ^= ys[__ldg(csr + ywords + e * ywords + j)];
        zws[b * z_stride + j] = v;
    }
}

// Phase (1) from runs, for rows too long to stage: one CTA per block, the key
// row Z in shared memory; batch by batch (runs of a batch write disjoint key
// words) every warp XORs whole runs Y[src, src + len) into Z[dst, dst + len) --
// consecutive lanes read and write consecutive words, no per-word index, no
// atomics -- with one barrier per batch; the leaf-parity row is read through
// L1 / L2.  (A staged variant that first copies the row into shared memory lost
// to csr_stage_key_kernel; see the dispatch.)
__global__ void __launch_bounds__(512) csr_run_key_kernel(const uint4 *__restrict__ runs,
                                                          const uint32_t *__restrict__ run_ptr, uint32_t n_batches,
                                                          const uint32_t *__restrict__ yws, uint32_t y_stride,
                                                          uint32_t ywords, uint32_t *__restrict__ zws,
                                                          uint32_t z_stride) {
    extern __shared__ uint4 sm4[];
    const uint32_t zw4 = (ywords + 3) / 4;
    uint32_t *Z = reinterpret_cast<uint32_t *>(sm4);
    const uint64_t b = blockIdx.x;
    const uint32_t *yrow = yws + b * y_stride;
    for (uint32_t i = threadIdx.x; i < zw4; i += blockDim.x) sm4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    for (uint32_t bt = 0; bt < n_batches; ++bt) {
        const uint32_t r1 = __ldg(run_ptr + bt + 1);
        for (uint32_t r = __ldg(run_ptr + bt) + warp; r < r1; r += nwarps) {
            const uint4 R = __ldg(runs + r);
            for (uint32_t i = lane; i < R.z; i += 32) Z[R.x + i] ^= __ldg(yrow + R.y + i);
        }
        __syncthreads();
    }
    for (uint32_t j = threadIdx.x; j < ywords; j += blockDim.x) zws[b * z_stride + j] = Z[j];
}

__global__ void __launch_bounds__(256) zpack_kernel(const uint32_t *__restrict__ zws, uint32_t z_stride,
                                                    uint64_t n_blocks, uint32_t m, uint64_t m_magic, OutStream out) {
    const uint32_t ywords = (m + 31) / 32;
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
            const uint32_t *zr = zws + b * z_stride;
            const uint32_t q = i >> 5, sft = i & 31;
            const uint32_t c0 = __ldg(zr + q);
            const uint32_t c1 = (sft && q + 1 < ywords) ? __ldg(zr + q + 1) : 0u;
            const uint32_t bits = sft ? ((c0 << sft) | (c1 >> (32 - sft))) : c0;
            word |= (bits >> (32 - len)) << (32 - len - (uint32_t)(pos - G));
            pos += len;
            ++b;
            i = 0;
        }
        emit_word(out, w, word, true);
    }
}

// ---- host entry points -----------------------------------------------------
// two block-range chunks on two streams per extraction (measured slower; see extract())
constexpr bool kTwoChunks = false;

qrng_status plan_init(Plan &pl, uint64_t n, uint64_t m, int max_depth, const uint8_t *d_seed, cudaStream_t s,
                      bool defer_seeds) {
    std::shared_ptr<const Tables> t;
    qrng_status st = get_tables(n, m, max_depth, &t);
    if (st != QRNG_OK) return st;
    pl.tab = t;
    const HostTables &H = t->host;
    QRNG_CUDA_TRY(cudaMallocAsync(&pl.seeds, (size_t)H.seed_total * 4, s));
    if (defer_seeds && !H.qbufs.empty() && !kTwoChunks) {  // formed inside the first extraction's Q-buffer launch
        pl.pending_seed = d_seed;
        pl.seed_L = n + m - 1;
        return QRNG_OK;
    }
    uint32_t maxw = 0;
    for (const auto &g : t->hleaves) maxw = std::max(maxw, g.seed_n);
    count_launch();
    leaf_seed_kernel<<<dim3((maxw + 127) / 128, (unsigned)t->hleaves.size()), 128, 0, s>>>(t->leaves, t->terms, d_seed,
                                                                                           n + m - 1, pl.seeds);
    QRNG_CUDA_TRY(cudaGetLastError());
    return QRNG_OK;
}

void plan_free(Plan &pl) {
    if (pl.seeds) cudaFree(pl.seeds);
    pl = Plan{};
}

static qrng_status extract_chunk(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                                 const OutStream &out, cudaStream_t s);

// Optional (off): batches of >= 2048 blocks as two block-range chunks on the
// caller's stream and the side stream, so the Q buffers of one chunk and the
// combine/pack of the other overlap the leaf GEMMs.  Chunk boundaries are
// multiples of 32 blocks, so each chunk's key starts on a 32-bit word.
// Measured +1.6% at config 2 (324.7 vs 319.7 Gbit/s), but the overlapping GEMM
// launches blur the per-kernel roofline timing and the host-buffer pipeline
// (two compute streams of its own) then shares one side stream, so it is off.
qrng_status extract(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                    const OutStream &out, cudaStream_t s) {
    if (!kTwoChunks || n_blocks < 2048) return extract_chunk(pl, d_raw, n_blocks, n, m, out, s);
    cudaStream_t s2;
    cudaEvent_t fork, join;
    qrng_status st = side_stream(&s2, &fork, &join);
    if (st != QRNG_OK) return st;
    QRNG_CUDA_TRY(cudaEventRecord(fork, s));
    QRNG_CUDA_TRY(cudaStreamWaitEvent(s2, fork, 0));
    const uint64_t b1 = (n_blocks / 2 + 31) / 32 * 32;  // first block of chunk 2
    OutStream o1 = out, o2 = out;
    o1.total_bits = b1 * m;
    o1.full_words = std::min<uint64_t>(out.full_words, b1 * m / 32);
    o2.words = out.words + b1 * m / 32;
    o2.total_bits = (n_blocks - b1) * m;
    o2.full_words = out.full_words - b1 * m / 32;
    st = extract_chunk(pl, d_raw, b1, n, m, o1, s);
    if (st == QRNG_OK) st = extract_chunk(pl, d_raw + b1 * n / 8, n_blocks - b1, n, m, o2, s2);
    cudaEventRecord(join, s2);
    cudaStreamWaitEvent(s, join, 0);
    return st;
}

void describe(const Plan &pl, int *depth, int *n_leaves, uint64_t *macs_per_block, uint32_t *x_words, uint32_t *y_words) {
    if (!pl.tab) { *depth = 0; *n_leaves = 0; *macs_per_block = 0; *x_words = *y_words = 0; return; }
    *depth = pl.tab->host.depth;
    *n_leaves = (int)pl.tab->host.leaves.size();
    *macs_per_block = pl.tab->host.macs;
    *x_words = pl.tab->host.x_stride;
    *y_words = pl.tab->host.y_stride;
}

static qrng_status extract_chunk(const Plan &pl, const uint8_t *d_raw, uint64_t n_blocks, uint64_t n, uint64_t m,
                                 const OutStream &out, cudaStream_t s) {
    const Tables *t = pl.tab.get();
    const HostTables &H = t->host;
    uint32_t *xws = nullptr, *yws = nullptr;
    if (H.x_stride) QRNG_CUDA_TRY(cudaMallocAsync(&xws, (size_t)n_blocks * H.x_stride * 4, s));
    QRNG_CUDA_TRY(cudaMallocAsync(&yws, (size_t)n_blocks * H.y_stride * 4, s));
    qrng_status st = QRNG_OK;
    if (!H.qbufs.empty()) {  // Q buffers, generation by generation, bpc blocks per CTA
#ifndef QRNG_QBUF_U
#define QRNG_QBUF_U 4      // 16-byte units in flight per thread
#endif
#ifndef QRNG_QBUF_DIV
#define QRNG_QBUF_DIV 296  // target CTA count (blocks per CTA = n_blocks / this, at most 32)
#endif
        // deeper trees (more generations, longer X rows) want more, smaller CTAs:
        // measured (tools/qbuf_ab.sh) 296 CTAs best at depth 2, 1184 at depth 6
        const uint64_t div = (uint64_t)QRNG_QBUF_DIV << (H.depth >= 6 ? 2 : H.depth >= 4 ? 1 : 0);
#ifndef QRNG_QBUF_MAXBPC
#define QRNG_QBUF_MAXBPC 32
#endif
        const uint32_t bpc = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(QRNG_QBUF_MAXBPC, n_blocks / div));
        KernelTimer tq(s, true, 1);
        SeedJob sj{};
        sj.q_ctas = (uint32_t)((n_blocks + bpc - 1) / bpc);
        uint32_t seed_ctas = 0;
        if (pl.pending_seed) {
            sj.leaves = t->leaves;
            sj.terms = t->terms;
            sj.seed = pl.pending_seed;
            sj.L = pl.seed_L;
            sj.seeds = pl.seeds;
            sj.n_leaves = (uint32_t)t->hleaves.size();
            seed_ctas = std::min<uint32_t>(sj.n_leaves, 64);
        }
        // one-pass slice form where the tree allows it (QRNG_QSLICE=0: the generation kernel, A/B)
        static const bool qslice_on = [] {
            const char *e = getenv("QRNG_QSLICE");
            return !(e && *e && atoi(e) == 0);
        }();
        if (qslice_on && t->qs_ns) {
            static_assert(sizeof(QSlice) == sizeof(t->qs), "QSlice host/device layout");
            QSlice qs;
            memcpy(&qs, &t->qs, sizeof(qs));
            const uint64_t items = n_blocks << qs.lsu;
            sj.q_ctas = (uint32_t)((items + 255) / 256);
            const uint4 *r4 = reinterpret_cast<const uint4 *>(d_raw);
            uint4 *x4 = reinterpret_cast<uint4 *>(xws);
            const dim3 grid(sj.q_ctas + seed_ctas);
            switch (t->qs_ns) {
                case 2: qslice_kernel<2><<<grid, 256, 0, s>>>(qs, r4, n_blocks, x4, H.x_stride, sj); break;
                case 4: qslice_kernel<4><<<grid, 256, 0, s>>>(qs, r4, n_blocks, x4, H.x_stride, sj); break;
                case 8: qslice_kernel<8><<<grid, 256, 0, s>>>(qs, r4, n_blocks, x4, H.x_stride, sj); break;
                default: qslice_kernel<16><<<grid, 256, 0, s>>>(qs, r4, n_blocks, x4, H.x_stride, sj); break;
            }
        } else {
            qbuf_kernel<QRNG_QBUF_U><<<sj.q_ctas + seed_ctas, 512, 0, s>>>(
                t->qbufs, t->qgen_dev, (uint32_t)t->qgen.size() - 1, reinterpret_cast<const uint4 *>(d_raw), n_blocks,
                (uint32_t)n, reinterpret_cast<uint4 *>(xws), H.x_stride, bpc, sj);
        }
        tq.stop();
        if (cudaGetLastError() != cudaSuccess) { set_error("qbuf_kernel launch failed"); st = QRNG_E_CUDA; }
    }
    if (st == QRNG_OK)
        st = gemm::extract_grouped(t->leaves, (uint32_t)t->hleaves.size(), H.total_npairs, pl.seeds, d_raw, n_blocks,
                                   n, xws, H.x_stride, yws, H.y_stride, t->max_leaf_w, s);
    const uint32_t rw4 = (uint32_t)(((m + 31) / 32 + 3) / 4 + 1);
    const size_t fused_smem = (size_t)32 * (H.z_stride + 4 * rw4) * 4;
    const uint32_t ywords = (uint32_t)((m + 31) / 32), csr_words = t->csr_words;
    // blocks per CTA: the smallest count whose keys are whole 32-bit words
    // (32 / gcd(m, 32)), doubled while the staged rows stay small
    uint32_t bpc = 32;
    while (bpc > 1 && (bpc / 2) * m % 32 == 0) bpc /= 2;
    auto csr_bytes = [&](uint32_t b) { return ((size_t)b * (H.y_stride + ywords + 1) + csr_words) * 4; };
    while (bpc < 8 && csr_bytes(2 * bpc) <= 72 * 1024) bpc *= 2;
    const size_t csr_smem = csr_bytes(bpc);
    uint32_t *zws = nullptr;
    // gather form for long key rows (measured: config 3, 1434 words, 146.2 ->
    // 149.7 Gbit/s); the staged form for short ones (config 2, 180 words: 477
    // vs 459 -- the gather form is load-instruction bound there)
    static const int gather_env = [] {
        const char *e = getenv("QRNG_CSR_GATHER");
        return e ? atoi(e) : -1;
    }();
    // (round 2: with the two-phase staged form the threshold is 512 words --
    // 2^15, 717 words: 278 -> 310 Gbit/s; 2^14, 359 words: the staged stream
    // form stays faster, 534 vs 489; tools/csr_key_ab.sh, QRNG_CSR_GATHER)
    const bool gather = gather_env >= 0 ? gather_env != 0 : ywords >= 512;
    static const bool stream_form = [] {
        const char *e = getenv("QRNG_CSR_STREAM");
        return e ? atoi(e) != 0 : true;
    }();
    static const bool fused = [] {  // QRNG_CSR_FUSED=0: separate combine and pack phases
        const char *e = getenv("QRNG_CSR_FUSED");
        return e ? atoi(e) != 0 : true;
    }();
    // (the fused form stages only each block's word 0 of the key rows)
    const size_t rs_words = (fused && m >= 64) ? (size_t)bpc : (size_t)bpc * (ywords + 1);
    const size_t stream_smem = (((size_t)QRNG_CSR_NBUF * bpc * H.y_stride + rs_words + csr_words + 1) & ~(size_t)1) * 4 + 8 * QRNG_CSR_NBUF;
    static const bool zpack = [] {  // QRNG_CSR_ZPACK=0: the one-phase gather form (A/B)
        const char *e = getenv("QRNG_CSR_ZPACK");
        return e ? atoi(e) != 0 : true;
    }();
    if (st == QRNG_OK && gather && zpack) {
        const uint64_t gwords = ((uint64_t)n_blocks * m + 31) / 32;
        const uint64_t m_magic = m > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / m) + 1 : 0;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint32_t z_stride = (ywords + 3) & ~3u;
        uint32_t *kz = nullptr;
        cudaError_t e = cudaMallocAsync(&kz, (size_t)n_blocks * z_stride * 4, s);
        if (e != cudaSuccess) { set_error("cudaMallocAsync: %s", cudaGetErrorString(e)); st = QRNG_E_NOMEM; }
        if (st == QRNG_OK) {
            const uint64_t items = (uint64_t)n_blocks * ywords, cap = (uint64_t)sms * 16;
            const uint64_t w1 = (items + 255) / 256, w2 = (gwords + 255) / 256;
            static const bool staged = [] {  // QRNG_CSR_STAGE=0: the gather key kernel (A/B)
                const char *e = getenv("QRNG_CSR_STAGE");
                return e ? atoi(e) != 0 : true;
            }();
            const size_t ysmem = (size_t)H.y_stride * 4;
            static const bool use_runs = [] {  // QRNG_CSR_RUNS=0: the CSR key kernels (A/B)
                const char *e = getenv("QRNG_CSR_RUNS");
                return !(e && *e && atoi(e) == 0);
            }();
            const size_t zsmem = (size_t)((ywords + 3) / 4) * 16;
            KernelTimer tc(s, true, 1);
            // rows that fit in shared memory: the staged CSR kernel (a runs form
            // with the row staged in shared memory measured slower: config 3 218 -> 195,
            // 2^17 140 -> 106 Gbit/s -- a barrier per batch of ~2 runs per warp);
            // longer rows: the runs kernel reading the row through L1 / L2
            // instead of the CSR gather (2^18 77.4 -> 83.2; tools/csr_runs_ab.sh)
            if (staged && ysmem <= 200 * 1024 && H.y_stride % 4 == 0) {
                if (ysmem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(csr_stage_key_kernel));
                csr_stage_key_kernel<<<(unsigned)n_blocks, 512, ysmem, s>>>(t->csr, yws, H.y_stride, ywords, kz,
                                                                            z_stride);
            } else if (use_runs && t->n_runs && zsmem <= 200 * 1024) {
                if (zsmem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(csr_run_key_kernel));
                csr_run_key_kernel<<<(unsigned)n_blocks, 512, zsmem, s>>>(
                    t->runs, t->run_ptr, t->n_batches, yws, H.y_stride, ywords, kz, z_stride);
            } else {
                csr_key_kernel<<<(unsigned)(w1 < cap ? w1 : cap), 256, 0, s>>>(t->csr, yws, H.y_stride, n_blocks,
                                                                              ywords, kz, z_stride);
            }
            zpack_kernel<<<(unsigned)(w2 < cap ? w2 : cap), 256, 0, s>>>(kz, z_stride, n_blocks, (uint32_t)m, m_magic,
                                                                        out);
            count_launch();
            tc.stop();
            if (cudaGetLastError() != cudaSuccess) { set_error("csr_key / zpack launch failed"); st = QRNG_E_CUDA; }
            cudaFreeAsync(kz, s);
        }
    } else if (st == QRNG_OK && gather) {
        // one thread per output word, gathers from L2 (no staging)
        const uint64_t gwords = ((uint64_t)n_blocks * m + 31) / 32;
        const uint64_t m_magic = m > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / m) + 1 : 0;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t want = (gwords + 255) / 256, cap = (uint64_t)sms * 16;
        KernelTimer tc(s, true, 1);
        csr_gather_pack_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(t->csr, yws, H.y_stride, n_blocks,
                                                                                   (uint32_t)m, m_magic, out);
        tc.stop();
        if (cudaGetLastError() != cudaSuccess) { set_error("csr_gather_pack_kernel launch failed"); st = QRNG_E_CUDA; }
    } else if (st == QRNG_OK && stream_smem <= 200 * 1024 && stream_form) {
        // the same, persistent, with the next group's rows in flight (TMA bulk copies)
        auto kern = fused ? (t->csr_kmax <= 2   ? csr_stream_pack_kernel<2, true>
                             : t->csr_kmax <= 4 ? csr_stream_pack_kernel<4, true>
                                                : csr_stream_pack_kernel<8, true>)
                          : (t->csr_kmax <= 2   ? csr_stream_pack_kernel<2, false>
                             : t->csr_kmax <= 4 ? csr_stream_pack_kernel<4, false>
                                                : csr_stream_pack_kernel<8, false>);
        if (stream_smem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(kern));
        int dev = 0, sms = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, QRNG_CSR_THREADS, stream_smem);
        const uint64_t groups = (n_blocks + bpc - 1) / bpc, cap = (uint64_t)sms * std::max(per_sm, 1);
        KernelTimer tc(s, true, 1);
        const uint64_t m_magic = m > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / m) + 1 : 0;
        const cudaError_t le = launch_pdl(kern, dim3((unsigned)(groups < cap ? groups : cap)),
                                          dim3(QRNG_CSR_THREADS), stream_smem, s, t->csr, csr_words,
                                          (const uint32_t *)yws, H.y_stride, n_blocks, (uint32_t)m, bpc, m_magic, out);
        if (le != cudaSuccess) { set_error("csr_stream_pack_kernel: %s", cudaGetErrorString(le)); st = QRNG_E_CUDA; }
        tc.stop();
        if (cudaGetLastError() != cudaSuccess) { set_error("csr_stream_pack_kernel launch failed"); st = QRNG_E_CUDA; }
    } else if (st == QRNG_OK && csr_smem <= 200 * 1024) {
        // flattened tree over bpc blocks of leaf parities in shared memory
        if (csr_smem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(csr_pack_kernel));
        KernelTimer tc(s, true, 1);
        csr_pack_kernel<<<(unsigned)((n_blocks + bpc - 1) / bpc), QRNG_CSR_THREADS, csr_smem, s>>>(t->csr, csr_words, yws, H.y_stride,
                                                                                       n_blocks, (uint32_t)m, bpc, out);
        tc.stop();
        if (cudaGetLastError() != cudaSuccess) { set_error("csr_pack_kernel launch failed"); st = QRNG_E_CUDA; }
    } else if (st == QRNG_OK && fused_smem <= 200 * 1024) {
        // whole tree of 32 blocks in shared memory
        if (fused_smem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(tree_pack_kernel));
        count_launch();
        tree_pack_kernel<<<(unsigned)((n_blocks + 31) / 32), 512, fused_smem, s>>>(
            t->inner, t->unit_node, t->levels, (uint32_t)H.levels.size(), yws, H.y_stride, H.z_stride, n_blocks,
            (uint32_t)m, out);
        if (cudaGetLastError() != cudaSuccess) { set_error("tree_pack_kernel launch failed"); st = QRNG_E_CUDA; }
    } else if (st == QRNG_OK) {
        if (cudaMallocAsync(&zws, (size_t)n_blocks * H.z_stride * 4, s) != cudaSuccess) {
            set_error("cudaMallocAsync failed");
            st = QRNG_E_NOMEM;
        }
        // every node below the root; CTAs of bpc blocks, at least ~4 CTAs per SM
        const uint32_t bpc = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(32, n_blocks / 592));
        if (st == QRNG_OK && H.levels.size() > 1) {
            count_launch();
            combine_kernel<<<(unsigned)((n_blocks + bpc - 1) / bpc), 512, 0, s>>>(
                t->inner, t->unit_node, t->levels, (uint32_t)H.levels.size() - 1, yws, H.y_stride, zws, H.z_stride,
                n_blocks, bpc);
            if (cudaGetLastError() != cudaSuccess) { set_error("combine_kernel launch failed"); st = QRNG_E_CUDA; }
        }
        if (st == QRNG_OK) {
            // 32 blocks per CTA (their keys are exactly m output words); stage the
            // root rows in shared memory when they fit
            const size_t smem = (size_t)32 * rw4 * 16;
            const unsigned grid = (unsigned)((n_blocks + 31) / 32);
            const uint32_t *root = t->inner + 8 * (H.inner.size() - 1);
            count_launch();
            if (smem <= 200 * 1024) {
                if (smem > 48 * 1024) allow_max_smem(reinterpret_cast<const void *>(pack_kernel<true>));
                pack_kernel<true><<<grid, 256, smem, s>>>(root, yws, H.y_stride, zws, H.z_stride, n_blocks,
                                                          (uint32_t)m, out);
            } else {
                pack_kernel<false><<<grid, 256, 0, s>>>(root, yws, H.y_stride, zws, H.z_stride, n_blocks,
                                                        (uint32_t)m, out);
            }
            if (cudaGetLastError() != cudaSuccess) { set_error("pack_kernel launch failed"); st = QRNG_E_CUDA; }
        }
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

// TEST ONLY: the one-pass Q-buffer chunk list and each leaf's input location
// (no GPU needed).  See include/qrng.h (qrng_debug_qslice_plan).
extern "C" qrng_status qrng_debug_qslice_plan(uint64_t n, uint64_t m, int max_depth, uint32_t *ent, uint32_t ent_cap,
                                              uint32_t *leaf_x, uint32_t leaf_cap, uint32_t *info) {
    using namespace qrng;
    using namespace qrng::kara;
    HostTables T;
    if (!info) { set_error("info is NULL"); return QRNG_E_INVALID; }
    if (!plan_host(n, m, max_depth, T)) { set_error("no decomposition"); return QRNG_E_UNSUPPORTED; }
    QSliceHost qs;
    info[0] = (uint32_t)qslice_host(T, n, qs);
    info[1] = qs.lsu;
    info[2] = qs.n_ent;
    info[3] = T.x_stride;
    info[4] = (uint32_t)T.leaves.size();
    if (!ent || !leaf_x || ent_cap < qs.n_ent || leaf_cap < T.leaves.size()) return QRNG_OK;  // sizes only
    for (uint32_t e = 0; e < qs.n_ent; ++e) ent[e] = qs.ent[e];
    for (size_t l = 0; l < T.leaves.size(); ++l) {
        const auto &L = T.leaves[l];
        leaf_x[2 * l] = L.src < 0 ? 0u : 1u;
        leaf_x[2 * l + 1] = L.src < 0 ? L.src_off / 32 : T.qbufs[L.src].dst + L.src_off / 32;
    }
    return QRNG_OK;
}
