// gbt.cu -- gbt_create / gbt_export / gbt_destroy / gbt_predict.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gbt.cuh"

namespace at {

constexpr int PRED_NW = 16;  // warps per block (tree slices); 32 candidates per tile

TreeGeo make_geo(const at_gbt_s *g, uint32_t buf_bytes, bool rank, int nbuf, int ring, int leaf_global)
{
    TreeGeo G{};
    G.nodes = rank ? (const uint8_t *)g->d_rk_nodes : (const uint8_t *)g->d_nodes;
    G.nbytes = rank ? 4 : 8;
    G.leaf = g->d_leaf;
    G.T = g->n_trees;
    G.T_pad = g->t_pad;
    G.D = g->depth;
    G.ni = (1 << g->depth) - 1;
    G.nl = 1 << g->depth;
    const uint32_t per_tree = (uint32_t)G.ni * (uint32_t)G.nbytes + (leaf_global ? 0u : (uint32_t)G.nl * 4u);
    G.leaf_global = leaf_global;
    int ch = (int)(buf_bytes / per_tree) / 2 * 2;   // even: chunk offsets and sizes stay 16-B aligned
    if (ch >= 32) ch = ch / 32 * 32;                 // whole 32-tree rounds: no idle walk slots
    if (ch < 2) ch = 2;
    if (ch > G.T_pad) ch = G.T_pad;
    G.CH = ch;
    G.NC = (G.T + ch - 1) / ch;
    G.chunk_bytes = (uint32_t)ch * per_tree;
    G.NBUF = nbuf;
    G.ring = ring;
    G.resident = G.NC <= nbuf;
    G.Tm = G.T;
    return G;
}

// Persistent scorer: one block per SM loops over 32-candidate tiles.  The ensemble streams (or
// stays resident) through the TMA tree pipeline of gbt.cuh; the candidate tiles are fetched by
// 1-D bulk copies (one 128-B row segment per feature, issued by warp 0's lanes) into two tile
// buffers, so the next tile's HBM read overlaps the current tile's tree walk.
struct PredSmemHdr {
    uint64_t tree_bar[2];
    uint64_t tile_bar[2];
};

// candidate tile = n_box 2-D TMA boxes of {32 candidates, box_rows features} of X[F][ld]
struct TileMap {
    CUtensorMap map;
    int n_box, box_rows;
};

// one tile = GRP groups of 32 candidates; group g of tile `tile` starts at candidate (tile GRP + g) 32
template <int GRP, class T>
__device__ __forceinline__ void tile_issue(const TileMap &tm, int64_t tile, T *dst, int tile_rows, uint64_t *bar)
{
    mbar_arrive_expect_tx(bar, (uint32_t)(GRP * tm.n_box * tm.box_rows * 32 * sizeof(T)));
    for (int g = 0; g < GRP; ++g)
        for (int b = 0; b < tm.n_box; ++b)
            tma_load_2d(dst + g * tile_rows * 32 + b * tm.box_rows * 32, &tm.map, (int)((tile * GRP + g) * 32),
                        b * tm.box_rows, bar);
}

// Persistent scorer: one block per SM loops over tiles of 32 GRP candidates.  The ensemble
// streams (or stays resident) through the TMA tree pipeline of gbt.cuh; candidate tiles arrive by
// 2-D TMA (tensor map over X[F][ld]).  GRP = 1: two tile buffers, the next tile's HBM read overlaps
// the current walk (small, resident ensembles: HBM-bound).  GRP = 2: one buffer of 64 candidates,
// so every streamed tree byte serves twice the candidates (large ensembles: L2-bound).
template <int GRP, int KM, bool RK, int ONLY = 0>
__global__ void __launch_bounds__((PRED_NW + 1) * 32, 1) predict_kernel(TreeGeo G, float base, int F, int tile_rows,
                                                                 const void *__restrict__ Xv, int64_t n, int64_t ld,
                                                                 float *__restrict__ score, uint8_t *__restrict__ slots,
                                                                 int use_bulk, const __grid_constant__ TileMap tm,
                                                                 const __grid_constant__ AcqArgs Q)
{
    using T = typename std::conditional<RK, uint32_t, float>::type;   // tile element: rank pair or feature value
    constexpr int NBUF = GRP == 1 ? 2 : 1;
    const T *X = (const T *)Xv;
    extern __shared__ __align__(128) unsigned char smraw[];
    PredSmemHdr &hd = *(PredSmemHdr *)smraw;
    float *part = (float *)(smraw + 128);                      // [GRP][KM][32][32]
    float *fk = part + GRP * KM * 32 * 32;                     // [GRP][KM][32] per-model scores (KM > 1)
    T *tiles = (T *)(fk + (KM > 1 ? GRP * KM * 32 : 0));      // [NBUF][GRP][tile_rows][32], tile_rows >= F
    uint8_t *bufs = (uint8_t *)(tiles + NBUF * GRP * tile_rows * 32);   // tree buffers (rows are 128 B)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_tiles = (n + 32 * GRP - 1) / (32 * GRP);
    const int64_t my_tiles = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int tstride = GRP * tile_rows * 32;
    if (threadIdx.x == 0) {
        mbar_init(&hd.tile_bar[0], 1);
        mbar_init(&hd.tile_bar[1], 1);
    }
    ts_start(G, bufs, hd.tree_bar);   // also fences the barrier initialisation
    __syncthreads();
    if (threadIdx.x == 0 && use_bulk) {
        for (int i = 0; i < NBUF && i < my_tiles; ++i)
            tile_issue<GRP>(tm, blockIdx.x + i * gridDim.x, tiles + i * tstride, tile_rows, &hd.tile_bar[i]);
    }
    ts_wait_resident(G, hd.tree_bar);
    uint32_t ph[2] = {0u, 0u};
    uint64_t c = 0;
    const uint64_t c_limit = (uint64_t)G.NC * (uint64_t)my_tiles;
    for (int64_t i = 0; i < my_tiles; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        const int tb = (int)(i % NBUF);
        T *tl = tiles + tb * tstride;
        const int64_t cand0 = tile * 32 * GRP + lane;
        bool ok[GRP];
#pragma unroll
        for (int g = 0; g < GRP; ++g) ok[g] = cand0 + 32 * g < n;
        if (use_bulk) {
            mbar_wait(&hd.tile_bar[tb], (uint32_t)((i / NBUF) & 1));
        } else {
            for (int g = 0; g < GRP; ++g)
                for (int f = warp; f < F && warp < PRED_NW; f += PRED_NW)
                    tl[g * tile_rows * 32 + f * 32 + lane] = ok[g] ? X[(int64_t)f * ld + cand0 + 32 * g] : (T)0;
            __syncthreads();
        }
        walk_pass<PRED_NW, GRP, KM, RK, false, PRED_NW, ONLY>(G, bufs, hd.tree_bar, ph, c, c_limit, tl, tile_rows * 32, lane, warp, part,
                                        KM * 1024, slots,
                                    n, cand0, ok);
        if (KM == 1) {
            if (warp < GRP) {
                if (ok[warp]) score[cand0 + 32 * warp] = gbt_combine(part + warp * 1024, lane, base);
            }
        } else {
            // warp (g, m) folds model m's partials in the canonical order; then warp g takes the acquisition
            if (warp < GRP * Q.K) {
                const int g = warp / Q.K, m = warp - g * Q.K;
                fk[(g * KM + m) * 32 + lane] = gbt_combine(part + (g * KM + m) * 1024, lane, Q.base[m]);
            }
            __syncthreads();
            if (warp < GRP && ok[warp]) {
                float mu, sd;
                const int64_t i = cand0 + 32 * warp;
                score[i] = acquisition(Q, fk + warp * KM * 32 + lane, 32, mu, sd);
                if (Q.mean) Q.mean[i] = mu;
                if (Q.std) Q.std[i] = sd;
            }
        }
        __syncthreads();   // part[] and the tile buffer are free again
        if (use_bulk && warp == PRED_NW && lane == 0 && i + NBUF < my_tiles) {   // the producer warp
            fence_proxy_async();
            tile_issue<GRP>(tm, tile + NBUF * gridDim.x, tl, tile_rows, &hd.tile_bar[tb]);
        }
    }
}

size_t tree_smem_bytes(const TreeGeo &G)
{
    return (size_t)2 * G.chunk_bytes + 128;
}

}  // namespace at

extern "C" {

int gbt_create(int32_t n_trees, int32_t depth, int32_t n_features, const uint16_t *feat, const float *thresh,
               const float *leaf, float base, at_gbt *out)
{
    if (!feat || !thresh || !leaf || !out) return at::fail(AT_EINVAL, "gbt_create: null pointer");
    if (n_trees < 1 || depth < 1 || depth > 8) return at::fail(AT_EUNSUPPORTED, "gbt_create: need n_trees >= 1, 1 <= depth <= 8");
    if (n_features < 1 || n_features > 65535) return at::fail(AT_EINVAL, "gbt_create: bad n_features");
    const int64_t ni = (1 << depth) - 1, nl = 1 << depth;
    std::vector<uint2> nodes((size_t)n_trees * ni);
    for (int64_t i = 0; i < (int64_t)nodes.size(); ++i) {
        if (feat[i] >= n_features) return at::fail(AT_EINVAL, "gbt_create: feature index >= n_features");
        uint32_t tb;
        std::memcpy(&tb, &thresh[i], 4);
        if (std::isnan(thresh[i])) return at::fail(AT_EINVAL, "gbt_create: NaN threshold");
        nodes[i] = make_uint2(feat[i], tb);
    }
    at_gbt g = new at_gbt_s();
    g->n_trees = n_trees;
    g->depth = depth;
    g->n_features = n_features;
    g->t_pad = (n_trees + 15) / 16 * 16;
    g->base = base;
    g->d_nodes = nullptr;
    g->d_leaf = nullptr;
    g->last = 0;
    if (cudaMallocAsync((void **)&g->d_nodes, (size_t)g->t_pad * ni * sizeof(uint2), 0) != cudaSuccess ||
        cudaMallocAsync((void **)&g->d_leaf, (size_t)g->t_pad * nl * sizeof(float), 0) != cudaSuccess ||
        cudaMemsetAsync(g->d_nodes, 0, (size_t)g->t_pad * ni * sizeof(uint2), 0) != cudaSuccess ||
        cudaMemsetAsync(g->d_leaf, 0, (size_t)g->t_pad * nl * sizeof(float), 0) != cudaSuccess) {
        cudaGetLastError();
        cudaFreeAsync(g->d_nodes, 0);
        delete g;
        return at::fail(AT_ENOMEM, "gbt_create: device allocation failed");
    }
    cudaError_t e1 = cudaMemcpy(g->d_nodes, nodes.data(), nodes.size() * sizeof(uint2), cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(g->d_leaf, leaf, (size_t)n_trees * nl * sizeof(float), cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaFreeAsync(g->d_nodes, 0);
        cudaFreeAsync(g->d_leaf, 0);
        delete g;
        return at::cuda_fail(e1 != cudaSuccess ? e1 : e2, "gbt_create upload");
    }
    *out = g;
    return AT_OK;
}

int gbt_info(at_gbt g, int32_t *n_trees, int32_t *depth, int32_t *n_features)
{
    if (!g) return at::fail(AT_EINVAL, "gbt_info: null model");
    if (n_trees) *n_trees = g->n_trees;
    if (depth) *depth = g->depth;
    if (n_features) *n_features = g->n_features;
    return AT_OK;
}

int gbt_export(at_gbt g, uint16_t *feat, float *thresh, float *leaf, float *base)
{
    if (!g) return at::fail(AT_EINVAL, "gbt_export: null model");
    AT_CUDA_TRY(cudaStreamSynchronize(g->last));   // the fit that wrote it may run on a non-blocking stream
    if (int rc = at::model_error(g)) return rc;
    const int64_t ni = (1 << g->depth) - 1, nl = 1 << g->depth;
    if (feat || thresh) {
        std::vector<uint2> nodes((size_t)g->n_trees * ni);
        AT_CUDA_TRY(cudaMemcpy(nodes.data(), g->d_nodes, nodes.size() * sizeof(uint2), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < nodes.size(); ++i) {
            if (feat) feat[i] = (uint16_t)nodes[i].x;
            if (thresh) std::memcpy(&thresh[i], &nodes[i].y, 4);
        }
    }
    if (leaf) AT_CUDA_TRY(cudaMemcpy(leaf, g->d_leaf, (size_t)g->n_trees * nl * sizeof(float), cudaMemcpyDeviceToHost));
    if (base) *base = g->base;
    return AT_OK;
}

// Eq. 4: f_global + f_local as one ensemble.  A depth-d tree inside a depth-D
// ensemble keeps heap nodes 0 .. 2^d - 2; its former leaf nodes and everything below them are
// pass-through (feature 0, threshold +inf), so former slot s always ends at slot s * 2^(D - d).
int gbt_concat(at_gbt a, at_gbt b, at_gbt *out)
{
    if (!a || !b || !out) return at::fail(AT_EINVAL, "gbt_concat: null handle");
    AT_CUDA_TRY(cudaStreamSynchronize(a->last));   // host-side construction from both models
    AT_CUDA_TRY(cudaStreamSynchronize(b->last));
    if (int rc = at::model_error(a)) return rc;
    if (int rc = at::model_error(b)) return rc;
    if (a->n_features != b->n_features) return at::fail(AT_EMISMATCH, "gbt_concat: different n_features");
    const int D = std::max(a->depth, b->depth);
    const int64_t NI = (1 << D) - 1, NL = 1 << D;
    const int T = a->n_trees + b->n_trees;
    std::vector<uint16_t> feat((size_t)T * NI, 0);
    std::vector<float> thr((size_t)T * NI, INFINITY), leaf((size_t)T * NL, 0.0f);
    int t0 = 0;
    for (at_gbt m : {a, b}) {
        const int64_t ni = (1 << m->depth) - 1, nl = 1 << m->depth;
        std::vector<uint16_t> f((size_t)m->n_trees * ni);
        std::vector<float> th((size_t)m->n_trees * ni), lv((size_t)m->n_trees * nl);
        const int rc = gbt_export(m, f.data(), th.data(), lv.data(), nullptr);
        if (rc) return rc;
        const int sh = D - m->depth;
        for (int t = 0; t < m->n_trees; ++t) {
            const size_t u = (size_t)(t0 + t);
            std::copy(f.begin() + (size_t)t * ni, f.begin() + (size_t)(t + 1) * ni, feat.begin() + u * NI);
            std::copy(th.begin() + (size_t)t * ni, th.begin() + (size_t)(t + 1) * ni, thr.begin() + u * NI);
            for (int64_t q = 0; q < nl; ++q) leaf[u * NL + ((size_t)q << sh)] = lv[(size_t)t * nl + q];
        }
        t0 += m->n_trees;
    }
    return gbt_create(T, D, a->n_features, feat.data(), thr.data(), leaf.data(), a->base + b->base, out);   // host fp32 add (SSE, RN)
}

int gbt_destroy(at_gbt g)
{
    if (!g) return AT_OK;
    // stream-ordered after the model's last enqueued use (predict / SA / fit output)
    cudaFreeAsync(g->d_nodes, g->last);
    cudaFreeAsync(g->d_leaf, g->last);
    if (g->d_rk_nodes) cudaFreeAsync(g->d_rk_nodes, g->last);
    if (g->d_thr_off) cudaFreeAsync(g->d_thr_off, g->last);
    if (g->d_thr_val) cudaFreeAsync(g->d_thr_val, g->last);
    if (g->h_err) {   // mapped word the fit's last kernel writes: freed after the model's stream drains
        cudaStreamSynchronize(g->last);
        cudaFreeHost(g->h_err);
    }
    delete g;
    return AT_OK;
}

}  // extern "C"

namespace at {

// ---------------------------------------------------------------- rank form (deep ensembles)
// Depth >= 7 ensembles stream through shared memory once per candidate tile, and a block's walks in
// flight are bounded by how many trees and candidates fit beside each other.  The rank form halves
// both: a node is one word {k | tile offset << 16} (k = the 1-based index of its threshold among the
// feature's sorted distinct thresholds) and a candidate feature is the u16 rank(x) = #{theta <= x},
// computed by rank_encode_kernel.  For thresholds theta_1 < ... < theta_m, rank(x) < k <=> not
// (theta_k <= x) <=> x < theta_k, so every branch -- and every score -- is bit-identical to the fp32
// walk; a NaN feature ranks 0xFFFF (goes right everywhere, like x < theta = false).
static int build_rank_form(at_gbt g)
{
    if (g->rk_state) return g->rk_state;
    g->rk_state = -1;
    if (g->n_features > 1022) return -1;   // tile byte offsets (F / 2) * 128 must fit 16 bits
    const int64_t ni = (1 << g->depth) - 1;
    std::vector<uint16_t> feat((size_t)g->n_trees * ni);
    std::vector<float> thr((size_t)g->n_trees * ni);
    if (gbt_export(g, feat.data(), thr.data(), nullptr, nullptr) != AT_OK) return -1;
    const int F = g->n_features;
    std::vector<std::vector<float>> vals(F);
    for (size_t i = 0; i < feat.size(); ++i) vals[feat[i]].push_back(thr[i]);
    std::vector<int32_t> off(F + 1, 0);
    std::vector<float> tab;
    for (int f = 0; f < F; ++f) {
        std::vector<float> &v = vals[f];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end(), [](float x, float y) { return x == y; }), v.end());   // -0 == +0
        if (v.size() > 65534) return -1;
        off[f] = (int32_t)tab.size();
        tab.insert(tab.end(), v.begin(), v.end());
    }
    off[F] = (int32_t)tab.size();
    std::vector<uint32_t> rk((size_t)g->t_pad * ni, 0u);   // padded trees: offset 0, k 0 (never walked)
    for (size_t i = 0; i < feat.size(); ++i) {
        const std::vector<float> &v = vals[feat[i]];
        const size_t k = (size_t)(std::lower_bound(v.begin(), v.end(), thr[i]) - v.begin()) + 1;
        const uint32_t off_f = ((uint32_t)feat[i] >> 1) * 128u + ((uint32_t)feat[i] & 1u) * 2u;   // byte in the tile
        rk[i] = (uint32_t)k | (off_f << 16);
    }
    if (cudaMalloc((void **)&g->d_rk_nodes, rk.size() * 4) != cudaSuccess ||
        cudaMalloc((void **)&g->d_thr_off, off.size() * 4) != cudaSuccess ||
        cudaMalloc((void **)&g->d_thr_val, std::max<size_t>(tab.size(), 1) * 4) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (cudaMemcpy(g->d_rk_nodes, rk.data(), rk.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(g->d_thr_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
        (!tab.empty() && cudaMemcpy(g->d_thr_val, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess))
        return -1;
    g->rk_state = 1;
    return 1;
}

// Xr[p][i] = rank(X[2p][i]) | rank(X[2p + 1][i]) << 16, rank = #{theta <= x} among the feature's
// sorted distinct thresholds (NaN ranks 0xFFFF).  Block = one feature pair x RE_CAND candidates: the
// pair's two tables are staged in shared memory (when they fit) and every thread runs branch-free
// binary searches (a fixed number of halvings per table) for 8 candidates at once.
constexpr int RE_NT = 256, RE_PER = 8, RE_CAND = RE_NT * RE_PER, RE_SMEM = 512;

// global-table fallback (a feature with more thresholds than the staging buffer holds)
__device__ __forceinline__ uint32_t rank_search_g(const float *__restrict__ tab, int len, float x)
{
    int lo = 0, hi = len;   // first theta > x
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(tab + mid) <= x) lo = mid + 1; else hi = mid;
    }
    return x != x ? 0xFFFFu : (uint32_t)lo;
}

// staged table padded with +inf to P - 1 entries (P a power of two > len, P <= 256): log2 P branch-free
// halvings, unrolled (the guards are block-uniform)
__device__ __forceinline__ uint32_t rank_search_s(const float *tab, int len, int P, float x)
{
    int lo = 0;
#pragma unroll
    for (int step = 128; step > 0; step >>= 1)
        if (step < P) lo += tab[lo + step - 1] <= x ? step : 0;
    return x != x ? 0xFFFFu : (uint32_t)min(lo, len);   // x = +inf also passes the padding
}

__global__ void __launch_bounds__(RE_NT) rank_encode_kernel(const float *__restrict__ X, int64_t n, int64_t ld, int F,
                                                            const int32_t *__restrict__ off,
                                                            const float *__restrict__ val, uint32_t *__restrict__ Xr,
                                                            int64_t ldr)
{
    __shared__ float st[RE_SMEM];
    const int p = blockIdx.y;
    const int f0 = 2 * p, f1 = 2 * p + 1 < F ? 2 * p + 1 : -1;
    const int b0 = off[f0], l0 = off[f0 + 1] - b0;
    const int b1 = f1 >= 0 ? off[f1] : 0, l1 = f1 >= 0 ? off[f1 + 1] - b1 : 0;
    int P0 = 1, P1 = 1;
    while (P0 <= l0) P0 *= 2;
    while (P1 <= l1) P1 *= 2;
    const bool staged = P0 <= 256 && P1 <= 256;   // block-uniform (fitted models: <= 255 cuts per feature)
    if (staged) {
        for (int q = threadIdx.x; q < P0; q += RE_NT) st[q] = q < l0 ? val[b0 + q] : __int_as_float(0x7f800000);
        for (int q = threadIdx.x; q < P1; q += RE_NT) st[P0 + q] = q < l1 ? val[b1 + q] : __int_as_float(0x7f800000);
    }
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * RE_CAND + threadIdx.x;
    float x0[RE_PER], x1[RE_PER];
#pragma unroll
    for (int k = 0; k < RE_PER; ++k) {
        const int64_t i = i0 + (int64_t)k * RE_NT;
        x0[k] = i < n ? X[(int64_t)f0 * ld + i] : 0.0f;
        x1[k] = (i < n && f1 >= 0) ? X[(int64_t)f1 * ld + i] : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < RE_PER; ++k) {
        const int64_t i = i0 + (int64_t)k * RE_NT;
        uint32_t r0, r1;
        if (staged) {
            r0 = rank_search_s(st, l0, P0, x0[k]);
            r1 = f1 >= 0 ? rank_search_s(st + P0, l1, P1, x1[k]) : 0u;
        } else {
            r0 = rank_search_g(val + b0, l0, x0[k]);
            r1 = f1 >= 0 ? rank_search_g(val + b1, l1, x1[k]) : 0u;
        }
        if (i < n) Xr[(int64_t)p * ldr + i] = r0 | (r1 << 16);
    }
}

// gbt_predict / gbt_predict_acq: one persistent scorer launch (KM = 1: one model; KM = 8: up to 8
// concatenated models of equal tree count with their acquisition)
static int predict_launch(at_gbt g, const float *d_feat, int64_t n, int64_t ld, float *d_score, uint8_t *d_leaf_slot,
                          const AcqArgs *acq, void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    const int KM = acq ? 8 : 1;
    const int F = g->n_features;
    const int n_box = (F + 255) / 256, box_rows = (F + n_box - 1) / n_box, tile_rows = n_box * box_rows;
    constexpr size_t SMEM_MAX = 227 * 1024;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        AT_CUDA_TRY(cudaGetDevice(&dev));
        AT_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    // rank form: deep ensembles that stream (4 candidate groups per tile, 16-tree chunks)
    const char *rk_e = getenv("AT_PREDICT_RANK");   // "0" forces the fp32 walk
    const bool want_rk = !acq && g->depth >= 7 && (!rk_e || atoi(rk_e) != 0) && n > 0;
    // the rank tables are built (once) from the model as its last writer left it, then this stream owns it
    const int rk_ok = want_rk ? build_rank_form(g) : 0;
    g->last = s;
    // candidate groups per tile: 4 (16-tree chunks: every streamed tree byte serves 128 candidates) when
    // there are >= 8 tiles per SM to balance, else 2 (32-tree chunks); with the streamed rank walk
    // (walk_stream_rank) 4 groups run config 5 at 10^7 candidates 1.18x faster.  AT_RK_GRP=2|4 forces it
    const char *rg_e = getenv("AT_RK_GRP");
    int nsm_rk = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm_rk, cudaDevAttrMultiProcessorCount, dev);
    }
    const int RGRP = rg_e ? (atoi(rg_e) == 4 ? 4 : 2) : (n >= (int64_t)nsm_rk * 8 * 128 ? 4 : 2);
    if (want_rk && rk_ok == 1) {
        const int P = (F + 1) / 2;   // u32 rank pairs per candidate
        const int pn_box = (P + 255) / 256, pbox_rows = (P + pn_box - 1) / pn_box, ptile_rows = pn_box * pbox_rows;
        TreeGeo G = make_geo(g, (RGRP == 2 ? 32 : 16) * ((uint32_t)((1 << g->depth) - 1) * 4u + (uint32_t)(1 << g->depth) * 4u),
                             true);
        const size_t smem = 128 + (size_t)RGRP * 32 * 32 * sizeof(float) + (size_t)RGRP * ptile_rows * 32 * 4 +
                            tree_smem_bytes(G);
        if (!G.resident && smem <= SMEM_MAX) {
            // the streamed rank pass only (no leaf slots, 16- or 32-tree chunks of depth 7-8 trees): a kernel
            // variant with only that walk compiled in
            const bool sr = !d_leaf_slot && !G.ring && G.NP <= 1 && (G.CH == PRED_NW || G.CH == 2 * PRED_NW) &&
                            G.D >= 7 && G.D <= 8;
            const void *rk_kern = RGRP == 2 ? (sr ? (const void *)predict_kernel<2, 1, true, 2> : (const void *)predict_kernel<2, 1, true>)
                                            : (sr ? (const void *)predict_kernel<4, 1, true, 2> : (const void *)predict_kernel<4, 1, true>);
            static size_t rk_attr[4] = {0, 0, 0, 0};
            const int rai = (RGRP == 2) + 2 * sr;
            if (smem > rk_attr[rai]) {
                AT_CUDA_TRY(cudaFuncSetAttribute(rk_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                rk_attr[rai] = smem;
            }
            pool_keep();   // the rank tiles below are stream-ordered scratch
            const int64_t ldr = (n + 3) / 4 * 4;   // 16-B rows for the tensor map
            uint32_t *Xr = nullptr;
            AT_CUDA_TRY(cudaMallocAsync((void **)&Xr, (size_t)P * ldr * 4, s));
            {
                ProfScope ps(AT_K_FEATURES, s);
                rank_encode_kernel<<<dim3((unsigned)((n + RE_CAND - 1) / RE_CAND), P), RE_NT, 0, s>>>(
                    d_feat, n, ld, F, g->d_thr_off, g->d_thr_val, Xr, ldr);
                note_launch();
                AT_LAUNCH_CHECK("rank_encode_kernel");
            }
            TileMap tm{};
            tm.n_box = pn_box;
            tm.box_rows = pbox_rows;
            int use_bulk = 0;
            {
                static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
                if (!encode) {
                    void *fn = nullptr;
                    cudaDriverEntryPointQueryResult q;
                    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                        q == cudaDriverEntryPointSuccess)
                        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
                }
                const cuuint64_t dims[2] = {(cuuint64_t)ldr, (cuuint64_t)P};
                const cuuint64_t strides[1] = {(cuuint64_t)ldr * 4};
                const cuuint32_t box[2] = {32u, (cuuint32_t)pbox_rows};
                const cuuint32_t estr[2] = {1u, 1u};
                use_bulk = encode && encode(&tm.map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void *)Xr, dims, strides, box,
                                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
            const int64_t tiles = (n + 32 * RGRP - 1) / (32 * RGRP);
            const unsigned blocks = (unsigned)std::min<int64_t>(tiles, n_sm);
            AcqArgs Q{};
            {
                ProfScope ps(AT_K_PREDICT, s);
#define AT_RK_LAUNCH(GR, ON)                                                                                          \
    predict_kernel<GR, 1, true, ON><<<blocks, (PRED_NW + 1) * 32, smem, s>>>(G, g->base, P, ptile_rows, Xr, n, ldr, d_score, \
                                                                          d_leaf_slot, use_bulk, tm, Q)
                if (RGRP == 2) {
                    if (sr) AT_RK_LAUNCH(2, 2); else AT_RK_LAUNCH(2, 0);
                } else {
                    if (sr) AT_RK_LAUNCH(4, 2); else AT_RK_LAUNCH(4, 0);
                }
#undef AT_RK_LAUNCH
                note_launch();
                AT_LAUNCH_CHECK("predict_kernel (rank form)");
            }
            AT_CUDA_TRY(cudaFreeAsync(Xr, s));
            return AT_OK;
        }
    }
    TreeGeo G = make_geo(g, acq ? 32 * 1024 : TREE_BUF_BYTES);
    if (acq) G.Tm = g->n_trees / acq->K;
    // GRP = 2 (64 candidates per tile, one buffer) when the ensemble streams and it fits
    auto smem_for = [&](int grp) {
        const int nbuf = grp == 1 ? 2 : 1;
        return 128 + (size_t)grp * KM * 32 * 32 * sizeof(float) + (KM > 1 ? (size_t)grp * KM * 32 * sizeof(float) : 0) +
               (size_t)nbuf * grp * tile_rows * 32 * sizeof(float) + tree_smem_bytes(G);
    };
    const int grp = (!acq && !G.resident && smem_for(2) <= SMEM_MAX) ? 2 : 1;
    const size_t smem = smem_for(grp);
    if (smem > SMEM_MAX) return fail(AT_EUNSUPPORTED, "gbt_predict: too many features for the smem tiles");
    // two groups on the generic streamed pass (a chunk barrier every chunk): a variant with only that walk
    const bool gen = !acq && grp == 2 && !G.resident && !G.ring && G.NP <= 1 &&
                     !(G.CH == PRED_NW && !d_leaf_slot && G.D >= 6 && G.D <= 8);
    const void *kern = acq ? (const void *)predict_kernel<1, 8, false>
                     : grp == 1 ? (const void *)predict_kernel<1, 1, false>
                     : gen ? (const void *)predict_kernel<2, 1, false, 3> : (const void *)predict_kernel<2, 1, false>;
    static size_t attr[4] = {0, 0, 0, 0};
    const int ai = acq ? 2 : gen ? 3 : grp - 1;
    if (smem > attr[ai]) {
        AT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[ai] = smem;
    }
    // TMA tensor map over X[F][ld] (needs 16-B aligned rows); otherwise plain loads
    TileMap tm{};
    tm.n_box = n_box;
    tm.box_rows = box_rows;
    int use_bulk = (ld % 4 == 0) && ((uintptr_t)d_feat % 16 == 0);
    if (use_bulk) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
        }
        const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)F};
        const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
        const cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
        const cuuint32_t estr[2] = {1u, 1u};
        if (!encode || encode(&tm.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)d_feat, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            use_bulk = 0;
    }
    const int64_t tiles = (n + 32 * grp - 1) / (32 * grp);
    const unsigned blocks = (unsigned)std::min<int64_t>(tiles, n_sm);
    AcqArgs Q{};
    if (acq) Q = *acq;
    ProfScope ps(AT_K_PREDICT, s);
    if (acq)
        predict_kernel<1, 8, false><<<blocks, (PRED_NW + 1) * 32, smem, s>>>(G, g->base, F, tile_rows, d_feat, n, ld, d_score,
                                                                d_leaf_slot, use_bulk, tm, Q);
    else if (grp == 1)
        predict_kernel<1, 1, false><<<blocks, (PRED_NW + 1) * 32, smem, s>>>(G, g->base, F, tile_rows, d_feat, n, ld, d_score,
                                                                d_leaf_slot, use_bulk, tm, Q);
    else if (gen)
        predict_kernel<2, 1, false, 3><<<blocks, (PRED_NW + 1) * 32, smem, s>>>(G, g->base, F, tile_rows, d_feat, n, ld,
                                                                   d_score, d_leaf_slot, use_bulk, tm, Q);
    else
        predict_kernel<2, 1, false><<<blocks, (PRED_NW + 1) * 32, smem, s>>>(G, g->base, F, tile_rows, d_feat, n, ld, d_score,
                                                                d_leaf_slot, use_bulk, tm, Q);
    note_launch();
    AT_LAUNCH_CHECK("predict_kernel");
    return AT_OK;
}

}  // namespace at

extern "C" {

int gbt_predict(at_gbt g, const float *d_feat, int64_t n, int64_t ld, float *d_score, uint8_t *d_leaf_slot,
                void *stream)
{
    if (!g) return at::fail(AT_EINVAL, "gbt_predict: null model");
    if (int rc = at::model_error(g)) return rc;
    if (n < 0) return at::fail(AT_EINVAL, "gbt_predict: n < 0");
    if (n == 0) return AT_OK;
    if (!d_feat || !d_score) return at::fail(AT_EINVAL, "gbt_predict: null buffer");
    if (ld < n) return at::fail(AT_EMISMATCH, "gbt_predict: ld < n");
    return at::predict_launch(g, d_feat, n, ld, d_score, d_leaf_slot, nullptr, stream);
}

int gbt_predict_acq(at_gbt g, const float *d_feat, int64_t n, int64_t ld, const at_acq_opts *o, float *d_score,
                    float *d_mean, float *d_std, void *stream)
{
    if (!g || !o) return at::fail(AT_EINVAL, "gbt_predict_acq: null model / options");
    if (int rc = at::model_error(g)) return rc;
    if (o->n_models < 1 || o->n_models > 8 || g->n_trees % o->n_models != 0)
        return at::fail(AT_EINVAL, "gbt_predict_acq: need 1 <= n_models <= 8 dividing n_trees");
    if (o->kind < AT_ACQ_MEAN || o->kind > AT_ACQ_EI) return at::fail(AT_EINVAL, "gbt_predict_acq: bad kind");
    if (n < 0) return at::fail(AT_EINVAL, "gbt_predict_acq: n < 0");
    if (n == 0) return AT_OK;
    if (!d_feat || !d_score) return at::fail(AT_EINVAL, "gbt_predict_acq: null buffer");
    if (ld < n) return at::fail(AT_EMISMATCH, "gbt_predict_acq: ld < n");
    at::AcqArgs Q{};
    Q.K = o->n_models;
    Q.kind = o->kind;
    Q.kappa = o->kappa;
    Q.best = o->best;
    for (int k = 0; k < 8; ++k) Q.base[k] = k < Q.K ? o->model_base[k] : 0.0f;
    Q.mean = d_mean;
    Q.std = d_std;
    return at::predict_launch(g, d_feat, n, ld, d_score, nullptr, &Q, stream);
}

}  // extern "C"
