// gbt.cu -- gbt_create / gbt_export / gbt_destroy / gbt_predict.
#include <cmath>
#include <cstring>
#include <vector>

#include "gbt.cuh"

namespace at {

constexpr int PRED_NW = 8;   // warps per block (tree slices); 32 candidates per block

TreeGeo make_geo(const at_gbt_s *g)
{
    TreeGeo G{};
    G.nodes = g->d_nodes;
    G.leaf = g->d_leaf;
    G.T = g->n_trees;
    G.T_pad = g->t_pad;
    G.D = g->depth;
    G.ni = (1 << g->depth) - 1;
    G.nl = 1 << g->depth;
    const uint32_t per_tree = (uint32_t)G.ni * 8u + (uint32_t)G.nl * 4u;
    int ch = (int)(TREE_BUF_BYTES / per_tree) / 16 * 16;
    if (ch < 16) ch = 16;
    if (ch > G.T_pad) ch = G.T_pad;
    G.CH = ch;
    G.NC = (G.T + ch - 1) / ch;
    G.chunk_bytes = (uint32_t)ch * per_tree;
    G.resident = G.NC <= 2;
    return G;
}

__global__ void __launch_bounds__(PRED_NW * 32) predict_kernel(TreeGeo G, float base, int F,
                                                              const float *__restrict__ X, int64_t n, int64_t ld,
                                                              float *__restrict__ score, uint8_t *__restrict__ slots)
{
    extern __shared__ __align__(128) unsigned char smraw[];
    float *tile = (float *)smraw;                                   // [F][32]
    float *part = tile + F * 32;                                    // [32][32]
    uint64_t *bar = (uint64_t *)(part + 32 * 32);                   // [2]
    uint8_t *bufs = (uint8_t *)(bar + 2) + 112;                     // 128-B aligned
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t cand = (int64_t)blockIdx.x * 32 + lane;
    const bool ok = cand < n;
    ts_start(G, bufs, bar);
    // stage the candidate tile: warp w loads rows w, w + NW, ... (one 128-B line per row)
    for (int f = warp; f < F; f += PRED_NW) tile[f * 32 + lane] = ok ? __ldcs(X + (int64_t)f * ld + cand) : 0.0f;
    __syncthreads();
    ts_wait_resident(G, bar);
    uint32_t ph[2] = {0u, 0u};
    uint64_t c = 0;
    walk_pass<PRED_NW>(G, bufs, bar, ph, c, (uint64_t)G.NC, tile, lane, warp, part, slots, n, cand, ok);
    if (warp == 0 && ok) score[cand] = gbt_combine(part, lane, base);
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
    if (cudaMalloc(&g->d_nodes, (size_t)g->t_pad * ni * sizeof(uint2)) != cudaSuccess ||
        cudaMalloc(&g->d_leaf, (size_t)g->t_pad * nl * sizeof(float)) != cudaSuccess ||
        cudaMemset(g->d_nodes, 0, (size_t)g->t_pad * ni * sizeof(uint2)) != cudaSuccess ||
        cudaMemset(g->d_leaf, 0, (size_t)g->t_pad * nl * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(g->d_nodes);
        delete g;
        return at::fail(AT_ENOMEM, "gbt_create: device allocation failed");
    }
    cudaError_t e1 = cudaMemcpy(g->d_nodes, nodes.data(), nodes.size() * sizeof(uint2), cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(g->d_leaf, leaf, (size_t)n_trees * nl * sizeof(float), cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaFree(g->d_nodes);
        cudaFree(g->d_leaf);
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

int gbt_destroy(at_gbt g)
{
    if (!g) return AT_OK;
    cudaFree(g->d_nodes);
    cudaFree(g->d_leaf);
    delete g;
    return AT_OK;
}

int gbt_predict(at_gbt g, const float *d_feat, int64_t n, int64_t ld, float *d_score, uint8_t *d_leaf_slot,
                void *stream)
{
    if (!g) return at::fail(AT_EINVAL, "gbt_predict: null model");
    if (n < 0) return at::fail(AT_EINVAL, "gbt_predict: n < 0");
    if (n == 0) return AT_OK;
    if (!d_feat || !d_score) return at::fail(AT_EINVAL, "gbt_predict: null buffer");
    if (ld < n) return at::fail(AT_EMISMATCH, "gbt_predict: ld < n");
    cudaStream_t s = (cudaStream_t)stream;
    const at::TreeGeo G = at::make_geo(g);
    const size_t smem = ((size_t)g->n_features * 32 + 32 * 32) * sizeof(float) + 16 + at::tree_smem_bytes(G);
    if (smem > 227 * 1024) return at::fail(AT_EUNSUPPORTED, "gbt_predict: too many features for the smem tile");
    static size_t attr = 0;
    if (smem > attr) {
        AT_CUDA_TRY(cudaFuncSetAttribute(at::predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    const int64_t blocks = (n + 31) / 32;
    at::ProfScope ps(AT_K_PREDICT, s);
    at::predict_kernel<<<(unsigned)blocks, at::PRED_NW * 32, smem, s>>>(G, g->base, g->n_features, d_feat, n, ld,
                                                                       d_score, d_leaf_slot);
    AT_LAUNCH_CHECK("predict_kernel");
    return AT_OK;
}

}  // extern "C"
