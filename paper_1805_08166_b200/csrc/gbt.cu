// gbt.cu -- gbt_create / gbt_export / gbt_destroy / gbt_predict.
#include <cmath>
#include <cstring>
#include <vector>

#include "gbt.cuh"

namespace at {

constexpr int PRED_NW = 8;   // warps per block (tree slices); 32 candidates per block

__global__ void __launch_bounds__(PRED_NW * 32) predict_kernel(const uint2 *__restrict__ nodes,
                                                              const float *__restrict__ leaf, int T, int D,
                                                              float base, int F, const float *__restrict__ X,
                                                              int64_t n, int64_t ld, float *__restrict__ score,
                                                              uint8_t *__restrict__ slots)
{
    extern __shared__ float sm[];
    float *tile = sm;             // [F][32]
    float *part = sm + F * 32;    // [32][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    const int64_t cand = c0 + lane;
    const bool ok = cand < n;
    // stage the candidate tile: warp w loads rows w, w + NW, ... (one 128-B line per row)
    for (int f = warp; f < F; f += PRED_NW) tile[f * 32 + lane] = ok ? __ldcs(X + (int64_t)f * ld + cand) : 0.0f;
    __syncthreads();
    gbt_walk_partials<PRED_NW>(nodes, leaf, T, D, tile, lane, warp, part, slots, n, cand, ok);
    __syncthreads();
    if (warp == 0 && ok) score[cand] = gbt_combine(part, lane, base);
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
    g->base = base;
    g->d_nodes = nullptr;
    g->d_leaf = nullptr;
    if (cudaMalloc(&g->d_nodes, nodes.size() * sizeof(uint2)) != cudaSuccess ||
        cudaMalloc(&g->d_leaf, (size_t)n_trees * nl * sizeof(float)) != cudaSuccess) {
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
    const size_t smem = ((size_t)g->n_features * 32 + 32 * 32) * sizeof(float);
    if (smem > 227 * 1024) return at::fail(AT_EUNSUPPORTED, "gbt_predict: too many features for the smem tile");
    static size_t attr = 0;
    if (smem > attr) {
        AT_CUDA_TRY(cudaFuncSetAttribute(at::predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
    }
    const int64_t blocks = (n + 31) / 32;
    at::ProfScope ps(AT_K_PREDICT, s);
    at::predict_kernel<<<(unsigned)blocks, at::PRED_NW * 32, smem, s>>>(g->d_nodes, g->d_leaf, g->n_trees, g->depth,
                                                                       g->base, g->n_features, d_feat, n, ld,
                                                                       d_score, d_leaf_slot);
    AT_LAUNCH_CHECK("predict_kernel");
    return AT_OK;
}

}  // extern "C"
