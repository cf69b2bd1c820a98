// features.cu -- features_extract: one thread per candidate, SoA [468][ld] fp32 output.
// Context columns are stored straight to HBM (each warp store = 32 consecutive floats,
// one 128-B line); the 120 relation columns, whose order of production is
// data-dependent, are staged in shared memory [120][BLOCK] (bank = thread) and then
// written out as coalesced rows.
#include "features.cuh"

namespace at {

constexpr int FEAT_BLOCK = 128;

struct GlobalSink {
    float *__restrict__ out;
    int64_t ld;
    int64_t i;
    float *stage;
    int tid;
    __device__ __forceinline__ void put(int f, float v) { __stcs(out + (int64_t)f * ld + i, v); }
    __device__ __forceinline__ void put_rel(int f, float v) { stage[(f - 342) * FEAT_BLOCK + tid] = v; }
};

__global__ void __launch_bounds__(FEAT_BLOCK) features_kernel(const SpaceDev *__restrict__ S,
                                                             const uint16_t *__restrict__ fact,
                                                             const uint64_t *__restrict__ idx, int64_t n,
                                                             float *__restrict__ out, int64_t ld)
{
    extern __shared__ float stage[];
    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.x * FEAT_BLOCK + tid;
    if (i >= n) return;
    const uint64_t g = __ldg(idx + i);
    const int nw = S->n_w;
    int w = 0;
    for (int q = 1; q < nw; ++q)
        if (g >= S->offset[q]) w = q;
    const WlDev &W = S->w[w];
    uint32_t local = (uint32_t)(g - S->offset[w]);
    if (g >= S->offset[nw]) {   // outside the space: clamped, reported as AT_ERANGE
        flag_range(S);
        local = 0;
    }
    uint32_t ch[MAXKNOBS];
    GlobalSink sk{out, ld, i, stage, tid};
    switch (W.tmpl) {
    case 0:
        decode_knobs<0>(W, local, ch);
        features_zero_cols<0>(sk);
        features_one<0>(W, fact, ch, sk);
        break;
    case 1:
        decode_knobs<1>(W, local, ch);
        features_zero_cols<1>(sk);
        features_one<1>(W, fact, ch, sk);
        break;
    default:
        decode_knobs<2>(W, local, ch);
        features_zero_cols<2>(sk);
        features_one<2>(W, fact, ch, sk);
        break;
    }
#pragma unroll 8
    for (int r = 0; r < 120; ++r) __stcs(out + (int64_t)(342 + r) * ld + i, stage[r * FEAT_BLOCK + tid]);
}

// Configuration features (reading Q44): per knob in knob order, a split knob's factor
// tuple (outer first), the reorder index, the unroll max-step value, the vectorize flag; fp32, SoA
// [AT_KNOB_FEATURES][ld], zero padded.  One thread per candidate, coalesced column stores.
template <int TMPL>
__device__ __forceinline__ int knob_columns(const WlDev &W, const uint16_t *__restrict__ fact, const uint32_t *ch,
                                            float *__restrict__ out, int64_t ld, int64_t i)
{
    int c = 0;
    constexpr int NS = TMPL == 0 ? 3 : TMPL == 1 ? 6 : 5;   // split knobs come first (axes 0 .. NS-1)
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        const int Lv = TMPL == 0 ? (j == 2 ? 2 : 3) : (j < 3 ? 4 : 2);
#pragma unroll
        for (int l = 0; l < Lv; ++l)
            __stcs(out + (int64_t)(c + l) * ld + i, __uint2float_rn(__ldg(fact + W.fact_off[j] + ch[j] * (uint32_t)Lv + l)));
        c += Lv;
    }
    if (TMPL == 0) {
        __stcs(out + (int64_t)c++ * ld + i, __uint2float_rn(W.unroll_vals[ch[3]]));
    } else {
        __stcs(out + (int64_t)c++ * ld + i, __uint2float_rn(ch[NS]));                       // reorder
        __stcs(out + (int64_t)c++ * ld + i, __uint2float_rn(W.unroll_vals[ch[NS + 1]]));    // unroll
        __stcs(out + (int64_t)c++ * ld + i, __uint2float_rn(ch[NS + 2]));                   // vectorize
    }
    return c;
}

__global__ void __launch_bounds__(256) knob_features_kernel(const SpaceDev *__restrict__ S,
                                                            const uint16_t *__restrict__ fact,
                                                            const uint64_t *__restrict__ idx, int64_t n,
                                                            float *__restrict__ out, int64_t ld)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t g = __ldg(idx + i);
    int w = 0;
    for (int q = 1; q < S->n_w; ++q)
        if (g >= S->offset[q]) w = q;
    const WlDev &W = S->w[w];
    uint32_t local = (uint32_t)(g - S->offset[w]);
    if (g >= S->offset[S->n_w]) {   // outside the space: clamped, reported as AT_ERANGE
        flag_range(S);
        local = 0;
    }
    uint32_t ch[MAXKNOBS];
    int c;
    switch (W.tmpl) {
    case 0: decode_knobs<0>(W, local, ch); c = knob_columns<0>(W, fact, ch, out, ld, i); break;
    case 1: decode_knobs<1>(W, local, ch); c = knob_columns<1>(W, fact, ch, out, ld, i); break;
    default: decode_knobs<2>(W, local, ch); c = knob_columns<2>(W, fact, ch, out, ld, i); break;
    }
    for (; c < AT_KNOB_FEATURES; ++c) __stcs(out + (int64_t)c * ld + i, 0.0f);
}

}  // namespace at

extern "C" int features_knobs(at_space sp, const uint64_t *d_idx, int64_t n, float *d_feat, int64_t ld, void *stream)
{
    if (!sp) return at::fail(AT_EINVAL, "features_knobs: null space");
    if (int rc = at::take_range_error(sp)) return rc;
    if (n < 0) return at::fail(AT_EINVAL, "features_knobs: n < 0");
    if (n == 0) return AT_OK;
    if (!d_idx || !d_feat) return at::fail(AT_EINVAL, "features_knobs: null buffer");
    if (ld < n) return at::fail(AT_EMISMATCH, "features_knobs: ld < n");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t blocks = (n + 255) / 256;
    if (blocks > 0x7FFFFFFF) return at::fail(AT_EUNSUPPORTED, "features_knobs: n too large for one launch");
    at::ProfScope ps(AT_K_FEATURES, s);
    at::knob_features_kernel<<<(unsigned)blocks, 256, 0, s>>>(sp->d_space, sp->d_fact, d_idx, n, d_feat, ld);
    at::note_launch();
    AT_LAUNCH_CHECK("knob_features_kernel");
    return AT_OK;
}

extern "C" int features_extract(at_space sp, const uint64_t *d_idx, int64_t n, float *d_feat, int64_t ld,
                                void *stream)
{
    if (!sp) return at::fail(AT_EINVAL, "features_extract: null space");
    if (int rc = at::take_range_error(sp)) return rc;
    if (n < 0) return at::fail(AT_EINVAL, "features_extract: n < 0");
    if (n == 0) return AT_OK;
    if (!d_idx || !d_feat) return at::fail(AT_EINVAL, "features_extract: null buffer");
    if (ld < n || ld % 4 != 0) return at::fail(AT_EMISMATCH, "features_extract: need ld >= n and ld % 4 == 0");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t smem = 120 * at::FEAT_BLOCK * sizeof(float);
    static bool attr = false;
    if (!attr) {
        AT_CUDA_TRY(cudaFuncSetAttribute(at::features_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int64_t blocks = (n + at::FEAT_BLOCK - 1) / at::FEAT_BLOCK;
    if (blocks > 0x7FFFFFFF) return at::fail(AT_EUNSUPPORTED, "features_extract: n too large for one launch");
    at::ProfScope ps(AT_K_FEATURES, s);
    at::features_kernel<<<(unsigned)blocks, at::FEAT_BLOCK, smem, s>>>(sp->d_space, sp->d_fact, d_idx, n, d_feat, ld); at::note_launch();
    AT_LAUNCH_CHECK("features_kernel");
    return AT_OK;
}
