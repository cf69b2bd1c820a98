// select.cu -- select_topk: diversity-aware greedy (Eq. 3) + epsilon-greedy random
// picks (Alg. 1); readings Q24-Q27.
//
// One block.  The pool (<= 1024 entries) and each entry's knob vector live in shared
// memory; the knob-value coverage of the selected set is a bitset per knob.  Each
// greedy pick is a block-wide argmax of gain = -z + alpha * newcov with the total
// order (gain desc, z asc, idx asc), so the pick does not depend on thread mapping.
// The standardisation (mean, std over the pool, fp64) and the random picks are
// inherently sequential and run on thread 0 in the prescribed order.
#include "at_common.cuh"

namespace at {

constexpr int SEL_THREADS = 256;
constexpr int SEL_MAXPOOL = 1024;
constexpr int COV_WORDS = 9;   // radix <= 288 per knob

struct Cand {
    double gain, z;
    uint64_t idx;
    int i;
};

__device__ __forceinline__ bool better(const Cand &a, const Cand &b)
{
    if (a.i < 0) return false;
    if (b.i < 0) return true;
    if (a.gain != b.gain) return a.gain > b.gain;
    if (a.z != b.z) return a.z < b.z;
    return a.idx < b.idx;
}

__device__ __forceinline__ bool sorted_has(const uint64_t *a, int64_t n, uint64_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == v;
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t *a, int64_t n, uint64_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(SEL_THREADS) select_kernel(const SpaceDev *__restrict__ S, int w0,
                                                            const uint64_t *__restrict__ pool_idx,
                                                            const float *__restrict__ pool_E, int n_pool_max,
                                                            int64_t pool_stride, const int32_t *__restrict__ d_pool_n,
                                                            const uint64_t *__restrict__ measured,
                                                            int64_t n_measured, int b, float eps, float alpha,
                                                            uint64_t seed, uint32_t round,
                                                            uint64_t *__restrict__ out, int64_t out_stride,
                                                            int32_t *__restrict__ out_n)
{
    __shared__ uint64_t s_idx[SEL_MAXPOOL];
    __shared__ double s_z[SEL_MAXPOOL];
    __shared__ uint16_t s_ch[SEL_MAXPOOL][MAXKNOBS];
    __shared__ unsigned char s_chosen[SEL_MAXPOOL];
    __shared__ uint32_t s_cov[MAXKNOBS][COV_WORDS];
    __shared__ Cand s_red[SEL_THREADS / 32];
    __shared__ double s_mu, s_sigma;
    __shared__ int s_cnt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // block q selects for workload w0 + q from its own pool (select_topk_batch: one launch for every
    // workload; select_topk: one block)
    const int q = blockIdx.x, w = w0 + q;
    pool_idx += (int64_t)q * pool_stride;
    pool_E += (int64_t)q * pool_stride;
    out += (int64_t)q * out_stride;
    out_n += q;
    int n_pool = n_pool_max;
    if (d_pool_n) n_pool = max(0, min(n_pool_max, d_pool_n[q]));
    const WlDev &W = S->w[w];
    const int nk = W.n_knobs;
    for (int i = tid; i < n_pool; i += SEL_THREADS) {
        const uint64_t gi = pool_idx[i];
        s_idx[i] = gi;
        s_chosen[i] = 0;
        uint32_t local = (uint32_t)(gi - W.offset);
        if (gi < W.offset || gi - W.offset >= W.size) {   // not in this workload: never picked, AT_ERANGE
            flag_range(S);
            s_chosen[i] = 1;
            local = 0;
        }
        for (int j = 0; j < MAXKNOBS; ++j) {
            if (j < nk) {
                const uint32_t q = local / W.radix[j];
                s_ch[i][j] = (uint16_t)(local - q * W.radix[j]);
                local = q;
            } else {
                s_ch[i][j] = 0;
            }
        }
    }
    for (int i = tid; i < MAXKNOBS * COV_WORDS; i += SEL_THREADS) (&s_cov[0][0])[i] = 0;
    if (tid == 0) {
        // standardised scores: fp64, sequential in pool order (reading Q24/Q27)
        double mu = 0.0, var = 0.0;
        for (int i = 0; i < n_pool; ++i) mu = mu + (double)pool_E[i];
        if (n_pool > 0) mu = mu / (double)n_pool;
        for (int i = 0; i < n_pool; ++i) {
            const double dd = (double)pool_E[i] - mu;
            var = var + dd * dd;
        }
        if (n_pool > 0) var = var / (double)n_pool;
        double sg = sqrt(var);
        if (sg == 0.0) sg = 1.0;
        s_mu = mu;
        s_sigma = sg;
        s_cnt = 0;
    }
    __syncthreads();
    for (int i = tid; i < n_pool; i += SEL_THREADS) s_z[i] = ((double)pool_E[i] - s_mu) / s_sigma;
    __syncthreads();

    int n_rand = (int)ceilf(__fmul_rn(eps, (float)b));   // Q26: ceil of the fp32 product
    if (n_rand > b) n_rand = b;
    const int n_g = b - n_rand;
    const int greedy = n_g < n_pool ? n_g : n_pool;
    for (int pick = 0; pick < greedy; ++pick) {
        Cand best{0.0, 0.0, 0, -1};
        for (int i = tid; i < n_pool; i += SEL_THREADS) {
            if (s_chosen[i]) continue;
            int newcov = 0;
            for (int j = 0; j < nk; ++j) {
                const uint32_t v = s_ch[i][j];
                newcov += ((s_cov[j][v >> 5] >> (v & 31)) & 1u) ? 0 : 1;
            }
            Cand c{(-s_z[i]) + (double)alpha * (double)newcov, s_z[i], s_idx[i], i};
            if (better(c, best)) best = c;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            Cand o;
            o.gain = __shfl_xor_sync(0xFFFFFFFFu, best.gain, off);
            o.z = __shfl_xor_sync(0xFFFFFFFFu, best.z, off);
            o.idx = __shfl_xor_sync(0xFFFFFFFFu, best.idx, off);
            o.i = __shfl_xor_sync(0xFFFFFFFFu, best.i, off);
            if (better(o, best)) best = o;
        }
        if (lane == 0) s_red[warp] = best;
        __syncthreads();
        if (tid == 0) {
            Cand bb = s_red[0];
            for (int q = 1; q < SEL_THREADS / 32; ++q)
                if (better(s_red[q], bb)) bb = s_red[q];
            if (bb.i >= 0) {   // (none left only when invalid pool entries were excluded)
                s_chosen[bb.i] = 1;
                out[s_cnt++] = bb.idx;
                for (int j = 0; j < nk; ++j) {
                    const uint32_t v = s_ch[bb.i][j];
                    s_cov[j][v >> 5] |= 1u << (v & 31);
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        // random picks uniformly over S_w, never measured, never selected (reading Q25)
        int cnt = s_cnt;
        const uint64_t lo = W.offset, size = W.size;
        const uint64_t n_meas_w = (uint64_t)(lower_bound(measured, n_measured, lo + size) -
                                             lower_bound(measured, n_measured, lo));
        for (uint32_t p = 0; cnt < b; ++p) {
            if (size - n_meas_w - (uint64_t)cnt == 0) break;
            uint64_t cand = 0;
            bool ok = false;
            for (uint32_t a = 0; a < 1024 && !ok; ++a) {
                const U4 r = philox(seed, p, a, round, TAG_EPS);
                cand = lo + mulhi64((uint64_t)r.x | ((uint64_t)r.y << 32), size);
                bool taken = n_measured && sorted_has(measured, n_measured, cand);
                for (int q = 0; q < cnt && !taken; ++q) taken = out[q] == cand;
                ok = !taken;
            }
            while (!ok) {
                cand = lo + ((cand - lo + 1) % size);
                bool taken = n_measured && sorted_has(measured, n_measured, cand);
                for (int q = 0; q < cnt && !taken; ++q) taken = out[q] == cand;
                ok = !taken;
            }
            out[cnt++] = cand;
        }
        *out_n = cnt;
    }
}

}  // namespace at

extern "C" int select_topk(at_space sp, int32_t workload, const uint64_t *d_pool_idx, const float *d_pool_score,
                           int64_t n_pool, const uint64_t *d_measured_sorted, int64_t n_measured,
                           const at_select_opts *o, uint64_t *d_out_idx, int32_t *d_out_n, void *stream)
{
    if (!sp || !o || !d_out_idx || !d_out_n) return at::fail(AT_EINVAL, "select_topk: null pointer");
    if (int rc = at::take_range_error(sp)) return rc;
    if (workload < 0 || workload >= sp->host.n_w) return at::fail(AT_ERANGE, "select_topk: workload out of range");
    if (n_pool < 0 || n_pool > at::SEL_MAXPOOL) return at::fail(AT_EUNSUPPORTED, "select_topk: pool must hold <= 1024");
    if (n_pool > 0 && (!d_pool_idx || !d_pool_score)) return at::fail(AT_EINVAL, "select_topk: null pool");
    if (o->b < 0 || !(o->eps >= 0.0f && o->eps <= 1.0f)) return at::fail(AT_EINVAL, "select_topk: need b >= 0, 0 <= eps <= 1");
    if (n_measured < 0 || (n_measured > 0 && !d_measured_sorted)) return at::fail(AT_EINVAL, "select_topk: bad measured list");
    for (int j = 0; j < sp->host.w[workload].n_knobs; ++j)
        if (sp->host.w[workload].radix[j] > 32 * at::COV_WORDS)
            return at::fail(AT_EUNSUPPORTED, "select_topk: knob radix > 288");
    cudaStream_t s = (cudaStream_t)stream;
    at::ProfScope ps(AT_K_SELECT, s);
    at::select_kernel<<<1, at::SEL_THREADS, 0, s>>>(sp->d_space, workload, d_pool_idx, d_pool_score, (int)n_pool, 0,
                                                    nullptr, d_measured_sorted, n_measured, o->b, o->eps, o->alpha,
                                                    o->seed, o->round, d_out_idx, 0, d_out_n); at::note_launch();
    AT_LAUNCH_CHECK("select_kernel");
    return AT_OK;
}

extern "C" int select_topk_batch(at_space sp, int32_t w0, int32_t n_w, const uint64_t *d_pool_idx,
                                 const float *d_pool_score, int64_t pool_stride, const int32_t *d_pool_n,
                                 int64_t n_pool_max, const uint64_t *d_measured_sorted, int64_t n_measured,
                                 const at_select_opts *o, uint64_t *d_out_idx, int32_t *d_out_n, void *stream)
{
    if (!sp || !o || !d_out_idx || !d_out_n) return at::fail(AT_EINVAL, "select_topk_batch: null pointer");
    if (int rc = at::take_range_error(sp)) return rc;
    if (n_w < 1 || w0 < 0 || w0 + n_w > sp->host.n_w) return at::fail(AT_ERANGE, "select_topk_batch: workloads out of range");
    if (n_pool_max < 0 || n_pool_max > at::SEL_MAXPOOL) return at::fail(AT_EUNSUPPORTED, "select_topk_batch: pools must hold <= 1024");
    if (pool_stride < n_pool_max) return at::fail(AT_EMISMATCH, "select_topk_batch: pool_stride < n_pool_max");
    if (n_pool_max > 0 && (!d_pool_idx || !d_pool_score)) return at::fail(AT_EINVAL, "select_topk_batch: null pools");
    if (o->b < 0 || !(o->eps >= 0.0f && o->eps <= 1.0f)) return at::fail(AT_EINVAL, "select_topk_batch: need b >= 0, 0 <= eps <= 1");
    if (n_measured < 0 || (n_measured > 0 && !d_measured_sorted)) return at::fail(AT_EINVAL, "select_topk_batch: bad measured list");
    for (int q = w0; q < w0 + n_w; ++q)
        for (int j = 0; j < sp->host.w[q].n_knobs; ++j)
            if (sp->host.w[q].radix[j] > 32 * at::COV_WORDS)
                return at::fail(AT_EUNSUPPORTED, "select_topk_batch: knob radix > 288");
    cudaStream_t s = (cudaStream_t)stream;
    at::ProfScope ps(AT_K_SELECT, s);
    at::select_kernel<<<n_w, at::SEL_THREADS, 0, s>>>(sp->d_space, w0, d_pool_idx, d_pool_score, (int)n_pool_max,
                                                      pool_stride, d_pool_n, d_measured_sorted, n_measured, o->b, o->eps,
                                                      o->alpha, o->seed, o->round, d_out_idx, o->b > 0 ? o->b : 1, d_out_n);
    at::note_launch();
    AT_LAUNCH_CHECK("select_kernel (batch)");
    return AT_OK;
}
