// fit.cu -- gbt_fit_hist: histogram GBT refit under the pairwise rank loss
// (Alg. 1 P:163 "update f-hat using D"; Eq. 2; readings Q16, Q17, Q34-Q37).
//
// Pipeline (all on `stream`, one process per GPU, histograms summed across ranks by
// the caller's all-reduce between levels):
//   1. cuts: per feature an LSD radix sort (4 x 8-bit passes, one block per feature,
//      stable warp-match ranking) of the order-preserving u32 keys, then the unique
//      values (<= max_bins) or the max_bins-quantile order statistics;  bins u8 [F][n].
//   2. per-workload dense ranks and group tables (once per fit).
//   3. per tree: Feistel/Philox positions -> group members; one block per group of
//      <= 64 computes both orders of every pair's Eq. 2 gradient / curvature, quantised
//      to int64 2^-32 fixed point (order-free sums -> bit-identical at any rank count);
//      per level: int64 histograms [node][F][bins] of the rank's sample slice
//      (shared-memory atomics, one block per feature), all-reduce, fp64 split search
//      (one block per node), partition of every sample; leaves -eta G / (H + lambda);
//      fp32 prediction update in tree order.
#include <algorithm>
#include <cmath>
#include <vector>

#include "at_common.cuh"

namespace at {

constexpr int FIT_MAXKEYS = 1024;
constexpr double FX = 1.0 / 4294967296.0;   // 2^-32

// ------------------------------------------------------------------ 1. cuts
__global__ void __launch_bounds__(1024) sort_feature_kernel(const float *__restrict__ X, int64_t ld, int64_t n,
                                                            uint32_t *__restrict__ bufA, uint32_t *__restrict__ bufB)
{
    __shared__ uint32_t wcount[32][257];
    __shared__ uint32_t base[256];
    __shared__ uint32_t tile_total[256];
    __shared__ int s_skip;
    const int f = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *src = bufA + (int64_t)f * n, *dst = bufB + (int64_t)f * n;
    for (int64_t i = tid; i < n; i += 1024) src[i] = fkey(X[(int64_t)f * ld + i]);
    if (tid == 0) s_skip = 0;
    __syncthreads();
    for (int pass = 0; pass < 4; ++pass) {
        const int sh = 8 * pass;
        if (tid < 256) base[tid] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += 1024) atomicAdd(&base[(src[i] >> sh) & 255u], 1u);
        __syncthreads();
        // a digit shared by every key (small integers have all-zero low mantissa bytes): the pass
        // would be the identity permutation, skip it
        if (tid < 256 && base[tid] == (uint32_t)n) s_skip = 1;
        __syncthreads();
        if (s_skip) {
            __syncthreads();
            if (tid == 0) s_skip = 0;
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            uint32_t run = 0;
            for (int d = 0; d < 256; ++d) { const uint32_t c = base[d]; base[d] = run; run += c; }
        }
        __syncthreads();
        for (int64_t t0 = 0; t0 < n; t0 += 1024) {
            for (int q = tid; q < 32 * 257; q += 1024) (&wcount[0][0])[q] = 0;
            __syncthreads();
            const int64_t i = t0 + tid;
            const bool ok = i < n;
            const uint32_t key = ok ? src[i] : 0u;
            const uint32_t dg = ok ? ((key >> sh) & 255u) : 256u;
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dg);
            const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            if (ok && rank == 0) wcount[warp][dg] = __popc(peers);
            __syncthreads();
            if (tid < 256) {
                uint32_t run = 0;
                for (int w = 0; w < 32; ++w) { const uint32_t c = wcount[w][tid]; wcount[w][tid] = run; run += c; }
                tile_total[tid] = run;
            }
            __syncthreads();
            if (ok) dst[base[dg] + wcount[warp][dg] + rank] = key;
            __syncthreads();
            if (tid < 256) base[tid] += tile_total[tid];
            __syncthreads();
        }
        uint32_t *t = src; src = dst; dst = t;
        __syncthreads();
    }
    // an odd number of performed passes leaves the sorted keys in bufB: the caller reads bufA
    if (src != bufA + (int64_t)f * n)
        for (int64_t i = tid; i < n; i += 1024) bufA[(int64_t)f * n + i] = src[i];
}

__global__ void __launch_bounds__(1024) cuts_kernel(const uint32_t *__restrict__ sorted, int64_t n, int B,
                                                    float *__restrict__ cuts, int32_t *__restrict__ ncuts)
{
    __shared__ int64_t wsum[32];
    __shared__ int64_t s_run;
    __shared__ int64_t s_U;
    const int f = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t *k = sorted + (int64_t)f * n;
    float *c = cuts + (int64_t)f * (B - 1);
    // number of unique values U
    int64_t cnt = 0;
    for (int64_t i = tid; i < n; i += 1024) cnt += (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
    if (lane == 0) wsum[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
        int64_t U = 0;
        for (int w = 0; w < 32; ++w) U += wsum[w];
        s_U = U;
        s_run = 0;
    }
    __syncthreads();
    const int64_t U = s_U;
    if (U <= B) {
        // cuts = u_2 .. u_U: the unique values in order, without the minimum
        for (int64_t t0 = 0; t0 < n; t0 += 1024) {
            const int64_t i = t0 + tid;
            const int flag = (i < n && (i == 0 || k[i] != k[i - 1])) ? 1 : 0;
            int incl = flag;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += y;
            }
            __syncthreads();
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            if (tid == 0) {
                int64_t r = 0;
                for (int w = 0; w < 32; ++w) { const int64_t x = wsum[w]; wsum[w] = r; r += x; }
            }
            __syncthreads();
            const int64_t before = s_run + wsum[warp] + incl - flag;   // uniques in [0, i)
            if (flag && i > 0) c[before - 1] = fkey_inv(k[i]);
            __syncthreads();
            if (tid == 1023) s_run = before + flag;
            __syncthreads();
        }
        if (tid == 0) ncuts[f] = (int32_t)(U - 1);
    } else if (tid == 0) {
        int nc = 0;
        for (int q = 0; q < B - 1; ++q) {
            const uint32_t v = k[((int64_t)(q + 1) * n) / B];
            if (v == k[0]) continue;
            if (nc > 0 && fkey(c[nc - 1]) == v) continue;
            c[nc++] = fkey_inv(v);
        }
        ncuts[f] = nc;
    }
}

__global__ void bins_kernel(const float *__restrict__ X, int64_t ld, int64_t n, int F, int B,
                            const float *__restrict__ cuts, const int32_t *__restrict__ ncuts,
                            uint8_t *__restrict__ bins)
{
    const int f = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = X[(int64_t)f * ld + i];
    const float *c = cuts + (int64_t)f * (B - 1);
    int lo = 0, hi = ncuts[f];   // upper_bound: number of cuts <= x
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (c[mid] <= x) lo = mid + 1; else hi = mid;
    }
    bins[(int64_t)f * n + i] = (uint8_t)lo;
}

// ------------------------------------------------------------------ 2. groups
// rank[i] = #{j < i : key[j] = key[i]} (the sample's position among its workload's samples, index
// order), counts, their exclusive prefix woff, and the group prefix gprefix.  Three passes so the
// 10^5-sample case is not one block: (1) per 1024-sample block, block-local ranks (warps in order)
// and the block's key counts bc[b][k]; (2) one thread per key turns bc into exclusive offsets over the
// blocks and builds the prefixes; (3) rank += the block's offset for the key.
__global__ void __launch_bounds__(1024) ranks_local_kernel(const uint16_t *__restrict__ key, int64_t n,
                                                           int32_t *__restrict__ rank, int32_t *__restrict__ bc)
{
    __shared__ int32_t cnt[FIT_MAXKEYS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    cnt[tid] = 0;   // FIT_MAXKEYS == blockDim.x
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * 1024 + tid;
    const bool ok = i < n && key[i] < FIT_MAXKEYS;   // a bad key is reported by key_check_kernel
    const uint32_t k = ok ? (uint32_t)key[i] : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, k);
    const int r = __popc(peers & ((1u << lane) - 1u));
    for (int w = 0; w < 32; ++w) {
        if (warp == w && ok) {
            rank[i] = cnt[k] + r;
            __syncwarp(peers);
            if (r == 0) cnt[k] += __popc(peers);
        }
        __syncthreads();
    }
    bc[(int64_t)blockIdx.x * FIT_MAXKEYS + tid] = cnt[tid];
}

__global__ void __launch_bounds__(1024) ranks_scan_kernel(int nb, int32_t *__restrict__ bc,
                                                          int32_t *__restrict__ counts, int32_t *__restrict__ woff,
                                                          int32_t *__restrict__ gprefix, int group_size)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = tid;   // FIT_MAXKEYS == 1024 == blockDim.x
    int32_t c = 0;
    for (int b = 0; b < nb; ++b) {   // exclusive offsets of key k over the blocks (coalesced over k)
        const int32_t x = bc[(int64_t)b * FIT_MAXKEYS + k];
        bc[(int64_t)b * FIT_MAXKEYS + k] = c;
        c += x;
    }
    // exclusive prefix sums of the counts and of the group counts over the FIT_MAXKEYS keys: one key
    // per thread, warp shuffles + one shared pass over the warp totals
    __shared__ int32_t wo[32], wg[32];
    const int32_t gk = (c + group_size - 1) / group_size;
    int32_t xo = c, xg = gk;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int32_t yo = __shfl_up_sync(0xFFFFFFFFu, xo, off), yg = __shfl_up_sync(0xFFFFFFFFu, xg, off);
        if (lane >= off) { xo += yo; xg += yg; }
    }
    if (lane == 31) { wo[warp] = xo; wg[warp] = xg; }
    __syncthreads();
    if (warp == 0) {
        int32_t a = wo[lane], b = wg[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t ya = __shfl_up_sync(0xFFFFFFFFu, a, off), yb = __shfl_up_sync(0xFFFFFFFFu, b, off);
            if (lane >= off) { a += ya; b += yb; }
        }
        wo[lane] = a - wo[lane];
        wg[lane] = b - wg[lane];
    }
    __syncthreads();
    counts[k] = c;
    woff[k] = wo[warp] + xo - c;
    gprefix[k] = wg[warp] + xg - gk;
    if (k == FIT_MAXKEYS - 1) gprefix[FIT_MAXKEYS] = wg[warp] + xg;
}

__global__ void ranks_add_kernel(const uint16_t *__restrict__ key, int64_t n, const int32_t *__restrict__ bc,
                                 int32_t *__restrict__ rank)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && key[i] < FIT_MAXKEYS) rank[i] += bc[(i >> 10) * FIT_MAXKEYS + key[i]];
}

__device__ __forceinline__ uint32_t feistel(uint32_t x, int h, uint64_t seed, uint32_t tree, uint32_t wkey)
{
    const uint32_t mask = (1u << h) - 1u;
    uint32_t L = x >> h, R = x & mask;
#pragma unroll
    for (uint32_t r = 0; r < 4; ++r) {
        const U4 o = philox(seed, R, tree, (wkey << 2) | r, TAG_GROUP_PERM);
        const uint32_t nL = R, nR = L ^ (o.x & mask);
        L = nL;
        R = nR;
    }
    return (L << h) | R;
}

__global__ void positions_kernel(const uint16_t *__restrict__ key, const int32_t *__restrict__ rank,
                                 const int32_t *__restrict__ counts, const int32_t *__restrict__ woff, int64_t n,
                                 uint64_t seed, uint32_t tree, int32_t *__restrict__ member,
                                 const int32_t *__restrict__ d_tree = nullptr)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (d_tree) tree = (uint32_t)*d_tree;   // per-tree graph: the tree index lives on the device
    const uint32_t k = key[i];
    const uint32_t nw = (uint32_t)counts[k];
    int bits = 0;
    while ((1ull << bits) < nw) ++bits;
    int h = (bits + 1) / 2;
    if (h < 1) h = 1;
    uint32_t y = feistel((uint32_t)rank[i], h, seed, tree, k);
    while (y >= nw) y = feistel(y, h, seed, tree, k);
    member[woff[k] + y] = (int32_t)i;
}

// One pair's Eq. 2 contribution to member a (cost ca, prediction fa) from partner (cc, fc), both
// orders of the pair, quantised to 2^-32 fixed point.
__device__ __forceinline__ void pair_term(float ca, float fa, float cc, float fc, long long &ga, long long &ha)
{
    if (cc == ca) return;                   // sign(c_i - c_j) = 0 contributes nothing
    const bool hi = ca > cc;                // a is the slower (i) of the pair
    const float fi = hi ? fa : fc, fj = hi ? fc : fa;
    const float d = __fsub_rn(fj, fi);
    const float e = exp_det(-d);
    const float rho = __fdiv_rn(1.0f, __fadd_rn(1.0f, e));
    const float hh = __fmul_rn(rho, __fsub_rn(1.0f, rho));
    const long long q = __double2ll_rn((double)rho * 4294967296.0);
    const long long qh = __double2ll_rn((double)hh * 4294967296.0);
    ga += hi ? -2 * q : 2 * q;              // both orders of Eq. 2 carry the same term
    ha += 2 * qh;
}

// Eq. 2 gradients of one group (members mem[0..m), costs sc[], predictions sp[] in shared memory),
// written to g[mem[a]], h[mem[a]].  SUB threads per member: thread (a, r) accumulates member a's
// share of its pairs with members c = r (mod SUB) (no atomics; each pair's rho is computed
// identically by both members), the SUB partial int64 sums are then added with xor shuffles
// (exact, order-free).
__device__ __forceinline__ void group_pair_grads(const int32_t *mem, int m, const float *sc, const float *sp,
                                                 int64_t *__restrict__ g, int64_t *__restrict__ h)
{
    constexpr int SUB = 4;
    for (int base = 0; base < m * SUB; base += blockDim.x) {
        const int tix = base + (int)threadIdx.x;
        const int a = tix / SUB, r = tix % SUB;
        long long ga = 0, ha = 0;
        if (a < m) {
            const float ca = sc[a], fa = sp[a];
            for (int c = r; c < m; c += SUB)
                if (c != a) pair_term(ca, fa, sc[c], sp[c], ga, ha);
        }
#pragma unroll
        for (int off = 1; off < SUB; off <<= 1) {
            ga += __shfl_xor_sync(0xFFFFFFFFu, ga, off);
            ha += __shfl_xor_sync(0xFFFFFFFFu, ha, off);
        }
        if (a < m && r == 0) {
            g[mem[a]] = ga;
            h[mem[a]] = ha;
        }
    }
}

__global__ void __launch_bounds__(256) grads_kernel(const int32_t *__restrict__ member,
                                                    const int32_t *__restrict__ counts,
                                                    const int32_t *__restrict__ woff,
                                                    const int32_t *__restrict__ gprefix, int group_size,
                                                    const float *__restrict__ cost, const float *__restrict__ pred,
                                                    int64_t *__restrict__ g, int64_t *__restrict__ h)
{
    extern __shared__ unsigned char smraw[];
    float *sc = (float *)smraw;
    float *sp = sc + group_size;
    __shared__ int s_w;
    const int b = blockIdx.x;
    if (b >= gprefix[FIT_MAXKEYS]) return;   // grids sized by an upper bound of the group count
    if (threadIdx.x == 0) {
        int lo = 0, hi = FIT_MAXKEYS;   // largest w with gprefix[w] <= b
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (gprefix[mid] <= b) lo = mid; else hi = mid;
        }
        s_w = lo;
    }
    __syncthreads();
    const int w = s_w;
    const int start = (b - gprefix[w]) * group_size;
    int m = counts[w] - start;
    if (m > group_size) m = group_size;
    const int32_t *mem = member + woff[w] + start;
    for (int a = threadIdx.x; a < m; a += blockDim.x) {
        const int i = mem[a];
        sc[a] = cost[i];
        sp[a] = pred[i];
    }
    __syncthreads();
    group_pair_grads(mem, m, sc, sp, g, h);
}

// Regression loss of P:175, sum_i (f_i - c_i)^2: g_i = 2 (f_i - c_i), h_i = 2 in 2^-32 fixed point
// (the difference in fp64 from the two fp32 values, one RN multiply by 2^33, round to nearest).
__device__ __forceinline__ void reg_grad(float f, float c, int64_t &g, int64_t &h)
{
    g = __double2ll_rn(2.0 * ((double)f - (double)c) * 4294967296.0);
    h = 2ll * 4294967296ll;
}

__global__ void reg_grads_kernel(const float *__restrict__ cost, const float *__restrict__ pred, int64_t n,
                                 int64_t *__restrict__ g, int64_t *__restrict__ h)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) reg_grad(pred[i], cost[i], g[i], h[i]);
}

// ------------------------------------------------------------------ 3. levels
// Histograms use a compact bin layout: feature f owns nb_f = ncuts_f + 1 cells starting at
// boff[f]; a level's buffer is hist[node][TB][2] int64 (TB = sum_f nb_f).
__global__ void bin_layout_kernel(const int32_t *__restrict__ ncuts, int F, int32_t *__restrict__ boff,
                                  int32_t *__restrict__ info /* [0] TB, [1] max nb, [4] n splittable */,
                                  int32_t *__restrict__ flist /* [F] splittable features, ascending */)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int32_t o = 0, mx = 0, nf = 0;
    for (int f = 0; f < F; ++f) {
        boff[f] = o;
        const int32_t nb = ncuts[f] + 1;
        o += nb;
        mx = nb > mx ? nb : mx;
        if (nb > 1) flist[nf++] = f;   // a feature without cuts (constant on D) can never split
    }
    boff[F] = o;
    info[0] = o;
    info[1] = mx;
    info[4] = nf;
    if (nf == 0) flist[0] = 0;   // no feature can split: one block on feature 0 (no cut) keeps every node a leaf
}

// the fit's input flags (info[2]: 1 non-finite cost, 2 group key >= 1024) -> the model's mapped error word
__global__ void fit_flag_kernel(const int32_t *__restrict__ info, uint32_t *err)
{
    *(volatile uint32_t *)err = (uint32_t)info[2];
    __threadfence_system();
}

// Exact 64-bit add into shared memory with two native 32-bit atomics (sm_100a has no native 64-bit
// shared atomic add: the 64-bit form compiles to a CAS loop).  The low word's returned old value
// tells whether this add wrapped; that carry goes into the high word with the value's high part,
// so the pair always holds the exact modular 64-bit sum, whatever the interleaving.
__device__ __forceinline__ void smem_add_u64(unsigned long long *cell, unsigned long long v)
{
    unsigned *w = (unsigned *)cell;   // little endian: w[0] low word, w[1] high word
    const unsigned lo = (unsigned)v;
    unsigned hi = (unsigned)(v >> 32);
    const unsigned old = atomicAdd(&w[0], lo);
    hi += (old + lo < old) ? 1u : 0u;
    if (hi) atomicAdd(&w[1], hi);
}

// Warp-aggregated exact int64 histogram update.  64-bit shared-memory atomics are CAS loops on
// sm_100a, so lanes hitting the same cell are first combined: peers = match_any(key); every
// lane sums its group's int64 values by walking the group's lanes with full-warp shuffles
// (trip count = the largest group, warp-uniform); the group's lowest lane does one atomic.
__device__ __forceinline__ void agg_add(unsigned long long *cells, int key, long long gv, long long hv)
{
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
    const int lane = threadIdx.x & 31;
    const int maxg = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)__popc(peers));
    long long sg = 0, sh = 0;
    unsigned m = peers;
    for (int k = 0; k < maxg; ++k) {
        const int src = m ? __ffs(m) - 1 : lane;
        const long long vg = __shfl_sync(0xFFFFFFFFu, gv, src);
        const long long vh = __shfl_sync(0xFFFFFFFFu, hv, src);
        if (m) {
            sg += vg;
            sh += vh;
            m &= m - 1;
        }
    }
    if (key >= 0 && lane == __ffs(peers) - 1) {
        smem_add_u64(&cells[2 * key], (unsigned long long)sg);
        smem_add_u64(&cells[2 * key + 1], (unsigned long long)sh);
    }
}

// grid (F, n_chunks): block (f, c) accumulates its sample chunk of the rank's slice for all nodes of
// the level in shared memory, then stores (1 chunk) or atomically adds (several chunks) into hist.
__global__ void __launch_bounds__(256) hist_kernel(const uint8_t *__restrict__ bins, const int32_t *__restrict__ node,
                                                   const int64_t *__restrict__ g, const int64_t *__restrict__ h,
                                                   int64_t hb, int64_t he, int64_t n, int64_t chunk,
                                                   const int32_t *__restrict__ boff, int TB, int first, int nn,
                                                   int use_smem, int64_t *__restrict__ hist)
{
    extern __shared__ unsigned long long shist[];
    const int f = blockIdx.x;
    const int nb = boff[f + 1] - boff[f];
    const int64_t cells = (int64_t)nn * nb * 2;
    const int64_t i0 = hb + (int64_t)blockIdx.y * chunk;
    int64_t i1 = i0 + chunk;
    if (i1 > he) i1 = he;
    const bool single = gridDim.y == 1;
    if (use_smem) {
        for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) shist[q] = 0ull;
        __syncthreads();
    }
    const uint8_t *bf = bins + (int64_t)f * n;
    for (int64_t i0w = i0; i0w < i1; i0w += blockDim.x) {
        const int64_t i = i0w + threadIdx.x;
        const bool ok = i < i1;
        const int key = ok ? (node[i] - first) * nb + bf[i] : -1;
        const long long gv = ok ? g[i] : 0, hv = ok ? h[i] : 0;
        if (use_smem) {
            agg_add(shist, key, gv, hv);   // exact: 2 x 32-bit atomics per distinct cell
        } else {
            // global cells of this feature: [node][TB] with stride TB, offset boff[f]
            const int nd = ok ? node[i] - first : 0;
            if (ok) {
                unsigned long long *cell = (unsigned long long *)(hist + ((int64_t)nd * TB + boff[f] + bf[i]) * 2);
                atomicAdd(cell, (unsigned long long)gv);
                atomicAdd(cell + 1, (unsigned long long)hv);
            }
        }
    }
    if (use_smem) {
        __syncthreads();
        for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) {
            const int64_t nd = q / (2 * nb), rem = q - nd * 2 * nb;
            int64_t *dst = hist + (nd * TB + boff[f]) * 2 + rem;
            if (single) *dst = (int64_t)shist[q];
            else if (shist[q]) atomicAdd((unsigned long long *)dst, shist[q]);
        }
    }
}

// tree 0 root histogram back to the dense [F][B][2] layout (parity hook)
__global__ void hist0_expand_kernel(const int64_t *__restrict__ hist, const int32_t *__restrict__ boff, int F, int B,
                                    int64_t *__restrict__ out, const int32_t *__restrict__ d_tree = nullptr)
{
    if (d_tree && *d_tree != 0) return;   // tree 0 only
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (int64_t)F * B) return;
    const int f = (int)(q / B), b = (int)(q - (int64_t)f * B);
    const int nb = boff[f + 1] - boff[f];
    out[2 * q] = b < nb ? hist[(int64_t)(boff[f] + b) * 2] : 0;
    out[2 * q + 1] = b < nb ? hist[(int64_t)(boff[f] + b) * 2 + 1] : 0;
}

struct SplitBest {
    double gain;
    int f, s;
};

// a before b in (gain desc, f asc, s asc); f < 0 = no split
__device__ __forceinline__ bool split_better(const SplitBest &a, const SplitBest &b)
{
    if (a.f < 0) return false;
    if (b.f < 0) return true;
    if (a.gain != b.gain) return a.gain > b.gain;
    if (a.f != b.f) return a.f < b.f;
    return a.s < b.s;
}

__device__ __forceinline__ SplitBest warp_best(SplitBest best)
{
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        SplitBest o;
        o.gain = __shfl_xor_sync(0xFFFFFFFFu, best.gain, off);
        o.f = __shfl_xor_sync(0xFFFFFFFFu, best.f, off);
        o.s = __shfl_xor_sync(0xFFFFFFFFu, best.s, off);
        if (split_better(o, best)) best = o;
    }
    return best;
}

// Best split of one (node, feature) histogram by one warp (exact int64 prefix sums by warp scans
// over 32-bin chunks, fp64 gain in the oracle's operation order).  Splits right after an empty bin repeat the previous split's (G_L, H_L) -- and its gain -- so the
// lower s wins the tie anyway; they are skipped.
template <class Cell>
__device__ __forceinline__ SplitBest scan_splits(const Cell *hf, int nb, long long Gi, long long Hi, double lam,
                                                 double mcw, int f, int lane)
{
    const int nc = nb - 1;
    const double G = (double)Gi * FX, H = (double)Hi * FX;
    const double parent = G * G / (H + lam);
    SplitBest best{0.0, -1, 0};
    long long carryG = 0, carryH = 0;
    for (int c0 = 0; c0 < nc; c0 += 32) {
        const int b = c0 + lane;   // split s = b + 1 puts bins <= b on the left
        long long vg = b < nc ? (long long)hf[2 * b] : 0, vh = b < nc ? (long long)hf[2 * b + 1] : 0;
        const long long own_g = vg, own_h = vh;
        if (__ballot_sync(0xFFFFFFFFu, vg != 0 || vh != 0) == 0) continue;   // empty chunk: carry unchanged
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long yg = __shfl_up_sync(0xFFFFFFFFu, vg, off);
            const long long yh = __shfl_up_sync(0xFFFFFFFFu, vh, off);
            if (lane >= off) { vg += yg; vh += yh; }
        }
        const long long GLi = carryG + vg, HLi = carryH + vh;
        carryG += __shfl_sync(0xFFFFFFFFu, vg, 31);
        carryH += __shfl_sync(0xFFFFFFFFu, vh, 31);
        if (b < nc && (own_g != 0 || own_h != 0)) {
            const double GL = (double)GLi * FX, HL = (double)HLi * FX;
            const double GR = (double)(Gi - GLi) * FX, HR = (double)(Hi - HLi) * FX;
            if (!(HL < mcw || HR < mcw)) {
                const double gain = (GL * GL / (HL + lam) + GR * GR / (HR + lam)) - parent;
                if (gain > 0.0) {
                    SplitBest cnd{gain, f, b + 1};
                    if (split_better(cnd, best)) best = cnd;
                }
            }
        }
    }
    return warp_best(best);
}

// single-rank fast path: block f builds the level's histograms of feature f in shared memory and
// scans its splits for every node (warp per node), so the level's histograms never touch HBM.
__global__ void __launch_bounds__(256, 4) hist_split_kernel(const uint8_t *__restrict__ bins,
                                                         const int32_t *__restrict__ node,
                                                         const int64_t *__restrict__ g, const int64_t *__restrict__ h,
                                                         int64_t n, const int32_t *__restrict__ boff, int F, int first,
                                                         int nn, double lam, double mcw,
                                                         uint8_t *__restrict__ dead,
                                                         double *__restrict__ best_gain, int32_t *__restrict__ best_s,
                                                         int64_t *__restrict__ hist0)
{
    extern __shared__ unsigned long long shist[];
    const int f = blockIdx.x;
    const int nb = boff[f + 1] - boff[f];
    const int64_t cells = (int64_t)nn * nb * 2;
    for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) shist[q] = 0ull;
    __syncthreads();
    const uint8_t *bf = bins + (int64_t)f * n;
    // samples in batches of 4 per thread: all loads of a batch are issued before any aggregation
    for (int64_t i0w = 0; i0w < n; i0w += 4 * (int64_t)blockDim.x) {
        int key[4];
        long long gv[4], hv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0w + u * (int64_t)blockDim.x + threadIdx.x;
            const bool ok = i < n;
            key[u] = ok ? (node[i] - first) * nb + bf[i] : -1;
            gv[u] = ok ? g[i] : 0;
            hv[u] = ok ? h[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) agg_add(shist, key[u], gv[u], hv[u]);
    }
    __syncthreads();
    if (hist0)
        for (int64_t q = threadIdx.x; q < cells; q += blockDim.x) hist0[(int64_t)boff[f] * 2 + q] = (int64_t)shist[q];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = warp; q < nn; q += blockDim.x >> 5) {
        if (dead[first + q]) {
            if (lane == 0) best_s[(int64_t)q * F + f] = 0;
            continue;
        }
        const unsigned long long *hf = shist + (int64_t)q * nb * 2;
        // node totals: every feature's bins partition the node's samples
        long long Gi = 0, Hi = 0;
        for (int b = lane; b < nb; b += 32) { Gi += (long long)hf[2 * b]; Hi += (long long)hf[2 * b + 1]; }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            Gi += __shfl_xor_sync(0xFFFFFFFFu, Gi, off);
            Hi += __shfl_xor_sync(0xFFFFFFFFu, Hi, off);
        }
        const SplitBest best = scan_splits(hf, nb, Gi, Hi, lam, mcw, f, lane);
        if (lane == 0) {
            best_gain[(int64_t)q * F + f] = best.gain;
            best_s[(int64_t)q * F + f] = best.f < 0 ? 0 : best.s;
        }
    }
}

// one warp per (node, feature): prefix sums over the feature's bins by warp scans (exact int64),
// every split s = 1..ncuts_f evaluated in fp64 in the oracle's operation order.
__global__ void __launch_bounds__(256) split_feature_kernel(const int64_t *__restrict__ hist,
                                                            const int32_t *__restrict__ boff, int TB, int F, int first,
                                                            int nn, double lam, double mcw,
                                                            const uint8_t *__restrict__ dead,
                                                            double *__restrict__ best_gain, int32_t *__restrict__ best_s)
{
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= nn * F) return;
    const int q = gw / F, f = gw - q * F;
    const int nd = first + q;
    if (dead[nd]) {
        if (lane == 0) best_s[(int64_t)q * F + f] = 0;
        return;
    }
    const int64_t *hn = hist + (int64_t)q * TB * 2;
    // node totals from feature 0 (every sample is in exactly one of its bins)
    long long Gi = 0, Hi = 0;
    const int nb0 = boff[1] - boff[0];
    for (int b = lane; b < nb0; b += 32) { Gi += hn[2 * b]; Hi += hn[2 * b + 1]; }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        Gi += __shfl_xor_sync(0xFFFFFFFFu, Gi, off);
        Hi += __shfl_xor_sync(0xFFFFFFFFu, Hi, off);
    }
    const SplitBest best = scan_splits(hn + (int64_t)boff[f] * 2, boff[f + 1] - boff[f], Gi, Hi, lam, mcw, f, lane);
    if (lane == 0) {
        best_gain[(int64_t)q * F + f] = best.gain;
        best_s[(int64_t)q * F + f] = best.f < 0 ? 0 : best.s;
    }
}

// one block per node: best over features (gain desc, feature asc), write the tree node
__global__ void __launch_bounds__(256) split_node_kernel(const double *__restrict__ best_gain,
                                                         const int32_t *__restrict__ best_s, int F, int first, int nn,
                                                         const float *__restrict__ cuts, int B,
                                                         uint8_t *__restrict__ dead, int32_t *__restrict__ split_f,
                                                         int32_t *__restrict__ split_s,
                                                         uint16_t *__restrict__ tree_feat, float *__restrict__ tree_thr)
{
    __shared__ SplitBest s_best[8];
    const int q = blockIdx.x, nd = first + q;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    SplitBest best{0.0, -1, 0};
    if (!dead[nd]) {
        for (int f = tid; f < F; f += 256) {
            const int s = best_s[(int64_t)q * F + f];
            if (s > 0) {
                SplitBest c{best_gain[(int64_t)q * F + f], f, s};
                if (split_better(c, best)) best = c;
            }
        }
    }
    best = warp_best(best);
    if (lane == 0) s_best[warp] = best;
    __syncthreads();
    if (tid == 0) {
        SplitBest b = s_best[0];
        for (int w = 1; w < 8; ++w)
            if (split_better(s_best[w], b)) b = s_best[w];
        if (b.f < 0) {
            // no valid split (or a dead node): pass-through, every sample goes left
            tree_feat[nd] = 0;
            tree_thr[nd] = __int_as_float(0x7f800000);
            split_f[nd] = -1;
            dead[2 * nd + 1] = 1;
            dead[2 * nd + 2] = 1;
        } else {
            tree_feat[nd] = (uint16_t)b.f;
            tree_thr[nd] = cuts[(int64_t)b.f * (B - 1) + b.s - 1];
            split_f[nd] = b.f;
            split_s[nd] = b.s;
        }
    }
}

// Split decision + partition in one launch (single rank, moderate n): every block decides all nn
// nodes of the level (warp per node; the per-feature bests are read 8 at a time so the loads are
// in flight together), block 0 stores the tree nodes and the dead flags, and each block then moves
// its samples to their children.  Saves a launch and a dependent round trip per level.
__global__ void __launch_bounds__(256) decide_partition_kernel(const double *__restrict__ best_gain,
                                                               const int32_t *__restrict__ best_s, int F, int first,
                                                               int nn, const float *__restrict__ cuts, int B,
                                                               uint8_t *__restrict__ dead, int32_t *__restrict__ split_f,
                                                               int32_t *__restrict__ split_s,
                                                               uint16_t *__restrict__ tree_feat,
                                                               float *__restrict__ tree_thr,
                                                               const uint8_t *__restrict__ bins, int64_t n,
                                                               int32_t *__restrict__ node)
{
    __shared__ int s_f[64], s_s[64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = warp; q < nn; q += blockDim.x >> 5) {
        const int nd = first + q;
        SplitBest best{0.0, -1, 0};
        if (!dead[nd]) {
            const double *bgq = best_gain + (int64_t)q * F;
            const int32_t *bsq = best_s + (int64_t)q * F;
            for (int f0 = 0; f0 < F; f0 += 32 * 8) {
                double gv[8];
                int sv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int f = f0 + 32 * u + lane;
                    sv[u] = f < F ? bsq[f] : 0;
                    gv[u] = f < F ? bgq[f] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (sv[u] > 0) {
                        SplitBest c{gv[u], f0 + 32 * u + lane, sv[u]};
                        if (split_better(c, best)) best = c;
                    }
                }
            }
        }
        best = warp_best(best);
        if (lane == 0) {
            s_f[q] = best.f;
            s_s[q] = best.s;
            if (blockIdx.x == 0) {
                if (best.f < 0) {
                    tree_feat[nd] = 0;
                    tree_thr[nd] = __int_as_float(0x7f800000);
                    split_f[nd] = -1;
                    dead[2 * nd + 1] = 1;
                    dead[2 * nd + 2] = 1;
                } else {
                    tree_feat[nd] = (uint16_t)best.f;
                    tree_thr[nd] = cuts[(int64_t)best.f * (B - 1) + best.s - 1];
                    split_f[nd] = best.f;
                    split_s[nd] = best.s;
                }
            }
        }
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nd = node[i];
    const int q = nd - first;
    const int sf = s_f[q];
    node[i] = (sf >= 0 && (int)bins[(int64_t)sf * n + i] >= s_s[q]) ? 2 * nd + 2 : 2 * nd + 1;
}

__global__ void partition_kernel(const uint8_t *__restrict__ bins, int64_t n, const int32_t *__restrict__ split_f,
                                 const int32_t *__restrict__ split_s, int32_t *__restrict__ node)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nd = node[i];
    const int sf = split_f[nd];
    int child = 2 * nd + 1;
    if (sf >= 0 && (int)bins[(int64_t)sf * n + i] >= split_s[nd]) child = 2 * nd + 2;
    node[i] = child;
}

__global__ void leafsum_kernel(const int32_t *__restrict__ node, const int64_t *__restrict__ g,
                               const int64_t *__restrict__ h, int64_t hb, int64_t he, int n_int,
                               int64_t *__restrict__ sums)
{
    const int64_t i = hb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= he) return;
    const int l = node[i] - n_int;
    atomicAdd((unsigned long long *)&sums[2 * l], (unsigned long long)g[i]);
    atomicAdd((unsigned long long *)&sums[2 * l + 1], (unsigned long long)h[i]);
}

__global__ void leaf_kernel(const int64_t *__restrict__ sums, int n_leaf, double eta, double lam,
                            float *__restrict__ leaf)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n_leaf) return;
    const double G = (double)sums[2 * l] * FX, H = (double)sums[2 * l + 1] * FX;
    leaf[l] = (float)(-(eta * (G / (H + lam))));
}

__global__ void pred_update_kernel(const int32_t *__restrict__ node, int64_t n, int n_int,
                                   const float *__restrict__ leaf, float *__restrict__ pred)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pred[i] = __fadd_rn(pred[i], leaf[node[i] - n_int]);
}

__global__ void pack_nodes_kernel(const uint16_t *__restrict__ feat, const float *__restrict__ thr, int64_t m,
                                  uint2 *__restrict__ nodes)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    nodes[i] = make_uint2(feat[i], __float_as_uint(thr[i]));
}

__global__ void finite_check_kernel(const float *__restrict__ c, int64_t n, int32_t *__restrict__ bad)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && !isfinite(c[i])) *bad = 1;
}

__global__ void key_check_kernel(const uint16_t *__restrict__ k, int64_t n, int32_t *__restrict__ bad)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && k[i] >= FIT_MAXKEYS) *bad = 2;
}


// ------------------------------------------------------------------ 3b. subtraction path (single rank, large n)
// Level-by-level like section 3, with the two standard GPU-histogram reductions of work:
//  * a node's samples are contiguous in a position array (perm), rebuilt per level by a scatter
//    (left children fill their parent's segment from the front, right children from the back; the
//    order inside a segment is arbitrary -- every consumer is an order-free integer sum);
//  * only the smaller child of every split node is histogrammed; the larger one is parent - smaller
//    (exact in int64), so a tree costs <= n (1 + (D - 1) / 2) sample visits instead of n D.
// A histogram block owns one node's sample chunk and a range of the splittable features whose cells
// fit in shared memory; a warp takes one sample (bins read as a row-major u8 row, 4 features per
// lane-load), lanes map to features, and each feature's cells sit in its lane's bank column, so one
// warp-wide atomic touches 32 distinct banks.  64-bit cells are two 32-bit words updated by native
// shared atomics with an explicit carry (smem_add_u64's rule); blocks flush with native 64-bit
// global atomics.  Node totals travel down the tree (left = the winning split's prefix sums, right =
// total - left), so the leaves need no extra pass.  Per level: split search (+ decisions), scatter
// (+ next work list), histograms of the smaller children, subtraction; one tree is one CUDA graph.
constexpr int SUB_NT = 1024;
constexpr int SUB_ROWS = 400;   // rows of 32 cells (+ 1 trash row): 4 planes x 4 B x 32 x 401 = 200 KB of shared memory
// default stripe cap (AT_SUB_ROWS overrides, within [B, SUB_ROWS]): 164 KB of shared histogram leaves
// the SM ~90 KB of L1 (measured on config 4: 37.8 ms at 290-320 rows vs 38.2 ms at 400)
constexpr int SUB_ROWS_DEF = 320;
constexpr int SUB_NQW = 4;      // row words per lane and sample: <= 512 features per range
constexpr int SUB_MAXR = 256;

// A feature range: compact features [k_lo, k_lo + nf).  Feature r (local index) lives in bank column
// r mod 32 of the block's shared histogram, at rows rowbase[k_lo + r] .. + nb - 1, so the lane that
// handles it (lane = r mod 32) owns that bank: one warp-wide atomic never conflicts.  Its bin byte
// sits in the sample's row at byte_off + 128 (r / 128) + 4 (r mod 32) + (r mod 128) / 32, so one
// 32-bit load per lane brings the bins of features 128u + 32j + lane, j = 0..3.
struct SubRange {
    int k_lo, nf, rows, byte_off;
};

// the subtraction path's layout, computed on the device from the cut counts (sub_layout_kernel), so a
// single-rank fit never reads them back: every launch is sized by an upper bound and reads these
struct SubDev {
    int Fs, FsP, NR, max_rows, NE, TB, target;
};

// one histogram block's work: positions [it.y, it.z) of node slot it.x, feature range R (the item and
// the range side by side, so a block's first loads do not depend on one another)
struct SubUnit {
    int4 it;
    SubRange R;
};

// zero 2 TB mult int64 cells with the whole grid (16-B stores); TB is read on the device
__device__ __forceinline__ void sub_zero_cells(int64_t *__restrict__ p, const SubDev *__restrict__ L, int mult)
{
    const int64_t m = (int64_t)L->TB * mult;   // pairs of cells
    longlong2 *q = (longlong2 *)p;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x)
        q[c] = make_longlong2(0, 0);
}

// items[0, m) x the NR ranges -> units, range-major (run by one block after its items are written)
__device__ __forceinline__ void sub_units(const int4 *__restrict__ items, int m, const SubRange *__restrict__ ranges,
                                          int NR, SubUnit *__restrict__ units, int32_t *__restrict__ n_units)
{
    for (int u = threadIdx.x; u < m * NR; u += blockDim.x) units[u] = SubUnit{items[u % m], ranges[u / m]};
    if (threadIdx.x == 0) *n_units = m * NR;
}

// one block; warp 0 lays out (lane l = bank column l): the splittable features in order, their
// bank-column rows (stripes of 32 features while every column still fits rows_cap, greedy -- the layout
// the host used to compute), the ranges, the row-byte inverse table and the split entries (feature,
// 32-split chunk).  With no splittable feature, feature 0 (one bin) stands in, so the root totals still
// come out of its histogram and every node stays a leaf.
__global__ void sub_layout_kernel(const int32_t *__restrict__ ncuts, const int32_t *__restrict__ boff, int F,
                                  int32_t *__restrict__ flist, int32_t *__restrict__ rowbase,
                                  int32_t *__restrict__ gbase, int32_t *__restrict__ nbk, int32_t *__restrict__ inv,
                                  int FsP_max, SubRange *__restrict__ rng, int32_t *__restrict__ ent_f,
                                  int32_t *__restrict__ ent_c, int nsm, int rows_cap, SubDev *__restrict__ L)
{
    for (int b = threadIdx.x; b < FsP_max; b += blockDim.x) inv[b] = -1;
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const unsigned below = (1u << lane) - 1u;
    // compaction of the splittable features (ascending), their cell bases and bin counts
    int Fs = 0;
    for (int f0 = 0; f0 < F; f0 += 32) {
        const int f = f0 + lane;
        const bool sp = f < F && ncuts[f] > 0;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, sp);
        if (sp) {
            const int k = Fs + __popc(m & below);
            flist[k] = f;
            gbase[k] = boff[f];
            nbk[k] = ncuts[f] + 1;
        }
        Fs += __popc(m);
    }
    if (Fs == 0) {
        if (lane == 0) { flist[0] = 0; gbase[0] = boff[0]; nbk[0] = 1; }
        Fs = 1;
    }
    __syncwarp();
    // ranges: add stripes of 32 features (feature k + nf + l on column l) while every column fits
    int FsP = 0, NR = 0, max_rows = 0;
    for (int k = 0; k < Fs;) {
        int col = 0, nf = 0;
        while (k + nf < Fs && nf < 128 * SUB_NQW) {
            const int m = min(32, Fs - (k + nf));
            const int nb = lane < m ? nbk[k + nf + lane] : 0;
            const bool fits = __all_sync(0xFFFFFFFFu, col + nb <= rows_cap);
            if (!fits && nf > 0) break;
            if (lane < m) rowbase[k + nf + lane] = col;
            col += nb;
            nf += m;
        }
        int rows = col;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) rows = max(rows, __shfl_xor_sync(0xFFFFFFFFu, rows, off));
        if (lane == 0) rng[NR] = SubRange{k, nf, rows, FsP};
        // row-byte inverse table of this range
        for (int r = lane; r < nf; r += 32) inv[FsP + 128 * (r / 128) + 4 * (r % 32) + (r % 128) / 32] = k + r;
        ++NR;
        max_rows = max(max_rows, rows);
        FsP += 128 * ((nf + 127) / 128);
        k += nf;
    }
    // split entries: feature k owns max(1, ceil(ncuts / 32)) consecutive entries (exclusive prefix)
    int NE = 0;
    for (int k0 = 0; k0 < Fs; k0 += 32) {
        const int k = k0 + lane;
        const int nchk = k < Fs ? max(1, (nbk[k] - 1 + 31) / 32) : 0;
        int x = nchk;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
            if (lane >= off) x += y;
        }
        const int e0 = NE + x - nchk;
        for (int c = 0; c < nchk; ++c) {
            ent_f[e0 + c] = flist[k];
            ent_c[e0 + c] = c;
        }
        NE += __shfl_sync(0xFFFFFFFFu, x, 31);
    }
    AT_DCHECK(FsP <= FsP_max);
    if (lane == 0) {
        L->Fs = Fs;
        L->FsP = FsP;
        L->NR = NR;
        L->max_rows = max_rows;
        L->NE = NE;
        L->TB = boff[F];
        L->target = max(1, nsm / NR);
    }
}

// bins [F][n] (column-major) -> binsR [n][FsP] in the ranges' byte order (inv[b] = compact feature
// at row byte b, -1 = padding)
__global__ void rowbins_kernel(const uint8_t *__restrict__ bins, int64_t n, const int32_t *__restrict__ flist,
                               const int32_t *__restrict__ inv, const SubDev *__restrict__ L, uint8_t *__restrict__ binsR)
{
    __shared__ uint8_t t[32][33];
    const int FsP = L->FsP;
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    for (int b0 = blockIdx.y * 32; b0 < FsP; b0 += gridDim.y * 32) {   // FsP known on the device only
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int b = b0 + r;
            const int64_t i = i0 + threadIdx.x;
            const int k = b < FsP ? inv[b] : -1;
            t[r][threadIdx.x] = (k >= 0 && i < n) ? bins[(int64_t)flist[k] * n + i] : (uint8_t)0;
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int64_t i = i0 + r;
            const int b = b0 + threadIdx.x;
            if (i < n && b < FsP) binsR[i * FsP + b] = t[threadIdx.x][r];
        }
        __syncthreads();
    }
}


// items[b] = {node slot, p0, p1, -}: block (b, r) adds positions [p0, p1) of perm (identity when
// perm == nullptr) into the cells of feature range r of hist[slot].  Warp w takes positions
// it.y + w + NW t (balanced to within one sample), 32 of them per batch (one coalesced load of their
// sample ids and gradients), then walks them with the next sample's row words in flight while the
// current one's atomics issue.
__global__ void __launch_bounds__(SUB_NT, 1) sub_hist_kernel(const uint8_t *__restrict__ binsR,
                                                             const SubDev *__restrict__ L,
                                                             const int32_t *__restrict__ perm,
                                                             const int64_t *__restrict__ g,
                                                             const int64_t *__restrict__ h,
                                                             const SubUnit *__restrict__ units,
                                                             const int32_t *__restrict__ n_units,
                                                             const int32_t *__restrict__ rowbase,
                                                             const int32_t *__restrict__ gbase,
                                                             const int32_t *__restrict__ nbk,
                                                             int64_t *__restrict__ hist, int hb, int he)
{
    extern __shared__ uint32_t sm[];
    // work unit blockIdx.x; the grid is an upper bound of the units (their count comes from the
    // device), the spare blocks exit at once
    const int FsP = L->FsP, TB = L->TB;
    const SubUnit U = units[blockIdx.x];   // (capacity-sized array: the load is in bounds either way)
    if ((int)blockIdx.x >= *n_units) return;
    const SubRange R = U.R;
    const int4 it = U.it;
    const int P = (R.rows + 1) * 32;   // + a trash row: empty slots (padding bytes are 0) add there
    uint32_t *glo = sm, *ghi = sm + P, *hlo = sm + 2 * P, *hhi = sm + 3 * P;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = SUB_NT / 32;
    for (int q = tid; q < 4 * P; q += SUB_NT) sm[q] = 0u;
    const int nqw = (R.nf + 127) >> 7;
    int rb[SUB_NQW][4];
#pragma unroll
    for (int u = 0; u < SUB_NQW; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = 128 * u + 32 * j + lane;
            rb[u][j] = (r < R.nf ? rowbase[R.k_lo + r] : R.rows) * 32 + lane;
        }
    __syncthreads();
    const uint8_t *rows = binsR + R.byte_off + 4 * lane;
    for (int t0 = 0; it.y + warp + NW * t0 < it.z; t0 += 32) {
        const int pl = it.y + warp + NW * (t0 + lane);
        const bool inseg = pl < it.z;
        const int ip = inseg ? (perm ? perm[pl] : pl) : 0;
        // multi-rank: this rank histograms only its own sample slice [hb, he) (the rest is all-reduced)
        const bool okp = inseg && ip >= hb && ip < he;
        const unsigned okm = __ballot_sync(0xFFFFFFFFu, okp);
        const int cnt = (int)__popc(okm);
        // compact the valid lanes to the front (lane k takes the k-th valid lane's sample)
        const int src = lane < cnt ? (int)__fns(okm, 0u, lane + 1) : 0;
        const int il = __shfl_sync(0xFFFFFFFFu, ip, src);
        const bool okl = lane < cnt;
        const unsigned long long gvl = okl ? (unsigned long long)g[il] : 0ull;
        const unsigned long long hvl = okl ? (unsigned long long)h[il] : 0ull;
        uint32_t w[SUB_NQW], wn[SUB_NQW];
        {
            const uint32_t *row = (const uint32_t *)(rows + (int64_t)__shfl_sync(0xFFFFFFFFu, il, 0) * FsP);
#pragma unroll
            for (int u = 0; u < SUB_NQW; ++u) w[u] = u < nqw ? row[32 * u] : 0u;
        }
        for (int sI = 0; sI < cnt; ++sI) {
            const int inext = __shfl_sync(0xFFFFFFFFu, il, (sI + 1) & 31);
            if (sI + 1 < cnt) {
                const uint32_t *row = (const uint32_t *)(rows + (int64_t)inext * FsP);
#pragma unroll
                for (int u = 0; u < SUB_NQW; ++u) wn[u] = u < nqw ? row[32 * u] : 0u;
            }
            const unsigned long long gv = __shfl_sync(0xFFFFFFFFu, gvl, sI);
            const unsigned long long hv = __shfl_sync(0xFFFFFFFFu, hvl, sI);
            if ((gv | hv) != 0ull) {   // warp-uniform: a zero-gradient sample contributes nothing
                const uint32_t gl = (uint32_t)gv, gh = (uint32_t)(gv >> 32), hl = (uint32_t)hv, hh = (uint32_t)(hv >> 32);
#pragma unroll
                for (int u = 0; u < SUB_NQW; ++u) {
                    if (u >= nqw) break;
                    // the 8 low-word atomics of the 4 slots first (their returns in flight together), then
                    // the 8 high words with their carries
                    int c[4];
                    uint32_t og[4], oh[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        c[j] = rb[u][j] + 32 * (int)((w[u] >> (8 * j)) & 255u);
                        AT_DCHECK(c[j] < P);
                        og[j] = atomicAdd(&glo[c[j]], gl);
                        oh[j] = atomicAdd(&hlo[c[j]], hl);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        atomicAdd(&ghi[c[j]], gh + ((og[j] + gl < og[j]) ? 1u : 0u));   // exact modular 64-bit sums
                        atomicAdd(&hhi[c[j]], hh + ((oh[j] + hl < oh[j]) ? 1u : 0u));
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < SUB_NQW; ++u) w[u] = wn[u];
        }
    }
    __syncthreads();
    // flush: lane = bank column, a warp walks a band of rows; each lane tracks the feature of its
    // column that holds the current row
    const int band = (R.rows + NW - 1) / NW;
    const int row0 = warp * band, row1 = min(R.rows, row0 + band);
    if (row0 < row1) {
        int r = lane;   // this column's features: lane, lane + 32, ...
        while (r < R.nf && rowbase[R.k_lo + r] + nbk[R.k_lo + r] <= row0) r += 32;
        int rbase = r < R.nf ? rowbase[R.k_lo + r] : 0x7FFFFFFF, rend = r < R.nf ? rbase + nbk[R.k_lo + r] : 0x7FFFFFFF;
        int cbase = r < R.nf ? gbase[R.k_lo + r] : 0;
        unsigned long long *hn = (unsigned long long *)(hist + (int64_t)it.x * TB * 2);
        for (int row = row0; row < row1; ++row) {
            if (row >= rend) {
                r += 32;
                rbase = r < R.nf ? rowbase[R.k_lo + r] : 0x7FFFFFFF;
                rend = r < R.nf ? rbase + nbk[R.k_lo + r] : 0x7FFFFFFF;
                cbase = r < R.nf ? gbase[R.k_lo + r] : 0;
            }
            if (row < rbase) continue;
            const int a = row * 32 + lane;
            const unsigned long long G = (unsigned long long)glo[a] | ((unsigned long long)ghi[a] << 32);
            const unsigned long long H = (unsigned long long)hlo[a] | ((unsigned long long)hhi[a] << 32);
            const int64_t cell = (int64_t)(cbase + row - rbase) * 2;
            if (G) atomicAdd(&hn[cell], G);
            if (H) atomicAdd(&hn[cell + 1], H);
        }
    }
}

// root items: chunks of [0, n) for node slot 0
__global__ void sub_root_items_kernel(int hb, int he, const SubDev *__restrict__ L, int4 *__restrict__ items,
                                      const SubRange *__restrict__ ranges, SubUnit *__restrict__ units,
                                      int32_t *__restrict__ n_units)
{
    const int target = L->target;
    const int n = he - hb;   // this rank's samples (all of them on one rank)
    const int ch = max(64, (n + target - 1) / target);
    const int m = (n + ch - 1) / ch;
    for (int b = threadIdx.x; b < m; b += blockDim.x) items[b] = make_int4(0, hb + b * ch, hb + min(n, (b + 1) * ch), 0);
    __syncthreads();
    sub_units(items, m, ranges, L->NR, units, n_units);
}

// root totals from the cells of the first splittable feature (its bins partition the samples),
// the root segment (this rank's n own samples), and (parity hook) the single cell of every constant feature
__global__ void sub_root_tot_kernel(int64_t *__restrict__ hist, const int32_t *__restrict__ boff,
                                    const int32_t *__restrict__ flist, int F, int n, int fill_const,
                                    int64_t *__restrict__ tot, int32_t *__restrict__ seg_start,
                                    int32_t *__restrict__ seg_cnt, const int32_t *__restrict__ d_tree)
{
    fill_const = fill_const && *d_tree == 0;   // the parity hook wants tree 0's root histogram
    __shared__ long long s_t[2];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        const int f = flist[0];
        long long G = 0, H = 0;
        for (int b = boff[f] + lane; b < boff[f + 1]; b += 32) { G += hist[2 * b]; H += hist[2 * b + 1]; }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            G += __shfl_xor_sync(0xFFFFFFFFu, G, off);
            H += __shfl_xor_sync(0xFFFFFFFFu, H, off);
        }
        if (lane == 0) {
            tot[0] = G; tot[1] = H; s_t[0] = G; s_t[1] = H;
            seg_start[0] = 0; seg_cnt[0] = n;
        }
    }
    __syncthreads();
    if (fill_const)
        for (int f = threadIdx.x; f < F; f += blockDim.x)
            if (boff[f + 1] - boff[f] == 1) { hist[2 * boff[f]] = s_t[0]; hist[2 * boff[f] + 1] = s_t[1]; }
}

// one warp, node q of the level: the winner over features, the tree node, the children's totals
// (run by the last block of sub_split_kernel; the per-feature bests come from other blocks: L2 loads)
__device__ __forceinline__ void sub_decide_node(int q, const double *__restrict__ best_gain,
                                                         const int32_t *__restrict__ best_s,
                                                         const int32_t *__restrict__ flist, int Fs, int first, int nn,
                                                         const float *__restrict__ cuts, int B,
                                                         const int64_t *__restrict__ hist,
                                                         const int32_t *__restrict__ boff, int TB,
                                                         uint8_t *__restrict__ dead, int32_t *__restrict__ split_f,
                                                         int32_t *__restrict__ split_s, uint16_t *__restrict__ tree_feat,
                                                         float *__restrict__ tree_thr, int64_t *__restrict__ tot,
                                                         int n_int, const int32_t *__restrict__ d_tree)
{
    tree_feat += (int64_t)*d_tree * n_int;   // this tree's nodes
    tree_thr += (int64_t)*d_tree * n_int;
    const int lane = threadIdx.x & 31;
    const int nd = first + q;
    SplitBest best{0.0, -1, 0};
    if (!dead[nd]) {
        const double *bgq = best_gain + (int64_t)q * Fs;
        const int32_t *bsq = best_s + (int64_t)q * Fs;
        for (int k0 = 0; k0 < Fs; k0 += 32 * 8) {   // 8 loads of each kind in flight per lane
            double gv[8];
            int sv[8], fv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int k = k0 + 32 * u + lane;
                sv[u] = k < Fs ? __ldcg(bsq + k) : 0;
                gv[u] = k < Fs ? __ldcg(bgq + k) : 0.0;
                fv[u] = k < Fs ? flist[k] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (sv[u] > 0) {
                    SplitBest c{gv[u], fv[u], sv[u]};
                    if (split_better(c, best)) best = c;
                }
        }
    }
    best = warp_best(best);
    const long long G = tot[2 * nd], H = tot[2 * nd + 1];
    if (best.f < 0) {
        if (lane == 0) {
            tree_feat[nd] = 0;
            tree_thr[nd] = __int_as_float(0x7f800000);
            split_f[nd] = -1;
            dead[2 * nd + 1] = 1;
            dead[2 * nd + 2] = 1;
            tot[2 * (2 * nd + 1)] = G; tot[2 * (2 * nd + 1) + 1] = H;
            tot[2 * (2 * nd + 2)] = 0; tot[2 * (2 * nd + 2) + 1] = 0;
        }
        return;
    }
    const int64_t *hf = hist + ((int64_t)q * TB + boff[best.f]) * 2;
    long long GL = 0, HL = 0;
    for (int b = lane; b < best.s; b += 32) { GL += hf[2 * b]; HL += hf[2 * b + 1]; }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        GL += __shfl_xor_sync(0xFFFFFFFFu, GL, off);
        HL += __shfl_xor_sync(0xFFFFFFFFu, HL, off);
    }
    if (lane == 0) {
        tree_feat[nd] = (uint16_t)best.f;
        tree_thr[nd] = cuts[(int64_t)best.f * (B - 1) + best.s - 1];
        split_f[nd] = best.f;
        split_s[nd] = best.s;
        tot[2 * (2 * nd + 1)] = GL; tot[2 * (2 * nd + 1) + 1] = HL;
        tot[2 * (2 * nd + 2)] = G - GL; tot[2 * (2 * nd + 2) + 1] = H - HL;
    }
}

// Best split over one 32-split chunk c of one feature: the carry (sums of the bins before the chunk)
// by a warp reduction, then the chunk's exact int64 prefix scan and fp64 gains in the oracle's order
// (scan_splits restricted to one chunk).
__device__ __forceinline__ SplitBest scan_chunk(const int64_t *hf, int nb, int c, long long Gi, long long Hi,
                                                double lam, double mcw, int f, int lane)
{
    const int nc = nb - 1;
    const double G = (double)Gi * FX, H = (double)Hi * FX;
    const double parent = G * G / (H + lam);
    SplitBest best{0.0, -1, 0};
    long long carryG = 0, carryH = 0;
    for (int b = lane; b < 32 * c; b += 32) { carryG += hf[2 * b]; carryH += hf[2 * b + 1]; }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        carryG += __shfl_xor_sync(0xFFFFFFFFu, carryG, off);
        carryH += __shfl_xor_sync(0xFFFFFFFFu, carryH, off);
    }
    const int b = 32 * c + lane;   // split s = b + 1 puts bins <= b on the left
    long long vg = b < nc ? hf[2 * b] : 0, vh = b < nc ? hf[2 * b + 1] : 0;
    const long long own_g = vg, own_h = vh;
    if (__ballot_sync(0xFFFFFFFFu, vg != 0 || vh != 0) == 0) return best;   // empty chunk: no new split
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long yg = __shfl_up_sync(0xFFFFFFFFu, vg, off);
        const long long yh = __shfl_up_sync(0xFFFFFFFFu, vh, off);
        if (lane >= off) { vg += yg; vh += yh; }
    }
    const long long GLi = carryG + vg, HLi = carryH + vh;
    if (b < nc && (own_g != 0 || own_h != 0)) {
        const double GL = (double)GLi * FX, HL = (double)HLi * FX;
        const double GR = (double)(Gi - GLi) * FX, HR = (double)(Hi - HLi) * FX;
        if (!(HL < mcw || HR < mcw)) {
            const double gain = (GL * GL / (HL + lam) + GR * GR / (HR + lam)) - parent;
            if (gain > 0.0) {
                SplitBest cnd{gain, f, b + 1};
                if (split_better(cnd, best)) best = cnd;
            }
        }
    }
    return warp_best(best);
}

// warp per (node, feature, 32-split chunk) entry: best split of the chunk from the node histogram and
// the node totals; the last warp to finish a node's entries (count in done[q]) decides that node
__global__ void __launch_bounds__(256) sub_split_kernel(const int64_t *__restrict__ hist,
                                                        const int32_t *__restrict__ boff,
                                                        const int32_t *__restrict__ ent_f,
                                                        const int32_t *__restrict__ ent_c, const SubDev *__restrict__ L,
                                                        int first, int nn, int64_t *__restrict__ tot, double lam,
                                                        double mcw, uint8_t *__restrict__ dead,
                                                        double *__restrict__ best_gain, int32_t *__restrict__ best_s,
                                                        const float *__restrict__ cuts, int B,
                                                        int32_t *__restrict__ split_f, int32_t *__restrict__ split_s,
                                                        uint16_t *__restrict__ tree_feat, float *__restrict__ tree_thr,
                                                        int n_int, const int32_t *__restrict__ d_tree,
                                                        unsigned *__restrict__ done)
{
    const int lane = threadIdx.x & 31;
    const int NE = L->NE, TB = L->TB;
    // warps stride over the entries (the grid is sized by an upper bound of NE)
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gw < nn * NE; gw += nwarps) {
        const int q = gw / NE, j = gw - q * NE;
        const int nd = first + q, f = ent_f[j];
        if (dead[nd]) {
            if (lane == 0) best_s[(int64_t)q * NE + j] = 0;
        } else {
            const SplitBest best = scan_chunk(hist + ((int64_t)q * TB + boff[f]) * 2, boff[f + 1] - boff[f], ent_c[j],
                                              tot[2 * nd], tot[2 * nd + 1], lam, mcw, f, lane);
            if (lane == 0) {
                best_gain[(int64_t)q * NE + j] = best.gain;
                best_s[(int64_t)q * NE + j] = best.f < 0 ? 0 : best.s;
            }
        }
        unsigned last = 0;
        if (lane == 0) {
            __threadfence();
            last = atomicAdd(&done[q], 1u) == (unsigned)(NE - 1);
        }
        last = __shfl_sync(0xFFFFFFFFu, last, 0);
        if (!last) continue;
        __threadfence();
        // entries in feature order, chunks ascending: the (gain desc, f asc, s asc) rule picks as before
        sub_decide_node(q, best_gain, best_s, ent_f, NE, first, nn, cuts, B, hist, boff, TB, dead, split_f, split_s,
                        tree_feat, tree_thr, tot, n_int, d_tree);
        if (lane == 0) done[q] = 0u;   // for the next level
    }
}

// one block: children's segments, the smaller child of every split node as histogram items (chunks
// of <= ch positions), and the (parent, smaller, larger) slot triples for the subtraction
__device__ __forceinline__ void sub_worklist(int first, int nn, const int32_t *__restrict__ split_f,
                                             int32_t *__restrict__ cursor, int32_t *__restrict__ seg_start,
                                    int32_t *__restrict__ seg_cnt, int target, int4 *__restrict__ items,
                                    int32_t *__restrict__ n_items, int4 *__restrict__ subs, int32_t *__restrict__ n_subs,
                                    int compact, const int64_t *__restrict__ tot, const SubRange *__restrict__ ranges,
                                    int NR, SubUnit *__restrict__ units, int32_t *__restrict__ n_units)
{
    __shared__ int s_cs[128], s_m0[129], s_s0[129], s_ch;
    const int q = threadIdx.x;
    const int cfirst = 2 * first + 1;   // first node of level d + 1
    int small = 0, st = 0, cs = 0, alive = 0;
    if (q < nn) {
        const int nd = first + q;
        const int L = __ldcg(cursor + 2 * q), Rc = __ldcg(cursor + 2 * q + 1), s0 = seg_start[nd];
        cursor[2 * q] = 0;   // for the next level's scatter
        cursor[2 * q + 1] = 0;
        seg_start[2 * nd + 1] = s0;
        seg_cnt[2 * nd + 1] = L;
        seg_start[2 * nd + 2] = s0 + L;
        seg_cnt[2 * nd + 2] = Rc;
        alive = split_f[nd] >= 0;
        // the child to histogram: the one with fewer samples; with R ranks the counts are per rank, so the
        // choice must come from replicated data instead -- the child with the smaller curvature sum H
        // (global, from the all-reduced histograms), which is what the sample count stands in for
        const bool left = compact ? tot[2 * (2 * nd + 1) + 1] <= tot[2 * (2 * nd + 2) + 1] : L <= Rc;
        small = left ? 2 * nd + 1 : 2 * nd + 2;
        st = left ? s0 : s0 + L;
        cs = left ? L : Rc;
        s_cs[q] = alive ? cs : 0;
    }
    __syncthreads();
    if (q == 0) {
        long long total = 0;
        for (int p = 0; p < nn; ++p) total += s_cs[p];
        const int ch = (int)max(64ll, (total + target - 1) / target);
        int m = 0, ns = 0;
        for (int p = 0; p < nn; ++p) {
            s_m0[p] = m;
            s_s0[p] = ns;
            m += (s_cs[p] + ch - 1) / ch;
            ns += split_f[first + p] >= 0 ? 1 : 0;
        }
        s_ch = ch;
        s_m0[nn] = m;
        *n_items = m;
        *n_subs = ns;
    }
    __syncthreads();
    if (q < nn && alive) {
        const int big = (small & 1) ? small + 1 : small - 1;
        const int ch = s_ch;
        int m = s_m0[q];
        subs[s_s0[q]] = make_int4(q, small - cfirst, big - cfirst, 0);
        // compact (multi-rank): the smaller child of parent q goes to slot q of a dense [nn] buffer, the
        // one that is all-reduced; else straight to its child slot
        const int slot = compact ? q : small - cfirst;
        for (int o = 0; o < cs; o += ch) items[m++] = make_int4(slot, st + o, st + min(cs, o + ch), 0);
    }
    __syncthreads();
    sub_units(items, s_m0[nn], ranges, NR, units, n_units);
}

// samples of level-d nodes move to their children: node ids, and positions in the parent's segment
// (left from the front, right from the back); cursor[2 q + right] counts them; the last block to
// finish builds the next level's work list
__global__ void __launch_bounds__(256) sub_scatter_kernel(const uint8_t *__restrict__ bins, int64_t n,
                                                          const int32_t *__restrict__ split_f,
                                                          const int32_t *__restrict__ split_s, int first, int nn,
                                                          int32_t *__restrict__ seg_start,
                                                          int32_t *__restrict__ seg_cnt,
                                                          int32_t *__restrict__ cursor, int32_t *__restrict__ node,
                                                          int32_t *__restrict__ perm, const SubDev *__restrict__ L,
                                                          int4 *__restrict__ items,
                                                          int32_t *__restrict__ n_items, int4 *__restrict__ subs,
                                                          int32_t *__restrict__ n_subs, unsigned *__restrict__ done,
                                                          int compact, int64_t *__restrict__ tot, int hb, int he,
                                                          const SubRange *__restrict__ ranges,
                                                          SubUnit *__restrict__ units, int32_t *__restrict__ n_units,
                                                          int64_t *__restrict__ zp, int zmult)
{
    __shared__ int sc[256], sbase[256];
    const int tid = threadIdx.x;
    sub_zero_cells(zp, L, zmult);   // the next histogram launch's slots (nobody reads them here)
    for (int q = tid; q < 2 * nn; q += blockDim.x) sc[q] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + tid;
    const bool ok = i < n;
    // every sample moves to its child (the partition is replicated on all ranks); positions are kept for
    // this rank's own samples [hb, he) only -- the ones it histograms
    const bool own = ok && i >= hb && i < he;
    int nd = 0, slot = 0, r = 0, right = 0;
    if (ok) {
        nd = node[i];
        const int sf = split_f[nd];
        right = (sf >= 0 && (int)bins[(int64_t)sf * n + i] >= split_s[nd]) ? 1 : 0;
        slot = (nd - first) * 2 + right;
        if (own) r = atomicAdd(&sc[slot], 1);
    }
    __syncthreads();
    for (int q = tid; q < 2 * nn; q += blockDim.x)
        if (sc[q]) sbase[q] = atomicAdd(&cursor[q], sc[q]);
    __syncthreads();
    if (ok) node[i] = 2 * nd + 1 + right;
    if (own) {
        const int o = sbase[slot] + r;
        perm[right ? seg_start[nd] + seg_cnt[nd] - 1 - o : seg_start[nd] + o] = (int32_t)i;
    }
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    sub_worklist(first, nn, split_f, cursor, seg_start, seg_cnt, L->target, items, n_items, subs,
                 n_subs, compact, tot, ranges, L->NR, units, n_units);
    if (tid == 0) *done = 0u;
}

// larger child = parent - smaller child, every cell (exact int64)
__global__ void sub_subtract_kernel(const int64_t *__restrict__ parent, int64_t *__restrict__ child,
                                    const SubDev *__restrict__ L, const int4 *__restrict__ subs,
                                    const int32_t *__restrict__ n_subs)
{
    const int TB = L->TB;
    if ((int)blockIdx.y >= *n_subs) return;
    const int4 s = subs[blockIdx.y];
    const int64_t m = 2 * (int64_t)TB;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x)
        child[s.z * m + c] = parent[s.x * m + c] - child[s.y * m + c];
}

// multi-rank: the all-reduced smaller children (dense slot q) -> both children: small = reduced,
// large = parent - small (exact int64)
__global__ void sub_expand_kernel(const int64_t *__restrict__ parent, const int64_t *__restrict__ small,
                                  int64_t *__restrict__ child, const SubDev *__restrict__ L, const int4 *__restrict__ subs,
                                  const int32_t *__restrict__ n_subs)
{
    const int TB = L->TB;
    if ((int)blockIdx.y >= *n_subs) return;
    const int4 s = subs[blockIdx.y];
    const int64_t m = 2 * (int64_t)TB;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = small[s.x * m + c];
        child[s.y * m + c] = v;
        child[s.z * m + c] = parent[s.x * m + c] - v;
    }
}

// zero 2 TB mult int64 cells (TB read on the device; 16-B stores), grid-stride
__global__ void sub_zero_kernel(int64_t *__restrict__ p, const SubDev *__restrict__ L, int mult)
{
    sub_zero_cells(p, L, mult);
}

// last level: every sample's leaf, prediction update in tree order
__global__ void sub_final_kernel(const uint8_t *__restrict__ bins, int64_t n, int32_t *__restrict__ node,
                                 const int32_t *__restrict__ split_f, const int32_t *__restrict__ split_s, int n_int,
                                 const float *__restrict__ leaf, float *__restrict__ pred, const int32_t *__restrict__ d_tree,
                                 int64_t *__restrict__ zp, const SubDev *__restrict__ L)
{
    sub_zero_cells(zp, L, 1);   // the next tree's root histogram (no histogram is read any more)
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    leaf += (int64_t)*d_tree * (n_int + 1);
    const int nd = node[i];
    node[i] = 0;   // every sample starts the next tree at the root
    const int sf = split_f[nd];
    const int child = (sf >= 0 && (int)bins[(int64_t)sf * n + i] >= split_s[nd]) ? 2 * nd + 2 : 2 * nd + 1;
    pred[i] = __fadd_rn(pred[i], leaf[child - n_int]);
}

// leaves of this tree from the level-D node totals: w = -eta G / (H + lambda)
__global__ void sub_leaf_kernel(const int64_t *__restrict__ sums, int n_leaf, double eta, double lam,
                                float *__restrict__ leaf, const int32_t *__restrict__ d_tree,
                                uint8_t *__restrict__ dead, int n_dead)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    for (int q = l; q < n_dead; q += gridDim.x * blockDim.x) dead[q] = 0;   // for the next tree
    if (l >= n_leaf) return;
    const double G = (double)sums[2 * l] * FX, H = (double)sums[2 * l + 1] * FX;
    leaf[(int64_t)*d_tree * n_leaf + l] = (float)(-(eta * (G / (H + lam))));
}

__global__ void sub_tree_next_kernel(int32_t *d_tree)
{
    *d_tree += 1;
}

// ------------------------------------------------------------------ 4. fused forest (single rank, small n)
// One cooperative launch fits the whole forest when the training set is small (Algorithm 1's D:
// hundreds to a few thousand measured configurations).  Block b owns features b, b + G, ...; each
// keeps, per feature, the samples in an order that is sorted by bin inside every node's segment
// (a stable partition per level keeps it so), so a node's split candidates are the ends of its
// bin runs and (G_L, H_L) are exact int64 prefix sums -- the same numbers as the histogram path
// (cells with no samples are skipped there; cells whose sums are zero tie with the previous split
// and lose to its smaller s), with O(n) work per feature and level instead of O(nodes x bins).
// The best (gain, f, s) of every node is a 128-bit atomic max on a key ordered like split_better;
// one grid barrier per level publishes it.  Per tree: gradients per group (members found by the
// inverse of the Feistel cycle walk, so no member table), barrier, D levels, then every block
// derives the leaves redundantly; the prediction update of tree t is applied by the owner of each
// sample's group in tree t + 1 (and once more after the last tree).
constexpr int FUSED_NMAX = 2048;
constexpr int FUSED_NT_MAX = 512;   // threads per block: 512 when every splittable feature gets a
                                     // block at 2 blocks / SM, else 256 (4 / SM)
constexpr int FUSED_NSUB = 8;   // sub-slots per node (block b uses b mod 8): bounds CAS contention

struct FusedArgs {
    const uint8_t *bins;
    const int32_t *ncuts;
    const float *cuts;
    int B, n, F, D, n_trees, GS, n_groups;
    const int32_t *counts, *woff, *gpre, *klist;
    const float *cost;
    float *pred[2];             // ping-pong: tree t reads pred[(t - 1) & 1], its chunk owners write pred[t & 1]
    int64_t *g, *h;
    uint16_t *gord, *gord0;
    uint8_t *gnode;
    unsigned long long *slot;   // [2 tree parities][n_int][FUSED_NSUB] x (lo, hi)
    uint16_t *t_feat;
    float *t_thr, *t_leaf;
    uint64_t seed;
    double lam, mcw, eta;
    unsigned *bar;
    int objective;              // AT_OBJ_RANK / AT_OBJ_REG
    const int32_t *flist;       // the features that can split (ncuts > 0), ascending; info[4] of them
    const int32_t *info;        // device sizes of the fit prep: [2] input flags, [3] groups, [4] splittable features
};

__host__ __device__ inline int fused_ep(int N, int NT)
{
    int EP = 1;                                      // positions per thread (power of two)
    while (EP * NT < N) EP <<= 1;
    return EP;
}

// per-block node tables and scan scratch (nodes of one level <= 128, children <= 256)
struct FusedTail {
    int32_t segP[260], segC[260];                   // parent / child segment bounds (positions)
    int32_t decf[128], decs[128];                   // level decisions (f, s); decf < 0: no split
    int32_t Rst[128], Ren[128];                     // right-going count before a segment / through its end
    long long baseG[128], baseH[128], endG[128], endH[128];   // prefix sums before / at the end of a node
    long long rbG[128], rbH[128], reG[128], reH[128];         // leaves: flagged prefix before / through a node
    unsigned nbh[128], nbl[128], nms[128];          // per-node best gain (hi, lo words) and its lowest s
    unsigned decw[128];                             // published decision words
    float lval[256];                                // leaf values of the current tree
    int32_t wsi[2][FUSED_NT_MAX / 32];              // scan scratch
    int32_t gpre[FIT_MAXKEYS + 1];                  // group prefix per workload (copy)
    long long wsl[2][2 * (FUSED_NT_MAX / 32)];
    uint8_t dead[512];
};

__host__ __device__ inline size_t fused_smem_bytes(int N, int GS)
{
    size_t b = 16 * (size_t)N;                       // sg sh (int64, by sample)
    b += 8 * 512;                                    // leaf sums (u64 [2^D][2]) / counting-sort counters
    b += 12 * (size_t)GS;                            // mem sc sp
    b += 4 * (size_t)N;                              // ordA ordB (u16)
    b += 5 * (size_t)N + 16;                         // natA natB sbin posbin leafof (u8)
    b = (b + 15) & ~(size_t)15;
    return b + sizeof(FusedTail);
}

__device__ __forceinline__ uint32_t feistel_inv(uint32_t y, int h, uint64_t seed, uint32_t tree, uint32_t wkey)
{
    // forward round r: (L, R) -> (R, L ^ F_r(R)); inverse: (L', R') -> (R' ^ F_r(L'), L')
    const uint32_t mask = (1u << h) - 1u;
    uint32_t L = y >> h, R = y & mask;
#pragma unroll
    for (int r = 3; r >= 0; --r) {
        const U4 o = philox(seed, L, tree, (wkey << 2) | (uint32_t)r, TAG_GROUP_PERM);
        const uint32_t pL = R ^ (o.x & mask), pR = L;
        L = pL;
        R = pR;
    }
    return (L << h) | R;
}

// 128-bit atomic max of (hi, lo) (unsigned lexicographic) at p[0] = lo, p[1] = hi
__device__ __forceinline__ void slot_max(unsigned long long *p, unsigned long long klo, unsigned long long khi)
{
    unsigned long long lo = 0, hi = 0;
    for (;;) {
        if (khi < hi || (khi == hi && klo <= lo)) return;
        unsigned long long olo, ohi;
        asm volatile("{\n.reg .b128 c, s, d;\nmov.b128 c, {%2, %3};\nmov.b128 s, {%4, %5};\n"
                     "atom.global.cas.b128 d, [%6], c, s;\nmov.b128 {%0, %1}, d;\n}"
                     : "=l"(olo), "=l"(ohi)
                     : "l"(lo), "l"(hi), "l"(klo), "l"(khi), "l"(p)
                     : "memory");
        if (olo == lo && ohi == hi) return;
        lo = olo;
        hi = ohi;
    }
}

// block-wide exclusive scan of one int per thread (thread order); `ws` must not be reused before
// the next __syncthreads after this call
template <int NW>
__device__ __forceinline__ int blk_excl_int(int v, int lane, int warp, int32_t *ws, int &total)
{
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    int o = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int u = ws[w];
        o += w < warp ? u : 0;
        tot += u;
    }
    total = tot;
    return o + x - v;
}

// the same for a pair of int64 (exact, order-free)
template <int NW>
__device__ __forceinline__ void blk_excl_i64x2(long long a, long long b, int lane, int warp, long long *ws,
                                               long long &oa, long long &ob)
{
    long long x = a, y = b;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const long long u = __shfl_up_sync(0xFFFFFFFFu, x, off), v = __shfl_up_sync(0xFFFFFFFFu, y, off);
        if (lane >= off) { x += u; y += v; }
    }
    if (lane == 31) { ws[2 * warp] = x; ws[2 * warp + 1] = y; }
    __syncthreads();
    long long pa = x - a, pb = y - b;
#pragma unroll
    for (int w = 0; w < NW; ++w)
        if (w < warp) { pa += ws[2 * w]; pb += ws[2 * w + 1]; }
    oa = pa;
    ob = pb;
}

// One cooperative launch fits the whole forest.  Block b owns feature b (and b + G, ... when F > G).
// Thread t owns the EP consecutive positions t EP .. t EP + EP - 1 of the block's feature order, so
// every per-position quantity of a level (sample, node, go-right flag, prefix sums, split key) stays
// in registers between the block scans:
//   partition: flags -> block scan -> right counts at segment bounds -> scatter of (sample, child);
//   prefix sums of (g, h) in the new order -> node bases / totals -> every run end's fp64 gain;
//   per-node max by native 32-bit shared atomics (gain high word, low word, then the lowest s among
//   equal gains), one 128-bit global atomic max per node on (gain, 0xFFFF - f, 0xFFFF - s).
#ifdef AT_FIT_TIMING
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_ft_work_max = 0ull, g_ft_grad_max = 0ull, g_ft_bar_ns = 0ull, g_ft_bar_n = 0ull;
#ifndef AT_FIT_BLOCKS_DUMP
#define AT_FIT_BLOCKS_DUMP 0
#endif
constexpr bool getenv_blocks_dump = AT_FIT_BLOCKS_DUMP;   // per-block work lines (tools/fit_blocks.py)
#define FT_MARK(k) do { if (threadIdx.x == 0) { unsigned long long _t = gtimer(); ft[k] += _t - ft_last; ft_last = _t; } } while (0)
#else
#define FT_MARK(k) do {} while (0)
#endif

template <int EP, int NT>
__global__ void __launch_bounds__(NT, NT == 512 ? (EP >= 4 ? 1 : 2) : (EP >= 8 ? 3 : 4)) fused_forest_kernel(FusedArgs A)
{
#ifdef AT_FIT_TIMING
    unsigned long long ft[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, ft_last = gtimer(), t_arr = 0;
#endif
    extern __shared__ __align__(16) unsigned char fsm[];
    const int N = A.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    int64_t *sg = (int64_t *)fsm, *sh = sg + N;
    unsigned long long *lsum = (unsigned long long *)(sh + N);   // [512]
    unsigned *cnt = (unsigned *)lsum;                            // counting sort scratch (init only)
    int32_t *mem = (int32_t *)(lsum + 512);
    float *sc = (float *)(mem + A.GS), *sp = sc + A.GS;
    uint16_t *ordA = (uint16_t *)(sp + A.GS), *ordB = ordA + N;
    uint8_t *natA = (uint8_t *)(ordB + N), *natB = natA + N, *sbin = natB + N, *posbin = sbin + N,
            *leafof = posbin + N + 16;
    FusedTail &T = *(FusedTail *)(fsm + ((((size_t)(leafof + N - fsm)) + 15) & ~(size_t)15));

    // blocks own the features that can split (constant ones never can: no cut), block b feature
    // flist[b] (and flist[b + G], ... when there are more than blocks)
    // the splittable-feature count and the group count come from the prep kernels on the device, so the
    // host launches this kernel without reading them back (gbt_fit_hist never syncs on this path)
    if (A.info[2] != 0) return;   // bad input: the model stays undefined, the fit's error word says so
    // the launch is sized for every feature; blocks beyond the splittable ones leave before the first
    // grid barrier, which then counts the G working blocks only
    const int F = max(A.info[4], 1), G = min((int)gridDim.x, F), D = A.D, n_groups = A.info[3];
    if ((int)blockIdx.x >= G) return;
    const int n_int = (1 << D) - 1, n_leaf = 1 << D;
    const bool resident = F <= G;
    unsigned epoch = 0;
    const int CM = A.GS / 8 > 8 ? A.GS / 8 : 8;
    const int chunks = (A.GS + CM - 1) / CM;
    for (int q = tid; q < 128; q += NT) { T.nbh[q] = 0; T.nbl[q] = 0; T.nms[q] = 0xFFFFFFFFu; }
    for (int q = tid; q <= FIT_MAXKEYS; q += NT) T.gpre[q] = A.gpre[q];

    // Grid-wide sync.  Every block arrives on one counter (a release add) and its thread 0 polls the
    // counter with acquire loads until all G blocks are in; then EVERY block reads the level's
    // FUSED_NSUB sub-slot keys per node and takes the decisions itself (no reducer, no publish /
    // poll hop: 1.9 -> ~1.4 us per barrier).  The sub-slots of a tree live in its parity half; block 0
    // zeroes tree t - 1's half after tree t's gradient barrier (every block has read it by then) and
    // writes the tree's nodes.  T.decw[q] gets the decisions.
    auto sync_all = [&](int t, int nn, int first) {
        __syncthreads();
        ++epoch;
        if (tid == 0) {
            // arrival: one release add (this block's writes, ordered before it by the __syncthreads,
            // PTX fences being cumulative), then acquire polls of the counter until every block is in
#ifdef AT_FIT_TIMING
            t_arr = gtimer();
#endif
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.bar) : "memory");
            const unsigned want = epoch * (unsigned)G;
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.bar) : "memory");
            while (v < want) {
                __nanosleep(20);
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(A.bar) : "memory");
            }
        }
        __syncthreads();
        // every block reduces the level's sub-slots itself (no reducer -> publish -> poll hop):
        // FUSED_NSUB consecutive lanes per node, max by xor shuffles within the group
        if (nn > 0) {
            const unsigned long long *sb = A.slot + (size_t)(t & 1) * 2 * FUSED_NSUB * n_int;
            for (int base = 0; base < nn * FUSED_NSUB; base += NT) {
                const int e = base + tid, q = e / FUSED_NSUB;
                unsigned long long lo = 0, hi = 0;
                if (q < nn) {
                    const ulonglong2 v = __ldcg((const ulonglong2 *)(sb + 2 * ((first + q) * FUSED_NSUB + (e % FUSED_NSUB))));
                    lo = v.x;
                    hi = v.y;
                }
#pragma unroll
                for (int off = FUSED_NSUB / 2; off >= 1; off >>= 1) {
                    const unsigned long long ol = __shfl_xor_sync(0xFFFFFFFFu, lo, off);
                    const unsigned long long oh = __shfl_xor_sync(0xFFFFFFFFu, hi, off);
                    if (oh > hi || (oh == hi && ol > lo)) { lo = ol; hi = oh; }
                }
                if (q < nn && e % FUSED_NSUB == 0) {
                    const unsigned word = hi == 0 ? 0xFFFFFFFFu
                                                  : ((0xFFFFu - (unsigned)((lo >> 16) & 0xFFFFu)) << 8) |
                                                        (0xFFFFu - (unsigned)(lo & 0xFFFFu));
                    T.decw[q] = word;
                    if (blockIdx.x == 0) {   // the tree's nodes
                        const int nd = first + q;
                        const unsigned bf = word >> 8, bs = word & 0xFFu;
                        A.t_feat[(size_t)t * n_int + nd] = word == 0xFFFFFFFFu ? (uint16_t)0 : (uint16_t)bf;
                        A.t_thr[(size_t)t * n_int + nd] = word == 0xFFFFFFFFu ? __int_as_float(0x7f800000)
                                                                               : A.cuts[(int64_t)bf * (A.B - 1) + bs - 1];
                    }
                }
            }
        }
        __syncthreads();
#ifdef AT_FIT_TIMING
        if (tid == 0 && blockIdx.x == 0) {   // block 0: its arrival -> release (includes waiting for the others)
            atomicAdd(&g_ft_bar_ns, gtimer() - t_arr);
            atomicAdd(&g_ft_bar_n, 1ull);
        }
#endif
    };

    // ---- init: bin-sorted order of every owned feature (counting sort; order inside a bin is free)
    for (int fi = blockIdx.x; fi < F; fi += G) {
        const int f = __ldg(A.flist + fi);
        for (int i = tid; i < N; i += NT) sbin[i] = A.bins[(int64_t)f * N + i];
        for (int b = tid; b < 512; b += NT) cnt[b] = 0;
        __syncthreads();
        for (int i = tid; i < N; i += NT) atomicAdd(&cnt[sbin[i]], 1u);
        __syncthreads();
        if (warp == 0) {
            unsigned v[8], a = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { v[k] = cnt[lane * 8 + k]; a += v[k]; }
            unsigned x = a;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned y = __shfl_up_sync(0xFFFFFFFFu, x, off);
                if (lane >= off) x += y;
            }
            unsigned o = x - a;
#pragma unroll
            for (int k = 0; k < 8; ++k) { cnt[256 + lane * 8 + k] = o; o += v[k]; }
        }
        __syncthreads();
        for (int i = tid; i < N; i += NT) ordA[atomicAdd(&cnt[256 + sbin[i]], 1u)] = (uint16_t)i;
        __syncthreads();
        for (int j = tid; j < N; j += NT) A.gord0[(int64_t)f * N + j] = ordA[j];
        __syncthreads();
    }

    uint16_t *ord = ordA, *ord2 = ordB;
    uint8_t *nat = natA, *nat2 = natB;
    for (int t = 0; t < A.n_trees; ++t) {
        unsigned long long *slot = A.slot;
        // ---- gradients (and the previous tree's prediction update)
        if (A.objective == AT_OBJ_REG) {   // per sample: grid-stride over the samples
            for (int i = blockIdx.x * NT + tid; i < N; i += G * NT) {
                float pv = __ldcg(A.pred[0] + i);   // tree 0: the initial predictions
                if (t > 0) {
                    pv = __fadd_rn(__ldcg(A.pred[(t - 1) & 1] + i), T.lval[leafof[i]]);
                    A.pred[t & 1][i] = pv;
                }
                int64_t gi, hi;
                reg_grad(pv, A.cost[i], gi, hi);
                A.g[i] = gi;
                A.h[i] = hi;
            }
        }
        for (int item = blockIdx.x; A.objective == AT_OBJ_RANK && item < n_groups * chunks; item += G) {
            const int grp = item / chunks, a0 = (item - grp * chunks) * CM;
            if (tid == 0) {
                int lo = 0, hi = FIT_MAXKEYS;   // largest w with gpre[w] <= grp
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (T.gpre[mid] <= grp) lo = mid; else hi = mid;
                }
                T.wsi[0][0] = lo;
            }
            __syncthreads();
            const int w = T.wsi[0][0];
            __syncthreads();   // rewritten by the next item
            const int nw = A.counts[w];
            const int start = (grp - T.gpre[w]) * A.GS;
            const int m = min(A.GS, nw - start);
            const int a1 = min(m, a0 + CM);
            if (a0 >= m) continue;   // block-uniform
            int bits = 0;
            while ((1ull << bits) < (unsigned long long)nw) ++bits;
            int hb = (bits + 1) / 2;
            if (hb < 1) hb = 1;
            for (int a = tid; a < m; a += NT) {
                uint32_t r = feistel_inv((uint32_t)(start + a), hb, A.seed, (uint32_t)t, (uint32_t)w);
                while (r >= (uint32_t)nw) r = feistel_inv(r, hb, A.seed, (uint32_t)t, (uint32_t)w);
                const int i = A.klist[A.woff[w] + (int)r];
                mem[a] = i;
                float pv = __ldcg(A.pred[0] + i);   // tree 0: the initial predictions
                if (t > 0) {
                    pv = __fadd_rn(__ldcg(A.pred[(t - 1) & 1] + i), T.lval[leafof[i]]);
                    if (a >= a0 && a < a1) A.pred[t & 1][i] = pv;   // the chunk owning the member writes it
                }
                sp[a] = pv;
                sc[a] = A.cost[i];
            }
            __syncthreads();
            // warp per member of the chunk, lanes over its partners
            for (int a = a0 + warp; a < a1; a += NW) {
                long long ga = 0, ha = 0;
                const float ca = sc[a], fa = sp[a];
                for (int c = lane; c < m; c += 32)
                    if (c != a) pair_term(ca, fa, sc[c], sp[c], ga, ha);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    ga += __shfl_xor_sync(0xFFFFFFFFu, ga, off);
                    ha += __shfl_xor_sync(0xFFFFFFFFu, ha, off);
                }
                if (lane == 0) {
                    A.g[mem[a]] = ga;
                    A.h[mem[a]] = ha;
                }
            }
            __syncthreads();
        }
        FT_MARK(0);
        sync_all(t, 0, 0);
        FT_MARK(1);

        if (blockIdx.x == 0)   // tree t - 1's slots (every block has read them): zero for tree t + 1
            for (int e = tid; e < 2 * FUSED_NSUB * n_int; e += NT)
                __stcg(A.slot + (size_t)((t + 1) & 1) * 2 * FUSED_NSUB * n_int + e, 0ull);
        for (int i = tid; i < N; i += NT) { sg[i] = __ldcg(A.g + i); sh[i] = __ldcg(A.h + i); }
        for (int q = tid; q < 512; q += NT) T.dead[q] = 0;
        if (tid == 0) { T.segP[0] = 0; T.segP[1] = N; }
        __syncthreads();

        for (int d = 0; d < D; ++d) {
            const int nn = 1 << d, first = nn - 1, nnP = nn >> 1;
            for (int fi = blockIdx.x; fi < F; fi += G) {
                const int f = __ldg(A.flist + fi);
                const int nc = A.ncuts[f];
                if (!resident) {
                    for (int i = tid; i < N; i += NT) sbin[i] = A.bins[(int64_t)f * N + i];
                    if (d > 0)
                        for (int j = tid; j < N; j += NT) {
                            ord[j] = A.gord[(int64_t)f * N + j];
                            nat[j] = A.gnode[(int64_t)f * N + j];
                        }
                    __syncthreads();
                } else if (t == 0 && d == 0) {
                    for (int i = tid; i < N; i += NT) sbin[i] = A.bins[(int64_t)f * N + i];
                    __syncthreads();
                }
                int iv[EP], qv[EP];   // sample and node of each owned position (in the level's order)
                if (d == 0) {
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        iv[k] = 0;
                        qv[k] = 0;
                        if (j < N) {
                            iv[k] = (int)__ldcg(A.gord0 + (int64_t)f * N + j);
                            ord[j] = (uint16_t)iv[k];
                            nat[j] = 0;
                        }
                    }
                    if (tid == 0) { T.segC[0] = 0; T.segC[1] = N; }
                } else {
                    // stable partition of every parent segment by the parent's decision
                    int fl[EP], c = 0;
#pragma unroll
                    for (int k = 0; k < EP; ++k) {   // all gathers of the thread in flight together
                        const int j = tid * EP + k;
                        fl[k] = 0;
                        iv[k] = 0;
                        qv[k] = 0;
                        int bv = 0, th = 1 << 30;
                        if (j < N) {
                            const int i = ord[j], q = nat[j], sf = T.decf[q];
                            AT_DCHECK(i < N && q < 128);
                            iv[k] = i;
                            qv[k] = q;
                            if (sf >= 0) {
                                th = T.decs[q];
                                bv = sf == f ? (int)sbin[i] : (int)__ldg(A.bins + (int64_t)sf * N + i);
                            }
                        }
                        fl[k] = bv >= th ? 1 : 0;
                        c += fl[k];
                    }
                    int rtot;
                    const int ex0 = blk_excl_int<NW>(c, lane, warp, T.wsi[0], rtot);
                    int ex = ex0;
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        if (j < N) {
                            const int q = qv[k];
                            if (j == T.segP[q]) T.Rst[q] = ex;
                            if (j + 1 == T.segP[q + 1]) T.Ren[q] = ex + fl[k];
                        }
                        ex += fl[k];
                    }
                    __syncthreads();
                    ex = ex0;
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        if (j < N) {
                            const int q = qv[k], s0 = T.segP[q], s1 = T.segP[q + 1];
                            const int r0 = T.Rst[q], nR = T.Ren[q] - r0, nL = (s1 - s0) - nR, rb = ex - r0;
                            const int np = fl[k] ? s0 + nL + rb : j - rb;
                            ord2[np] = (uint16_t)iv[k];
                            nat2[np] = (uint8_t)(2 * q + fl[k]);
                        }
                        ex += fl[k];
                    }
                    for (int q = tid; q < nnP; q += NT) {
                        const int s0 = T.segP[q], s1 = T.segP[q + 1];
                        const int nR = s1 > s0 ? T.Ren[q] - T.Rst[q] : 0;
                        T.segC[2 * q] = s0;
                        T.segC[2 * q + 1] = s1 - nR;
                    }
                    if (tid == 0) T.segC[nn] = N;
                    __syncthreads();
                    { uint16_t *tq = ord; ord = ord2; ord2 = tq; }
                    { uint8_t *tq = nat; nat = nat2; nat2 = tq; }
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        if (j < N) { iv[k] = ord[j]; qv[k] = nat[j]; }
                    }
                }
                FT_MARK(5);   // (instrumented builds: partition)
                // prefix sums of (g, h) in this order; node bases and totals
                long long pg[EP], ph[EP];
                int qb[EP];   // node << 8 | bin of each owned position
                long long ag = 0, ah = 0;
#pragma unroll
                for (int k = 0; k < EP; ++k) {
                    const int j = tid * EP + k;
                    long long g = 0, h = 0;
                    qb[k] = 0;
                    if (j < N) {
                        const int i = iv[k], b = sbin[i];
                        g = sg[i];
                        h = sh[i];
                        qb[k] = (qv[k] << 8) | b;
                        posbin[j] = (uint8_t)b;
                    }
                    ag += g;
                    ah += h;
                    pg[k] = ag;
                    ph[k] = ah;
                }
                long long og, oh;
                blk_excl_i64x2<NW>(ag, ah, lane, warp, T.wsl[0], og, oh);
                {
                    long long prg = og, prh = oh;
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        pg[k] += og;
                        ph[k] += oh;
                        if (j < N) {
                            const int q = qb[k] >> 8;
                            if (j == T.segC[q]) { T.baseG[q] = prg; T.baseH[q] = prh; }
                            if (j + 1 == T.segC[q + 1]) { T.endG[q] = pg[k]; T.endH[q] = ph[k]; }
                        }
                        prg = pg[k];
                        prh = ph[k];
                    }
                }
                __syncthreads();
                FT_MARK(6);   // (prefix sums)
                // every run end of every node: the split s = b + 1 (left = bins <= b), fp64 gain in
                // the oracle's operation order
                unsigned long long gk[EP];
                {
                    int lastq = -1;
                    long long bG = 0, bH = 0, Gi = 0, Hi = 0;
                    double parent = 0.0;
#pragma unroll
                    for (int k = 0; k < EP; ++k) {
                        const int j = tid * EP + k;
                        gk[k] = 0ull;
                        if (j >= N) continue;
                        const int q = qb[k] >> 8, b = qb[k] & 0xFF;
                        if (T.dead[first + q] || b >= nc) continue;
                        const int s1 = T.segC[q + 1];
                        const int nb = j + 1 >= s1 ? -1 : (k + 1 < EP ? (qb[k + 1] & 0xFF) : (int)posbin[j + 1]);
                        if (nb == b) continue;
                        if (q != lastq) {
                            lastq = q;
                            bG = T.baseG[q];
                            bH = T.baseH[q];
                            Gi = T.endG[q] - bG;
                            Hi = T.endH[q] - bH;
                            const double Gd = (double)Gi * FX, Hd = (double)Hi * FX;
                            parent = Gd * Gd / (Hd + A.lam);
                        }
                        const long long GLi = pg[k] - bG, HLi = ph[k] - bH;
                        const double GL = (double)GLi * FX, HL = (double)HLi * FX;
                        const double GR = (double)(Gi - GLi) * FX, HR = (double)(Hi - HLi) * FX;
                        if (HL < A.mcw || HR < A.mcw) continue;
                        const double gain = (GL * GL / (HL + A.lam) + GR * GR / (HR + A.lam)) - parent;
                        if (gain > 0.0) gk[k] = (unsigned long long)__double_as_longlong(gain);
                    }
                }
#ifdef AT_FIT_TIMING
                __syncthreads();   // (instrumented builds: the gains alone)
                FT_MARK(8);
#endif
                // per-node max: gain high word, low word, then the lowest s among equal gains
#pragma unroll
                for (int k = 0; k < EP; ++k)
                    if (gk[k]) atomicMax(&T.nbh[(qb[k] >> 8)], (unsigned)(gk[k] >> 32));
                __syncthreads();
#pragma unroll
                for (int k = 0; k < EP; ++k)
                    if (gk[k] && (unsigned)(gk[k] >> 32) == T.nbh[(qb[k] >> 8)]) atomicMax(&T.nbl[(qb[k] >> 8)], (unsigned)gk[k]);
                __syncthreads();
#pragma unroll
                for (int k = 0; k < EP; ++k)
                    if (gk[k] && gk[k] == (((unsigned long long)T.nbh[(qb[k] >> 8)] << 32) | T.nbl[(qb[k] >> 8)]))
                        atomicMin(&T.nms[(qb[k] >> 8)], (unsigned)((qb[k] & 0xFF) + 1));
                __syncthreads();
                FT_MARK(7);   // (gains + per-node shared maxima)
                for (int q = tid; q < nn; q += NT) {
                    const unsigned long long gb = ((unsigned long long)T.nbh[q] << 32) | T.nbl[q];
                    if (gb)
                        slot_max(slot + (size_t)(t & 1) * 2 * FUSED_NSUB * n_int +
                                     2 * ((first + q) * FUSED_NSUB + (blockIdx.x & (FUSED_NSUB - 1))),
                                 ((unsigned long long)(0xFFFFu - (unsigned)f) << 16) |
                                     (unsigned long long)(0xFFFFu - T.nms[q]),
                                 gb);
                    T.nbh[q] = 0;
                    T.nbl[q] = 0;
                    T.nms[q] = 0xFFFFFFFFu;
                }
                if (!resident)
                    for (int j = tid; j < N; j += NT) {
                        A.gord[(int64_t)f * N + j] = ord[j];
                        A.gnode[(int64_t)f * N + j] = nat[j];
                    }
                __syncthreads();
            }
            FT_MARK(2);
            sync_all(t, nn, first);
            FT_MARK(3);
            // the level's decisions (identical in every block; a dead node never has a split)
            for (int q = tid; q < nn; q += NT) {
                const int nd = first + q;
                const unsigned word = T.decw[q];
                if (word == 0xFFFFFFFFu) {
                    T.decf[q] = -1;
                    T.decs[q] = 0;
                    T.dead[2 * nd + 1] = 1;
                    T.dead[2 * nd + 2] = 1;
                } else {
                    T.decf[q] = (int)(word >> 8);
                    T.decs[q] = (int)(word & 0xFFu);
                }
            }
            for (int q = tid; q <= nn; q += NT) T.segP[q] = T.segC[q];
            __syncthreads();
        }
        // ---- leaves (every block, from its first feature's final order): the last level's decisions
        // as go-right flags per owned position, one block scan of the flagged (g, h), so each node's
        // right-child sums are two prefix values at its segment bounds and the left child is the node
        // total (the last level's bases / ends) minus them -- exact int64, no atomics
        {
            const int f = __ldg(A.flist + blockIdx.x);
            if (!resident) {
                for (int j = tid; j < N; j += NT) {
                    ord[j] = A.gord[(int64_t)f * N + j];
                    nat[j] = A.gnode[(int64_t)f * N + j];
                }
                __syncthreads();
            }
            long long rg[EP], rh[EP];
            int qv[EP];
            long long ag = 0, ah = 0;
#pragma unroll
            for (int k = 0; k < EP; ++k) {   // all gathers of the thread in flight together
                const int j = tid * EP + k;
                int fl = 0, q = 0, i = 0;
                if (j < N) {
                    i = ord[j];
                    q = nat[j];
                    const int sf = T.decf[q];
                    if (sf >= 0) fl = (int)__ldg(A.bins + (int64_t)sf * N + i) >= T.decs[q] ? 1 : 0;
                    leafof[i] = (uint8_t)(2 * q + fl);
                }
                qv[k] = q;
                if (fl) { ag += sg[i]; ah += sh[i]; }
                rg[k] = ag;
                rh[k] = ah;
            }
            long long og, oh;
            blk_excl_i64x2<NW>(ag, ah, lane, warp, T.wsl[1], og, oh);
            {
                long long pg = og, ph = oh;
#pragma unroll
                for (int k = 0; k < EP; ++k) {
                    const int j = tid * EP + k;
                    const long long ig = og + rg[k], ih = oh + rh[k];
                    if (j < N) {
                        const int q = qv[k];
                        if (j == T.segP[q]) { T.rbG[q] = pg; T.rbH[q] = ph; }
                        if (j + 1 == T.segP[q + 1]) { T.reG[q] = ig; T.reH[q] = ih; }
                    }
                    pg = ig;
                    ph = ih;
                }
            }
            __syncthreads();
            for (int l = tid; l < n_leaf; l += NT) {
                const int q = l >> 1;
                const bool any = T.segP[q + 1] > T.segP[q];
                const long long RG = any ? T.reG[q] - T.rbG[q] : 0, RH = any ? T.reH[q] - T.rbH[q] : 0;
                const long long NG = any ? T.endG[q] - T.baseG[q] : 0, NH = any ? T.endH[q] - T.baseH[q] : 0;
                const long long LGi = (l & 1) ? RG : NG - RG, LHi = (l & 1) ? RH : NH - RH;
                const double Gd = (double)LGi * FX, Hd = (double)LHi * FX;
                const float v = (float)(-(A.eta * (Gd / (Hd + A.lam))));
                T.lval[l] = v;
                if (blockIdx.x == 0) A.t_leaf[(size_t)t * n_leaf + l] = v;
            }
            __syncthreads();
        }
    }
#ifdef AT_FIT_TIMING
    FT_MARK(4);
    if (threadIdx.x == 0 && getenv_blocks_dump) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        printf("FTBLK %d %u %d %d %llu %llu\n", (int)blockIdx.x, smid, __ldg(A.flist + blockIdx.x),
               A.ncuts[__ldg(A.flist + blockIdx.x)], (ft[2] + ft[5] + ft[6] + ft[7] + ft[8]) / A.n_trees,
               ft[8] / A.n_trees);
    }
    if (threadIdx.x == 0) {
        atomicMax(&g_ft_work_max, ft[2] + ft[5] + ft[6] + ft[7] + ft[8]);
        atomicMax(&g_ft_grad_max, ft[0]);
        __threadfence();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("fused forest ns/tree (block 0, G=%d): grads %llu gsync %llu | levels: work %llu sync %llu | "
               "decide+leaves %llu | max over blocks: grads %llu work %llu (from earlier-finishing blocks)\n", G,
               ft[0] / A.n_trees, ft[1] / A.n_trees, ft[2] / A.n_trees + ft[5] / A.n_trees + ft[6] / A.n_trees +
               ft[7] / A.n_trees + ft[8] / A.n_trees, ft[3] / A.n_trees, ft[4] / A.n_trees,
               g_ft_grad_max / A.n_trees, g_ft_work_max / A.n_trees);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("level work split (ns/tree): partition %llu prefix %llu gains %llu maxima %llu slot+store %llu\n",
               ft[5] / A.n_trees, ft[6] / A.n_trees, ft[8] / A.n_trees, ft[7] / A.n_trees, ft[2] / A.n_trees);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("barrier (last arriver: arrival -> release seen): %llu ns avg over %llu\n",
               g_ft_bar_n ? g_ft_bar_ns / g_ft_bar_n : 0ull, g_ft_bar_n);
#endif
    // the last tree's prediction update
    const int TT = A.n_trees;
    for (int i = blockIdx.x * NT + tid; i < N; i += G * NT)
        A.pred[TT & 1][i] = __fadd_rn(__ldcg(A.pred[(TT - 1) & 1] + i), T.lval[leafof[i]]);
}

__global__ void klist_kernel(const uint16_t *__restrict__ key, const int32_t *__restrict__ rank,
                             const int32_t *__restrict__ woff, int64_t n, int32_t *__restrict__ klist)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) klist[woff[key[i]] + rank[i]] = (int32_t)i;
}

}  // namespace at

namespace {

struct Ws {
    cudaStream_t s;
    std::vector<void *> ptrs;
    int err = 0;
    template <class T> T *get(size_t count)
    {
        void *p = nullptr;
        if (cudaMallocAsync(&p, count * sizeof(T) + 16, s) != cudaSuccess) {
            cudaGetLastError();
            err = AT_ENOMEM;
            return nullptr;
        }
        ptrs.push_back(p);
        return (T *)p;
    }
    ~Ws()
    {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
};

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace at {
// Q40: bootstrap multiset of model `model`: row r <- sample (u * n) >> 32, u = Philox(r, model, round, TAG_BOOT).x
__global__ void bootstrap_kernel(const float *__restrict__ X, int64_t n, int64_t ld, int F, const float *__restrict__ c,
                                 const uint16_t *__restrict__ key, uint32_t model, uint64_t seed, uint32_t round,
                                 float *__restrict__ Xo, int64_t ldo, float *__restrict__ co, uint16_t *__restrict__ ko,
                                 int64_t *__restrict__ io)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const U4 u = philox(seed, (uint32_t)r, model, round, TAG_BOOT);
    const int64_t i = (int64_t)(((uint64_t)u.x * (uint64_t)n) >> 32);
    for (int f = blockIdx.y; f < F; f += gridDim.y) Xo[(int64_t)f * ldo + r] = X[(int64_t)f * ld + i];
    if (blockIdx.y == 0) {
        co[r] = c[i];
        ko[r] = key[i];
        if (io) io[r] = i;
    }
}
}  // namespace at

extern "C" int bootstrap_resample(const float *d_feat, int64_t n, int64_t ld, int32_t F, const float *d_cost,
                                  const uint16_t *d_key, int32_t model, uint64_t seed, uint32_t round,
                                  float *d_feat_out, int64_t ld_out, float *d_cost_out, uint16_t *d_key_out,
                                  int64_t *d_idx_out, void *stream)
{
    using namespace at;
    if (n < 0 || n > 0xFFFFFFFFll || F < 1) return fail(AT_EINVAL, "bootstrap_resample: bad n / n_features");
    if (n == 0) return AT_OK;
    if (!d_feat || !d_cost || !d_key || !d_feat_out || !d_cost_out || !d_key_out)
        return fail(AT_EINVAL, "bootstrap_resample: null buffer");
    if (ld < n || ld_out < n) return fail(AT_EMISMATCH, "bootstrap_resample: ld < n");
    cudaStream_t s = (cudaStream_t)stream;
    const dim3 grid(nblk(n, 256), (unsigned)std::min(F, 64));
    bootstrap_kernel<<<grid, 256, 0, s>>>(d_feat, n, ld, F, d_cost, d_key, (uint32_t)model, seed, round, d_feat_out,
                                          ld_out, d_cost_out, d_key_out, d_idx_out);
    note_launch();
    AT_LAUNCH_CHECK("bootstrap_kernel");
    return AT_OK;
}

extern "C" int gbt_fit_hist(const float *d_feat, int64_t n, int64_t ld, int32_t F, const float *d_cost,
                            const uint16_t *d_group_key, int64_t hb, int64_t he, const at_fit_opts *o, at_gbt *out,
                            void *stream)
{
    using namespace at;
    if (!o || !out) return fail(AT_EINVAL, "gbt_fit_hist: null options/output");
    if (n == 0) return fail(AT_EEMPTY, "gbt_fit_hist: empty training set");
    if (n < 0 || n > 0x7FFFFFFF) return fail(AT_EINVAL, "gbt_fit_hist: bad n");
    if (!d_feat || !d_cost || !d_group_key) return fail(AT_EINVAL, "gbt_fit_hist: null buffer");
    if (ld < n || F < 1 || F > 65535) return fail(AT_EMISMATCH, "gbt_fit_hist: bad ld / n_features");
    if (o->depth < 1 || o->depth > 8) return fail(AT_EUNSUPPORTED, "gbt_fit_hist: depth must be in [1, 8]");
    if (o->max_bins < 2 || o->max_bins > 256) return fail(AT_EUNSUPPORTED, "gbt_fit_hist: max_bins must be in [2, 256]");
    if (o->n_trees < 1 || o->group_size < 2 || o->group_size > 1024) return fail(AT_EINVAL, "gbt_fit_hist: bad n_trees / group_size");
    if (o->objective != AT_OBJ_RANK && o->objective != AT_OBJ_REG) return fail(AT_EINVAL, "gbt_fit_hist: bad objective");
    if (hb < 0 || he < hb || he > n) return fail(AT_EINVAL, "gbt_fit_hist: bad histogram slice");
    if (!o->allreduce && (hb != 0 || he != n)) return fail(AT_EINVAL, "gbt_fit_hist: a slice needs an allreduce");
    cudaStream_t s = (cudaStream_t)stream;
    pool_keep();   // the workspace below is stream-ordered scratch
    const int D = o->depth, B = o->max_bins, GS = o->group_size;
    const int n_int = (1 << D) - 1, n_leaf = 1 << D;
    const double lam = (double)o->lambda, mcw = (double)o->min_child_weight, eta = (double)o->eta;

    Ws ws;
    ws.s = s;
    int32_t *d_info = ws.get<int32_t>(8);
    uint32_t *sortA = ws.get<uint32_t>((size_t)F * n);
    uint32_t *sortB = ws.get<uint32_t>((size_t)F * n);
    float *cuts = ws.get<float>((size_t)F * (B - 1));
    int32_t *ncuts = ws.get<int32_t>(F);
    int32_t *boff = ws.get<int32_t>(F + 1);
    int32_t *flist = ws.get<int32_t>(F);
    uint8_t *bins = ws.get<uint8_t>((size_t)F * n);
    int32_t *rank = ws.get<int32_t>(n);
    int32_t *counts = ws.get<int32_t>(FIT_MAXKEYS);
    int32_t *woff = ws.get<int32_t>(FIT_MAXKEYS);
    int32_t *gpre = ws.get<int32_t>(FIT_MAXKEYS + 1);
    int32_t *member = ws.get<int32_t>(n);
    int64_t *g = ws.get<int64_t>(n);
    int64_t *h = ws.get<int64_t>(n);
    float *pred = ws.get<float>(n);
    int32_t *node = ws.get<int32_t>(n);
    const int max_nn = 1 << (D - 1);
    int64_t *lsum = ws.get<int64_t>((size_t)n_leaf * 2);
    uint8_t *dead = ws.get<uint8_t>(n_int + n_leaf);
    int32_t *split_f = ws.get<int32_t>(n_int);
    int32_t *split_s = ws.get<int32_t>(n_int);
    double *best_gain = ws.get<double>((size_t)max_nn * F);
    int32_t *best_s = ws.get<int32_t>((size_t)max_nn * F);
    uint16_t *t_feat = ws.get<uint16_t>((size_t)o->n_trees * n_int);
    float *t_thr = ws.get<float>((size_t)o->n_trees * n_int);
    float *t_leaf = ws.get<float>((size_t)o->n_trees * n_leaf);
    if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: workspace allocation failed");

    // input checks + cuts + groups.  A single-rank fit (one fused launch for n <= FUSED_NMAX, else the
    // subtraction path laid out on the device) reads every size it needs on the device and never
    // synchronizes; the multi-rank and level-by-level paths read the sizes back once
    const char *fused_e = getenv("AT_FIT_FUSED");   // "0" forces the level-by-level path
    const int fused_env = fused_e ? atoi(fused_e) : 1;
    const bool fused_path = fused_env && !o->allreduce && !o->d_hist0_out && n <= FUSED_NMAX;
    const char *sub_e = getenv("AT_FIT_SUB");   // "0" forces the plain level-by-level path
    const bool multi = o->allreduce != nullptr;
    // histogram subtraction (section 3b) for larger n (any n with AT_FIT_FUSED=0 on one rank); F bounded
    // so every feature range fits SUB_MAXR (nbk <= 256 < SUB_ROWS keeps every stripe in a block's rows)
    const bool sub_path = (!sub_e || atoi(sub_e) != 0) && (!multi || n > FUSED_NMAX) && F <= 32 * SUB_MAXR;
    bool synced = !(fused_path || (sub_path && !multi));
    int info[8] = {0};
    std::vector<int32_t> ncuts_h(F);
    {
        ProfScope ps(AT_K_FIT_PREP, s);
        AT_CUDA_TRY(cudaMemsetAsync(d_info, 0, 8 * sizeof(int32_t), s));
        finite_check_kernel<<<nblk(n, 256), 256, 0, s>>>(d_cost, n, d_info + 2); note_launch();
        key_check_kernel<<<nblk(n, 256), 256, 0, s>>>(d_group_key, n, d_info + 2); note_launch();
        sort_feature_kernel<<<F, 1024, 0, s>>>(d_feat, ld, n, sortA, sortB); note_launch();
        cuts_kernel<<<F, 1024, 0, s>>>(sortA, n, B, cuts, ncuts); note_launch();
        bin_layout_kernel<<<1, 32, 0, s>>>(ncuts, F, boff, d_info, flist); note_launch();
        bins_kernel<<<dim3(nblk(n, 256), F), 256, 0, s>>>(d_feat, ld, n, F, B, cuts, ncuts, bins); note_launch();
        {
            const int nbk = (int)((n + 1023) / 1024);
            int32_t *bc = ws.get<int32_t>((size_t)nbk * FIT_MAXKEYS);
            if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: workspace allocation failed");
            ranks_local_kernel<<<nbk, 1024, 0, s>>>(d_group_key, n, rank, bc); note_launch();
            ranks_scan_kernel<<<1, 1024, 0, s>>>(nbk, bc, counts, woff, gpre, GS); note_launch();
            ranks_add_kernel<<<nblk(n, 256), 256, 0, s>>>(d_group_key, n, bc, rank); note_launch();
        }
        AT_CUDA_TRY(cudaMemcpyAsync(d_info + 3, gpre + FIT_MAXKEYS, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        if (o->d_base_margin)   // initial predictions: f_global(x_i) for a transfer-learning fit (Eq. 4)
            AT_CUDA_TRY(cudaMemcpyAsync(pred, o->d_base_margin, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
        else
            AT_CUDA_TRY(cudaMemsetAsync(pred, 0, sizeof(float) * n, s));
        AT_LAUNCH_CHECK("fit prep");
    }
    if (synced) {
        AT_CUDA_TRY(cudaMemcpyAsync(info, d_info, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        AT_CUDA_TRY(cudaMemcpyAsync(ncuts_h.data(), ncuts, F * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        AT_CUDA_TRY(cudaStreamSynchronize(s));
        if (info[2] == 1) return fail(AT_EINVAL, "gbt_fit_hist: non-finite cost");
        if (info[2] == 2) return fail(AT_EUNSUPPORTED, "gbt_fit_hist: group key >= 1024");
    }
    // (read back below for the paths that need them on the host)
    int TB = info[0], max_nb = info[1], n_groups = info[3];
    // the fitted ensemble handle (both paths)
    auto finish = [&]() -> int {
        // the fitted ensemble handle
        at_gbt gm = new at_gbt_s();
        gm->n_trees = o->n_trees;
        gm->depth = D;
        gm->n_features = F;
        gm->t_pad = (o->n_trees + 15) / 16 * 16;
        gm->base = 0.0f;
        gm->d_nodes = nullptr;
        gm->d_leaf = nullptr;
        gm->last = s;
        if (cudaMallocAsync((void **)&gm->d_nodes, sizeof(uint2) * (size_t)gm->t_pad * n_int, s) != cudaSuccess ||
            cudaMallocAsync((void **)&gm->d_leaf, sizeof(float) * (size_t)gm->t_pad * n_leaf, s) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeAsync(gm->d_nodes, s);
            delete gm;
            return fail(AT_ENOMEM, "gbt_fit_hist: model allocation failed");
        }
        AT_CUDA_TRY(cudaMemsetAsync(gm->d_nodes, 0, sizeof(uint2) * (size_t)gm->t_pad * n_int, s));
        AT_CUDA_TRY(cudaMemsetAsync(gm->d_leaf, 0, sizeof(float) * (size_t)gm->t_pad * n_leaf, s));
        pack_nodes_kernel<<<nblk((int64_t)o->n_trees * n_int, 256), 256, 0, s>>>(t_feat, t_thr, (int64_t)o->n_trees * n_int,
                                                                                 gm->d_nodes); note_launch();
        AT_CUDA_TRY(cudaMemcpyAsync(gm->d_leaf, t_leaf, sizeof(float) * (size_t)o->n_trees * n_leaf,
                                    cudaMemcpyDeviceToDevice, s));
        if (o->d_pred_out) AT_CUDA_TRY(cudaMemcpyAsync(o->d_pred_out, pred, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
        if (!synced) {   // input flags found on the device travel with the model (at_gbt_s::h_err)
            if (cudaHostAlloc((void **)&gm->h_err, sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess) {
                cudaGetLastError();
                gm->h_err = nullptr;
                gbt_destroy(gm);
                return fail(AT_ENOMEM, "gbt_fit_hist: mapped error word allocation failed");
            }
            *gm->h_err = 0u;
            uint32_t *d_err = nullptr;
            AT_CUDA_TRY(cudaHostGetDevicePointer((void **)&d_err, gm->h_err, 0));
            fit_flag_kernel<<<1, 1, 0, s>>>(d_info, d_err); note_launch();
        }
        AT_LAUNCH_CHECK("fit finish");
        *out = gm;
        return AT_OK;
    };

    // small single-rank fits: the whole forest in one cooperative launch (fused_forest_kernel), sized for
    // all F features (the splittable ones are known only on the device)
    if (fused_path) {
        int dev = 0, nsm = 0, coop = 0, per = 0;
        AT_CUDA_TRY(cudaGetDevice(&dev));
        AT_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        AT_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        const int nF = F;   // an upper bound of the splittable features (blocks own them; the rest idle)
        // the kernel variant: 512 threads per block when every splittable feature still gets its own
        // resident block at 2 blocks / SM, else 256 threads (4 / SM)
        const void *fk = nullptr;
        int NT = 512, fep = 1;
        size_t fsm = 0;
        static size_t fused_attr[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        static int trim_env = -1;
        if (trim_env < 0) {
            const char *e = getenv("AT_FIT_NT_TRIM");   // "0": keep 256 threads at 8 positions each
            trim_env = e ? atoi(e) : 1;
        }
        for (int pass = 0; pass < 2; ++pass) {
            NT = pass == 0 ? 512 : 256;
            fep = fused_ep((int)n, NT);
            fsm = fused_smem_bytes((int)n, GS);
            int fslot = (pass == 0 ? 0 : 4) + (fep == 1 ? 0 : fep == 2 ? 1 : fep == 4 ? 2 : 3);
            if (NT == 512)
                fk = fep == 1 ? (const void *)fused_forest_kernel<1, 512> : fep == 2 ? (const void *)fused_forest_kernel<2, 512>
                   : (const void *)fused_forest_kernel<4, 512>;
            else
                fk = fep == 1   ? (const void *)fused_forest_kernel<1, 256> : fep == 2 ? (const void *)fused_forest_kernel<2, 256>
                   : fep == 4 ? (const void *)fused_forest_kernel<4, 256> : (const void *)fused_forest_kernel<8, 256>;
            if (NT == 256 && fep == 8 && trim_env) {
                // 8 positions per thread: only ceil(n / 256) warps hold positions (1536 -> 6 of 8); drop the
                // idle warps, whose block barriers and scans are pure overhead
                const int nt = (int)((n + 255) / 256) * 32;
                if (nt < 256) {
                    NT = nt;
                    fk = nt == 160 ? (const void *)fused_forest_kernel<8, 160> : nt == 192 ? (const void *)fused_forest_kernel<8, 192>
                       : (const void *)fused_forest_kernel<8, 224>;
                    fslot = 8 + (nt / 32 - 5);
                }
            }
            if (fused_attr[fslot] < fsm) {
                AT_CUDA_TRY(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
                fused_attr[fslot] = fsm;
            }
            AT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fk, NT, fsm));
            // 512 threads while they keep 2 blocks per SM (n <= 1024): 296 resident blocks hold the
            // splittable features of typical databases (config 2: 284); the count itself is only known on
            // the device, which falls back to blocks walking several features when it is larger
            if (pass == 0 && per > 0 && (nF <= per * nsm || per >= 2)) break;
        }
        if (coop && per > 0) {
            // blocks for the splittable features only (all constant: one block on feature 0, which has no
            // cut, so every node stays a pass-through and the leaves are the node totals)
            const int G = (int)std::min<int64_t>(nF, (int64_t)per * nsm);
            const bool resident = nF <= G;
            int32_t *klist = ws.get<int32_t>(n);
            unsigned long long *slot = ws.get<unsigned long long>((size_t)2 * 2 * FUSED_NSUB * n_int);   // 2 tree parities
            unsigned *bar = ws.get<unsigned>(32);
            uint16_t *gord = resident ? nullptr : ws.get<uint16_t>((size_t)F * n);
            uint16_t *gord0 = ws.get<uint16_t>((size_t)F * n);   // initial bin-sorted orders
            uint8_t *gnode = resident ? nullptr : ws.get<uint8_t>((size_t)F * n);
            if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: workspace allocation failed");
            AT_CUDA_TRY(cudaMemsetAsync(bar, 0, 32 * sizeof(unsigned), s));
            AT_CUDA_TRY(cudaMemsetAsync(slot, 0, sizeof(unsigned long long) * 2 * 2 * FUSED_NSUB * n_int, s));
            klist_kernel<<<nblk(n, 256), 256, 0, s>>>(d_group_key, rank, woff, n, klist); note_launch();
            AT_LAUNCH_CHECK("klist");
            FusedArgs fa;
            fa.bins = bins; fa.ncuts = ncuts; fa.cuts = cuts; fa.B = B;
            fa.flist = flist; fa.info = d_info;
            fa.n = (int)n; fa.F = F; fa.D = D; fa.n_trees = o->n_trees; fa.GS = GS;
            fa.counts = counts; fa.woff = woff; fa.gpre = gpre; fa.klist = klist;
            float *pred2 = ws.get<float>(n);
            if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: workspace allocation failed");
            fa.cost = d_cost; fa.g = g; fa.h = h;
            fa.pred[0] = (o->n_trees & 1) ? pred2 : pred;   // the final predictions land in pred
            fa.pred[1] = (o->n_trees & 1) ? pred : pred2;
            if (fa.pred[0] != pred)   // pred[0] holds the initial predictions (tree 0 reads them)
                AT_CUDA_TRY(cudaMemcpyAsync(fa.pred[0], pred, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
            fa.objective = o->objective;
            fa.gord = gord; fa.gord0 = gord0; fa.gnode = gnode; fa.slot = slot;
            fa.t_feat = t_feat; fa.t_thr = t_thr; fa.t_leaf = t_leaf;
            fa.seed = o->seed; fa.lam = lam; fa.mcw = mcw; fa.eta = eta; fa.bar = bar;
            void *args[] = {&fa};
            {
                ProfScope ps(AT_K_FIT_GRAPH, s);
                AT_CUDA_TRY(cudaLaunchCooperativeKernel(fk, dim3(G), dim3(NT), args,
                                                        fsm, s));
                note_launch();
            }
            return finish();
        }
    }

    if (fused_path && !sub_path) {   // no cooperative launch possible: the sizes are read back after all
        AT_CUDA_TRY(cudaMemcpyAsync(info, d_info, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        AT_CUDA_TRY(cudaMemcpyAsync(ncuts_h.data(), ncuts, F * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        AT_CUDA_TRY(cudaStreamSynchronize(s));
        synced = true;
        if (info[2] == 1) return fail(AT_EINVAL, "gbt_fit_hist: non-finite cost");
        if (info[2] == 2) return fail(AT_EUNSUPPORTED, "gbt_fit_hist: group key >= 1024");
        TB = info[0];
        max_nb = info[1];
        n_groups = info[3];
    }
    // a single-rank fit has no host callback between levels: its launches are captured once into a
    // CUDA graph and launched as one unit (no host round trips for ~10 launches per level)
    auto run_captured = [&](auto &&enqueue, int reps) -> int {
        static thread_local cudaStream_t cs = nullptr;
        if (!cs) AT_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        prof_suspend(true);
        cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) { prof_suspend(false); return cuda_fail(e, "gbt_fit_hist: begin capture"); }
        const int rc = enqueue(cs);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(cs, &graph);
        prof_suspend(false);
        if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
        if (e != cudaSuccess) return cuda_fail(e, "gbt_fit_hist: end capture");
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(e, "gbt_fit_hist: graph instantiate");
        {
            ProfScope ps(AT_K_FIT_GRAPH, s);
            for (int r = 0; r < reps && e == cudaSuccess; ++r) e = cudaGraphLaunch(exec, s);
        }
        cudaGraphExecDestroy(exec);
        if (e != cudaSuccess) return cuda_fail(e, "gbt_fit_hist: graph launch");
        return AT_OK;
    };

    // histogram subtraction over node-contiguous positions (section 3b).  The layout (splittable
    // features, bank-column stripes, split entries, TB) is computed on the device by sub_layout_kernel and
    // every launch below is sized by an upper bound of it, so one rank never reads anything back.  With R
    // ranks every rank keeps the whole (replicated) partition and builds the smaller children's histograms
    // over its own sample slice [hb, he) only; one int64 all-reduce per level (the dense smaller-children
    // buffer, sized by the cut counts TB read back above) makes them global, so every decision is
    // replicated exactly.
    if (sub_path) {
        int dev = 0, nsm = 0;
        AT_CUDA_TRY(cudaGetDevice(&dev));
        AT_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const int NR_max = (F + 31) / 32;                     // a range holds >= min(32, rest) features
        const int FsP_max = F + 128 * NR_max;                 // each range's bytes padded to 128
        const int NE_max = F * std::max(1, (B + 30) / 32);    // (feature, 32-split chunk) entries
        const int64_t TB_cap = synced ? (int64_t)TB : (int64_t)F * B;
        const int max_items = nsm + max_nn + 1;               // target (<= nsm) root chunks, + nn per level
        uint8_t *binsR = ws.get<uint8_t>((size_t)n * FsP_max);
        int32_t *perm = ws.get<int32_t>(n);
        int32_t *d_tab = ws.get<int32_t>(3 * (size_t)F + FsP_max);   // rowbase, gbase, nbk, inv
        SubRange *d_rng = ws.get<SubRange>(NR_max);
        SubDev *d_L = ws.get<SubDev>(1);
        int32_t *d_ent = ws.get<int32_t>(2 * (size_t)NE_max);   // [feature of entry][chunk of entry]
        int4 *items = ws.get<int4>(max_items);
        int4 *subs = ws.get<int4>(max_nn + 1);
        int32_t *cnts = ws.get<int32_t>(4);   // [0] n_items, [1] n_subs, [2] n_units
        int32_t *cursor = ws.get<int32_t>(2 * max_nn);
        int32_t *seg_start = ws.get<int32_t>(n_int + n_leaf);
        int32_t *seg_cnt = ws.get<int32_t>(n_int + n_leaf);
        int64_t *tot = ws.get<int64_t>(2 * (size_t)(n_int + n_leaf));
        int64_t *hA = ws.get<int64_t>((size_t)max_nn * TB_cap * 2);
        int64_t *hB = ws.get<int64_t>((size_t)max_nn * TB_cap * 2);
        int64_t *hS = multi ? ws.get<int64_t>((size_t)max_nn * TB * 2) : nullptr;   // dense smaller children
        double *bg = ws.get<double>((size_t)max_nn * NE_max);
        int32_t *bs = ws.get<int32_t>((size_t)max_nn * NE_max);
        int32_t *d_tree = ws.get<int32_t>(1);
        int4 *root_items = ws.get<int4>(max_items);
        const int wu_root = std::max(nsm, NR_max);   // root units <= target NR <= max(nsm, NR)
        SubUnit *units = ws.get<SubUnit>((size_t)wu_root + (size_t)max_nn * NR_max);   // + nn NR per level
        SubUnit *root_units = ws.get<SubUnit>(wu_root);
        int32_t *root_n = ws.get<int32_t>(4);
        unsigned *done = ws.get<unsigned>(2 + max_nn);   // last-block counter of the scatter, per-node split counters
        if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: workspace allocation failed");
        // a range's rows <= max(rows_cap, B) (its first stripe always goes in; a stripe of one feature
        // each takes <= B rows): the shared histogram is sized by that bound
        const char *rc_e = getenv("AT_SUB_ROWS");
        const int rows_cap = std::min(SUB_ROWS, std::max(B, rc_e ? atoi(rc_e) : SUB_ROWS_DEF));
        const size_t hsm = (size_t)4 * 32 * (std::max(rows_cap, B) + 1) * sizeof(uint32_t);
        int32_t *d_rowbase = d_tab, *d_gbase = d_tab + F, *d_nbk = d_tab + 2 * F, *d_inv = d_tab + 3 * F;
        sub_layout_kernel<<<1, 256, 0, s>>>(ncuts, boff, F, flist, d_rowbase, d_gbase, d_nbk, d_inv, FsP_max, d_rng,
                                            d_ent, d_ent + NE_max, nsm, rows_cap, d_L);
        note_launch();
        rowbins_kernel<<<dim3(nblk(n, 32), std::min(4u, nblk(FsP_max, 32))), dim3(32, 8), 0, s>>>(bins, n, flist, d_inv,
                                                                                                  d_L, binsR);
        note_launch();
        AT_LAUNCH_CHECK("layout/rowbins");
        static size_t sub_attr = 0;
        if (sub_attr < hsm) {
            AT_CUDA_TRY(cudaFuncSetAttribute(sub_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
            sub_attr = hsm;
        }
        // one tree is captured once and its graph launched n_trees times: the tree index lives on the
        // device (d_tree, advanced by the graph's last node), so the host cost per fit is one capture
        AT_CUDA_TRY(cudaMemsetAsync(d_tree, 0, sizeof(int32_t), s));
        AT_CUDA_TRY(cudaMemsetAsync(done, 0, (2 + max_nn) * sizeof(unsigned), s));
        AT_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * 2 * max_nn, s));
        AT_CUDA_TRY(cudaMemsetAsync(node, 0, sizeof(int32_t) * n, s));
        AT_CUDA_TRY(cudaMemsetAsync(dead, 0, n_int + n_leaf, s));
        // spare histogram blocks read a unit past the count before they exit: keep it initialised
        AT_CUDA_TRY(cudaMemsetAsync(units, 0, sizeof(SubUnit) * ((size_t)wu_root + (size_t)max_nn * NR_max), s));
        AT_CUDA_TRY(cudaMemsetAsync(root_units, 0, sizeof(SubUnit) * (size_t)wu_root, s));
        sub_zero_kernel<<<2 * nsm, 256, 0, s>>>(hA, d_L, 1);   // tree 0's root (each tree zeroes the next one's)
        note_launch();
        sub_root_items_kernel<<<1, 256, 0, s>>>((int)hb, (int)he, d_L, root_items, d_rng, root_units, root_n);
        note_launch();
        // group count bounded by n / GS + one partial group per present key
        const int grad_grid = synced ? n_groups : (int)(n / GS + std::min<int64_t>(n, FIT_MAXKEYS));
        auto enqueue_sub = [&](cudaStream_t s) -> int {
            {
                ProfScope ps(AT_K_FIT_GRAD, s);
                if (o->objective == AT_OBJ_REG) {
                    reg_grads_kernel<<<nblk(n, 256), 256, 0, s>>>(d_cost, pred, n, g, h); note_launch();
                } else {
                    positions_kernel<<<nblk(n, 256), 256, 0, s>>>(d_group_key, rank, counts, woff, n, o->seed, 0u,
                                                                  member, d_tree); note_launch();
                    if (grad_grid > 0) {
                        grads_kernel<<<grad_grid, 256, (size_t)GS * 2 * sizeof(float), s>>>(member, counts, woff, gpre,
                                                                                            GS, d_cost, pred, g, h);
                        note_launch();
                    }
                }
                AT_LAUNCH_CHECK("fit gradients");
            }
            int64_t *hp = hA, *hc = hB;   // node[] and dead[] were zeroed by the previous tree (or below)
            {
                ProfScope ps(AT_K_FIT_HIST, s);
                sub_hist_kernel<<<wu_root, SUB_NT, hsm, s>>>(binsR, d_L, nullptr, g, h, root_units, root_n,
                                                             d_rowbase, d_gbase, d_nbk, hp, (int)hb, (int)he);
                note_launch();
                AT_LAUNCH_CHECK("root histogram");
                if (multi && o->allreduce(hp, 2 * (int64_t)TB, o->ctx, stream))
                    return fail(AT_ECUDA, "gbt_fit_hist: allreduce callback failed");
                const int want_h0 = o->d_hist0_out != nullptr;
                sub_root_tot_kernel<<<1, 256, 0, s>>>(hp, boff, flist, F, (int)(he - hb), want_h0, tot, seg_start, seg_cnt,
                                                      d_tree); note_launch();
                if (want_h0) {
                    hist0_expand_kernel<<<nblk((int64_t)F * B, 256), 256, 0, s>>>(hp, boff, F, B, o->d_hist0_out,
                                                                                 d_tree);
                    note_launch();
                }
                AT_LAUNCH_CHECK("root histogram");
            }
            for (int d = 0; d < D; ++d) {
                const int first = (1 << d) - 1, nn = 1 << d;
                {
                    ProfScope ps(AT_K_FIT_SPLIT, s);
                    sub_split_kernel<<<std::min<unsigned>(nblk((int64_t)nn * NE_max, 8), 8 * nsm), 256, 0, s>>>(
                        hp, boff, d_ent, d_ent + NE_max, d_L, first, nn, tot, lam, mcw, dead, bg, bs, cuts, B, split_f,
                        split_s, t_feat, t_thr, n_int, d_tree, done + 2);
                    note_launch();
                    AT_LAUNCH_CHECK("split/decide");
                }
                if (d == D - 1) break;
                {
                    ProfScope ps(AT_K_FIT_SPLIT, s);
                    sub_scatter_kernel<<<nblk(n, 256), 256, 0, s>>>(bins, n, split_f, split_s, first, nn, seg_start,
                                                                    seg_cnt, cursor, node, perm, d_L, items, cnts,
                                                                    subs, cnts + 1, done + 1, multi ? 1 : 0, tot,
                                                                    (int)hb, (int)he, d_rng, units, cnts + 2,
                                                                    multi ? hS : hc, multi ? nn : 2 * nn);
                    note_launch();
                    AT_LAUNCH_CHECK("scatter");
                }
                if (multi) {
                    {
                        ProfScope ps(AT_K_FIT_HIST, s);
                        sub_hist_kernel<<<wu_root + nn * NR_max, SUB_NT, hsm, s>>>(binsR, d_L, perm, g, h, units, cnts + 2,
                                                                                   d_rowbase, d_gbase, d_nbk, hS,
                                                                                   (int)hb, (int)he);
                        note_launch();
                        AT_LAUNCH_CHECK("histograms");
                    }
                    if (o->allreduce(hS, 2 * (int64_t)TB * nn, o->ctx, stream))
                        return fail(AT_ECUDA, "gbt_fit_hist: allreduce callback failed");
                    {
                        ProfScope ps(AT_K_FIT_HIST, s);
                        sub_expand_kernel<<<dim3(64, nn), 256, 0, s>>>(hp, hS, hc, d_L, subs, cnts + 1);
                        note_launch();
                        AT_LAUNCH_CHECK("expand");
                    }
                    std::swap(hp, hc);
                    continue;
                }
                {
                    ProfScope ps(AT_K_FIT_HIST, s);
                    sub_hist_kernel<<<wu_root + nn * NR_max, SUB_NT, hsm, s>>>(binsR, d_L, perm, g, h, units, cnts + 2,
                                                                               d_rowbase, d_gbase, d_nbk, hc, 0, (int)n);
                    note_launch();
                    sub_subtract_kernel<<<dim3(64, nn), 256, 0, s>>>(hp, hc, d_L, subs, cnts + 1);
                    note_launch();
                    AT_LAUNCH_CHECK("histograms");
                }
                std::swap(hp, hc);
            }
            {
                ProfScope ps(AT_K_FIT_UPDATE, s);
                sub_leaf_kernel<<<nblk(n_leaf, 256), 256, 0, s>>>(tot + 2 * (size_t)n_int, n_leaf, eta, lam, t_leaf,
                                                                  d_tree, dead, n_int + n_leaf);
                note_launch();
                sub_final_kernel<<<nblk(n, 256), 256, 0, s>>>(bins, n, node, split_f, split_s, n_int, t_leaf, pred,
                                                              d_tree, hA, d_L);
                note_launch();
                sub_tree_next_kernel<<<1, 1, 0, s>>>(d_tree);
                note_launch();
                AT_LAUNCH_CHECK("leaf/pred update");
            }
            return AT_OK;
        };
        if (multi) {   // host callbacks between levels: enqueued tree by tree (the tree index is on the device)
            for (int t = 0; t < o->n_trees; ++t) {
                const int rc = enqueue_sub(s);
                if (rc) return rc;
            }
        } else {
            const int rc = run_captured(enqueue_sub, o->n_trees);
            if (rc) return rc;
        }
        return finish();
    }

    int64_t *hist = ws.get<int64_t>((size_t)max_nn * TB * 2);
    if (ws.err) return fail(AT_ENOMEM, "gbt_fit_hist: histogram allocation failed");

    const size_t grad_smem = (size_t)GS * 2 * sizeof(float);
    const int64_t ns = he - hb;
    const int64_t n_chunks = ns <= 4096 ? 1 : std::min<int64_t>((ns + 4095) / 4096, 64);
    const int64_t chunk = n_chunks ? (ns + n_chunks - 1) / n_chunks : 0;
    static size_t hist_attr = 0;
    if (hist_attr == 0) {
        AT_CUDA_TRY(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        AT_CUDA_TRY(cudaFuncSetAttribute(hist_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        hist_attr = 160 * 1024;
    }
    // all trees are enqueued by one function; a single-rank fit (no host callback between levels) is
    // captured once into a CUDA graph and launched as one unit, so ~15 launches per tree cost no host
    // round trips.
    auto enqueue_trees = [&](cudaStream_t s) -> int {
        for (int t = 0; t < o->n_trees; ++t) {
            {
                ProfScope ps(AT_K_FIT_GRAD, s);
                if (o->objective == AT_OBJ_REG) {
                    reg_grads_kernel<<<nblk(n, 256), 256, 0, s>>>(d_cost, pred, n, g, h); note_launch();
                } else {
                    positions_kernel<<<nblk(n, 256), 256, 0, s>>>(d_group_key, rank, counts, woff, n, o->seed,
                                                                  (uint32_t)t, member); note_launch();
                    if (n_groups > 0) {
                        grads_kernel<<<n_groups, 256, grad_smem, s>>>(member, counts, woff, gpre, GS, d_cost, pred, g,
                                                                      h);
                        note_launch();
                    }
                }
                AT_LAUNCH_CHECK("fit gradients");
            }
            AT_CUDA_TRY(cudaMemsetAsync(node, 0, sizeof(int32_t) * n, s));
            AT_CUDA_TRY(cudaMemsetAsync(dead, 0, n_int + n_leaf, s));
            uint16_t *tf = t_feat + (size_t)t * n_int;
            float *tt = t_thr + (size_t)t * n_int;
            for (int d = 0; d < D; ++d) {
                const int first = (1 << d) - 1, nn = 1 << d;
                const size_t cells = (size_t)nn * TB * 2;
                const size_t smem = (size_t)nn * max_nb * 2 * sizeof(int64_t);
                const int use_smem = smem <= 160 * 1024;
                const bool want_h0 = t == 0 && d == 0 && o->d_hist0_out;
                if (!o->allreduce && use_smem) {
                    // single rank: histograms stay in shared memory, split scan fused
                    {
                        ProfScope ps(AT_K_FIT_HIST, s);
                        hist_split_kernel<<<F, 256, smem, s>>>(bins, node, g, h, n, boff, F, first, nn, lam, mcw, dead,
                                                               best_gain, best_s, want_h0 ? hist : nullptr); note_launch();
                        AT_LAUNCH_CHECK("hist_split_kernel");
                    }
                    if (want_h0) {
                        hist0_expand_kernel<<<nblk((int64_t)F * B, 256), 256, 0, s>>>(hist, boff, F, B,
                                                                                     o->d_hist0_out);
                        note_launch();
                    }
                    ProfScope ps(AT_K_FIT_SPLIT, s);
                    if (n <= 65536 && nn <= 64) {
                        decide_partition_kernel<<<nblk(n, 256), 256, 0, s>>>(best_gain, best_s, F, first, nn, cuts, B,
                                                                            dead, split_f, split_s, tf, tt, bins, n,
                                                                            node); note_launch();
                    } else {
                        split_node_kernel<<<nn, 256, 0, s>>>(best_gain, best_s, F, first, nn, cuts, B, dead,
                                                             split_f, split_s, tf, tt); note_launch();
                        partition_kernel<<<nblk(n, 256), 256, 0, s>>>(bins, n, split_f, split_s, node); note_launch();
                    }
                    AT_LAUNCH_CHECK("split/partition");
                    continue;
                }
                {
                    ProfScope ps(AT_K_FIT_HIST, s);
                    if (n_chunks != 1 || !use_smem || ns == 0)
                        AT_CUDA_TRY(cudaMemsetAsync(hist, 0, cells * sizeof(int64_t), s));
                    if (ns > 0) {
                        hist_kernel<<<dim3(F, (unsigned)n_chunks), 256, use_smem ? smem : 0, s>>>(
                            bins, node, g, h, hb, he, n, chunk, boff, TB, first, nn, use_smem, hist);
                        note_launch();
                    }
                    AT_LAUNCH_CHECK("hist_kernel");
                }
                if (o->allreduce) {
                    const int rc = o->allreduce(hist, (int64_t)cells, o->ctx, stream);
                    if (rc) return fail(AT_ECUDA, "gbt_fit_hist: allreduce callback failed");
                }
                if (want_h0) {
                    hist0_expand_kernel<<<nblk((int64_t)F * B, 256), 256, 0, s>>>(hist, boff, F, B, o->d_hist0_out);
                    note_launch();
                }
                {
                    ProfScope ps(AT_K_FIT_SPLIT, s);
                    split_feature_kernel<<<nblk((int64_t)nn * F, 8), 256, 0, s>>>(hist, boff, TB, F, first, nn, lam,
                                                                                  mcw, dead, best_gain, best_s); note_launch();
                    split_node_kernel<<<nn, 256, 0, s>>>(best_gain, best_s, F, first, nn, cuts, B, dead, split_f, split_s,
                                                         tf, tt); note_launch();
                    partition_kernel<<<nblk(n, 256), 256, 0, s>>>(bins, n, split_f, split_s, node); note_launch();
                    AT_LAUNCH_CHECK("split/partition");
                }
            }
            {
                ProfScope ps(AT_K_FIT_UPDATE, s);
                AT_CUDA_TRY(cudaMemsetAsync(lsum, 0, sizeof(int64_t) * 2 * n_leaf, s));
                if (he > hb) { leafsum_kernel<<<nblk(he - hb, 256), 256, 0, s>>>(node, g, h, hb, he, n_int, lsum); note_launch(); }
                AT_LAUNCH_CHECK("leafsum");
            }
            if (o->allreduce) {
                const int rc = o->allreduce(lsum, (int64_t)2 * n_leaf, o->ctx, stream);
                if (rc) return fail(AT_ECUDA, "gbt_fit_hist: allreduce callback failed");
            }
            {
                ProfScope ps(AT_K_FIT_UPDATE, s);
                float *tl = t_leaf + (size_t)t * n_leaf;
                leaf_kernel<<<nblk(n_leaf, 256), 256, 0, s>>>(lsum, n_leaf, eta, lam, tl); note_launch();
                pred_update_kernel<<<nblk(n, 256), 256, 0, s>>>(node, n, n_int, tl, pred); note_launch();
                AT_LAUNCH_CHECK("leaf/pred update");
            }
        }
        return AT_OK;
    };
    if (o->allreduce) {
        const int rc = enqueue_trees(s);
        if (rc) return rc;
    } else {
        const int rc = run_captured(enqueue_trees, 1);
        if (rc) return rc;
    }
    return finish();
}
