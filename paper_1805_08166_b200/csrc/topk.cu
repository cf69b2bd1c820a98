// topk.cu -- distinct top-K of collected candidates (a7; Alg. 1 P:152 "collect candidates",
// reading Q23: unique by idx, measured excluded, ordered by (E asc, idx asc)).
//
// A candidate is the 64-bit key (order-preserving bits of E) << 32 | local idx, so the
// (E, idx) order is plain u64 order and -- because E is a function of idx -- duplicates
// of a configuration are equal keys.  Every block sorts a 4096-key tile in shared
// memory (bitonic), drops repeats and keeps its K smallest distinct keys; the
// per-block lists are reduced again by the same kernel until one list remains.  The
// K smallest distinct keys of a union are always inside the union of the per-part
// K smallest distinct keys, so the result is exact and independent of the tiling.
#include "at_common.cuh"
#include "topk.cuh"

#include <algorithm>

namespace at {

constexpr int TK_TILE = 4096;
constexpr int TK_THREADS = 1024;
constexpr uint64_t KEY_NONE = ~0ull;

__device__ __forceinline__ bool in_sorted(const uint64_t *__restrict__ a, int64_t n, uint64_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && __ldg(a + lo) == v;
}

// mode 0: raw SA keys [steps + 1][n_chains] filtered by chain workload == w and not measured
// mode 1: lists [n_lists][n_w][k_in] of (idx, score) with counts, workload w, not measured
// mode 2: partial key lists (already filtered), plain reduction
struct TkSrc {
    int mode;
    const uint64_t *keys;
    int64_t n;               // number of source keys (mode 0: (steps+1)*n_chains; 1: n_lists*k_in; 2: count)
    int64_t n_chains;
    const uint16_t *chain_w;
    const int32_t *chain_list, *list_n;
    int w;
    uint64_t offset_w;
    const uint64_t *l_idx;
    const float *l_score;
    const int32_t *l_n;
    int n_w, k_in;
    const uint64_t *measured;
    int64_t n_measured;
    // batched over workloads (blockIdx.y = workload w + y): per-y strides of the mode-2 input keys and
    // of the chain lists, and every workload's index offset
    int64_t key_stride, list_stride;
    uint64_t offsets[MAXW];
    const int32_t *fb;       // nullable: per batch row y, 0 = the threshold fast path already wrote it (skip)
};

// the block's view of its workload (blockIdx.y)
struct TkW {
    int w;
    uint64_t offset_w;
    const uint64_t *keys;
    const int32_t *chain_list;
};

__device__ __forceinline__ uint64_t tk_load(const TkSrc &S, const TkW &V, int64_t i)
{
    if (i >= S.n) return KEY_NONE;
    if (S.mode == 2) return __ldg(V.keys + i);
    uint64_t key, gidx;
    if (S.mode == 0 && V.chain_list) {
        // the workload's own chains only: i = step * cnt + j
        const int64_t cnt = __ldg(S.list_n + V.w);
        if (cnt == 0) return KEY_NONE;
        const int64_t st = i / cnt, j = i - st * cnt;
        if (st * S.n_chains >= S.n) return KEY_NONE;
        key = __ldg(S.keys + st * S.n_chains + __ldg(V.chain_list + j));
        gidx = V.offset_w + (key & 0xFFFFFFFFull);
    } else if (S.mode == 0) {
        const int64_t c = i % S.n_chains;
        if (S.chain_w && (int)__ldg(S.chain_w + c) != V.w) return KEY_NONE;
        key = __ldg(S.keys + i);
        gidx = V.offset_w + (key & 0xFFFFFFFFull);
    } else {
        const int64_t l = i / S.k_in, j = i - l * S.k_in;
        if (j >= __ldg(S.l_n + l * S.n_w + V.w)) return KEY_NONE;
        const int64_t at = (l * S.n_w + V.w) * S.k_in + j;
        gidx = __ldg(S.l_idx + at);
        key = ((uint64_t)fkey(__ldg(S.l_score + at)) << 32) | (uint64_t)(gidx - V.offset_w);
    }
    (void)gidx;   // measured configurations are dropped after the tile's sort (see topk_tile_kernel)
    return key;
}

__global__ void __launch_bounds__(TK_THREADS) topk_tile_kernel(TkSrc S, int K, uint64_t *__restrict__ out,
                                                               int64_t out_stride)
{
    if (S.fb && !S.fb[blockIdx.y]) return;   // this workload was resolved by the fast path
    TkW V;
    V.w = S.w + (int)blockIdx.y;
    V.offset_w = S.offsets[V.w];
    V.keys = S.keys + (int64_t)blockIdx.y * S.key_stride;
    V.chain_list = S.chain_list ? S.chain_list + (int64_t)blockIdx.y * S.list_stride : nullptr;
    out += (int64_t)blockIdx.y * out_stride;
    __shared__ uint64_t s[TK_TILE];
    __shared__ int wsum[TK_THREADS / 32];
    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * TK_TILE;
    int anyv = 0;
    for (int i = tid; i < TK_TILE; i += TK_THREADS) {
        s[i] = tk_load(S, V, base + i);
        anyv |= s[i] != KEY_NONE;
    }
    if (!__syncthreads_or(anyv)) {   // an empty tile (other workloads' chains, padding lists): empty list
        for (int i = tid; i < K; i += TK_THREADS) out[(int64_t)blockIdx.x * K + i] = KEY_NONE;
        return;
    }
    for (int k = 2; k <= TK_TILE; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < TK_TILE; i += TK_THREADS) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
    // distinct: keep keys that differ from their predecessor
    constexpr int PER = TK_TILE / TK_THREADS;   // 4 consecutive keys per thread
    const int lane = tid & 31, warp = tid >> 5;
    uint64_t v[PER];
    int flag[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int i = tid * PER + q;
        v[q] = s[i];
        flag[q] = (v[q] != KEY_NONE) && (i == 0 || s[i - 1] != v[q]);
    }
    // block exclusive scan of per-thread counts; returns this thread's offset, total in *tot
    auto scan = [&](int c, int *tot) {
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += y;
        }
        __syncthreads();   // wsum reuse
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int x = wsum[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
                if (lane >= off) x += y;
            }
            wsum[lane] = x;   // inclusive
        }
        __syncthreads();
        *tot = wsum[31];
        return incl - c + (warp > 0 ? wsum[warp - 1] : 0);
    };
    // measured configurations: checked only for the distinct keys that can reach the first K --
    // ranks [0, K), then [K, K + m) for the m measured among those, ... (rarely more than one round)
    if (S.n_measured && S.mode != 2) {
        int c0 = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) c0 += flag[q];
        int tot;
        const int r0 = scan(c0, &tot);
        __shared__ int s_m;
        int lo = 0, hi = K;
        while (lo < tot) {
            if (tid == 0) s_m = 0;
            __syncthreads();
            int r = r0, m = 0;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                if (flag[q]) {
                    if (r >= lo && r < hi && in_sorted(S.measured, S.n_measured, V.offset_w + (v[q] & 0xFFFFFFFFull))) {
                        flag[q] = 2;   // measured: dropped below
                        ++m;
                    }
                    ++r;
                }
            }
            if (m) atomicAdd(&s_m, m);
            __syncthreads();
            const int mm = s_m;
            __syncthreads();   // every warp has read s_m before thread 0 resets it
            if (mm == 0) break;
            lo = hi;
            hi += mm;
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) flag[q] = flag[q] == 1 ? 1 : 0;
    }
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) cnt += flag[q];
    int total_valid;
    int pos = scan(cnt, &total_valid);
    uint64_t *o = out + (int64_t)blockIdx.x * K;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        if (flag[q]) {
            if (pos < K) o[pos] = v[q];
            ++pos;
        }
    }
    for (int i = total_valid + tid; i < K; i += TK_THREADS) o[i] = KEY_NONE;
}

__global__ void topk_finish_kernel(const uint64_t *__restrict__ keys, int64_t key_stride, int K, TkSrc S,
                                   uint64_t *__restrict__ out_idx, float *__restrict__ out_score,
                                   int32_t *__restrict__ out_n)
{
    if (S.fb && !S.fb[blockIdx.y]) return;   // resolved by the fast path
    // blockIdx.y = workload S.w + y: its list, its offset, its output rows
    keys += (int64_t)blockIdx.y * key_stride;
    const uint64_t offset_w = S.offsets[S.w + blockIdx.y];
    out_idx += (int64_t)blockIdx.y * K;
    out_score += (int64_t)blockIdx.y * K;
    out_n += blockIdx.y;
    // single block: keys are sorted and distinct with KEY_NONE padding
    __shared__ int n_valid;
    if (threadIdx.x == 0) n_valid = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < K; i += blockDim.x) {
        const uint64_t k = keys[i];
        if (k != KEY_NONE) {
            out_idx[i] = offset_w + (k & 0xFFFFFFFFull);
            out_score[i] = fkey_inv((uint32_t)(k >> 32));
            atomicAdd(&n_valid, 1);
        } else {
            out_idx[i] = 0;
            out_score[i] = 0.f;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out_n = n_valid;
}

__global__ void chain_lists_kernel(const uint16_t *__restrict__ chain_w, int64_t n_chains, int n_w,
                                   int32_t *__restrict__ list, int32_t *__restrict__ cnt)
{
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chains) return;
    const int w = chain_w[c];
    if (w >= n_w) return;
    list[(int64_t)w * n_chains + atomicAdd(&cnt[w], 1)] = (int32_t)c;   // order free: the top-K is tiling-invariant
}

void topk_chain_lists(const uint16_t *chain_w, int64_t n_chains, int n_w, int32_t *list, int32_t *cnt, cudaStream_t s)
{
    chain_lists_kernel<<<(unsigned)((n_chains + 255) / 256), 256, 0, s>>>(chain_w, n_chains, n_w, list, cnt);
    at::note_launch();
}

// ---------------------------------------------------------------- threshold fast path (SA keys)
// The distinct top-K of a workload's 10^6..10^7 SA keys lies far in the low tail.  Two histogram
// sweeps over the key array (coalesced, every workload at once: the key's workload is its chain's)
// find, per workload, an order-preserving 22-bit key prefix below which at least M keys lie (11 bits,
// then 11 more inside the crossing bin); one more sweep compacts those keys; one block per workload
// sorts them, takes the distinct unmeasured ones in order and writes the first K.  M = 12288 leaves
// room for the heavy duplication of annealed chains (a chain parked at a minimum proposes the same
// neighbours again and again).  If the candidates overflow TKF_CAP or hold fewer than K distinct
// unmeasured keys while keys above the threshold exist, the workload is flagged and the exact tile
// reduction (topk_run) runs for it alone.  Either way the result is the distinct top-K: the fast path
// takes the K smallest distinct unmeasured keys of a set holding every key up to its threshold.
constexpr int TKF_BINS = 2048;
constexpr int TKF_CAP = 16384;
constexpr int TKF_M = 12288;
constexpr int TKF_GRID = 296;   // blocks of the sweeps (2 per SM), grid-stride over the key array

struct TkFast {
    uint32_t *hist;     // [n_batch][TKF_BINS]
    uint32_t *cnt;      // [n_batch] candidates appended
    uint32_t *bstar;    // [n_batch] threshold: level 0 the 11-bit bin, level 1 the 22-bit prefix (key >> 42)
    uint32_t *need;     // [n_batch] keys still needed inside the level-0 bin (0: take every key)
    uint64_t *cand;     // [n_batch][TKF_CAP]
    int32_t *fb;        // [n_batch] 1: fall back to the tile reduction
    uint32_t M;
};

// the batch row of flat key i (step-major [step][chain]): its chain's workload - S.w, or -1
__device__ __forceinline__ int tkf_row(const TkSrc &S, int64_t i, int n_batch)
{
    const int64_t c = i % S.n_chains;
    const int w = S.chain_w ? (int)__ldg(S.chain_w + c) : 0;
    const int y = w - S.w;
    return (y >= 0 && y < n_batch) ? y : -1;
}

__global__ void __launch_bounds__(TK_THREADS) tkf_hist_kernel(TkSrc S, TkFast F, int level, int n_batch)
{
    extern __shared__ uint32_t h[];   // [n_batch][TKF_BINS]
    for (int b = threadIdx.x; b < n_batch * TKF_BINS; b += TK_THREADS) h[b] = 0u;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * TK_THREADS + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * TK_THREADS) {
        const int y = tkf_row(S, i, n_batch);
        if (y < 0) continue;
        const uint64_t key = __ldg(S.keys + i);
        if (!level) {
            atomicAdd(&h[y * TKF_BINS + (int)(key >> 53)], 1u);
        } else if (F.need[y] != 0u && (key >> 53) == (uint64_t)F.bstar[y]) {
            atomicAdd(&h[y * TKF_BINS + (int)((key >> 42) & (TKF_BINS - 1))], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < n_batch * TKF_BINS; b += TK_THREADS)
        if (h[b]) atomicAdd(&F.hist[b], h[b]);
}

// one block per batch row: the smallest bin whose cumulative count reaches M (all bins if fewer)
__global__ void __launch_bounds__(TK_THREADS) tkf_thresh_kernel(TkFast F, int level)
{
    __shared__ uint32_t ws[TK_THREADS / 32];
    __shared__ uint32_t s_b;
    const int y = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int PER = TKF_BINS / TK_THREADS;
    uint32_t v[PER], c = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        v[q] = F.hist[(int64_t)y * TKF_BINS + tid * PER + q];
        c += v[q];
    }
    uint32_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += u;
    }
    if (lane == 31) ws[warp] = incl;
    if (tid == 0) s_b = TKF_BINS - 1;
    __syncthreads();
    if (warp == 0) {
        uint32_t x = ws[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, x, off);
            if (lane >= off) x += u;
        }
        ws[lane] = x;
    }
    __syncthreads();
    uint32_t run = incl - c + (warp > 0 ? ws[warp - 1] : 0u);
    __shared__ uint32_t s_need;
    if (tid == 0) s_need = 0u;
    __syncthreads();
    // level 0: M keys wanted; level 1: the keys still needed inside the level-0 bin
    const uint32_t want = level ? F.need[y] : F.M;
    if (level && want == 0u) return;   // the level-0 threshold already takes every key
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const uint32_t before = run;
        run += v[q];
        if (before < want && run >= want) {   // exactly one bin crosses the target
            s_b = (uint32_t)(tid * PER + q);
            s_need = want - before;
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (!level) {
            // fewer than M keys in the row (s_b stayed the last bin): take every key
            F.need[y] = s_b == (uint32_t)(TKF_BINS - 1) && ws[31] < want ? 0u : s_need;
            F.bstar[y] = s_b;
        } else {
            F.bstar[y] = (F.bstar[y] << 11) | s_b;   // a 22-bit threshold prefix
        }
        F.cnt[y] = 0u;
    }
}

__global__ void __launch_bounds__(TK_THREADS) tkf_compact_kernel(TkSrc S, TkFast F, int n_batch)
{
    for (int64_t i = (int64_t)blockIdx.x * TK_THREADS + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * TK_THREADS) {
        const int y = tkf_row(S, i, n_batch);
        if (y < 0) continue;
        const uint64_t key = __ldg(S.keys + i);
        // threshold on key >> 42 (22 bits); a row with fewer than M keys takes them all
        const uint64_t bs = F.need[y] == 0u ? 0x3FFFFFull : (uint64_t)F.bstar[y];
        if ((key >> 42) > bs) continue;
        const uint32_t pos = atomicAdd(&F.cnt[y], 1u);
        if (pos < (uint32_t)TKF_CAP) F.cand[(int64_t)y * TKF_CAP + pos] = key;
    }
}

// one block per batch row: sort the candidates, take the distinct unmeasured ones in order, write the
// first K -- or flag the row for the tile reduction
__global__ void __launch_bounds__(TK_THREADS) tkf_final_kernel(TkSrc S, TkFast F, int K, uint64_t *__restrict__ out_idx,
                                                               float *__restrict__ out_score, int32_t *__restrict__ out_n)
{
    extern __shared__ uint64_t sk[];   // [TKF_CAP]
    __shared__ int ws[TK_THREADS / 32];
    const int y = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = F.cnt[y];
    if (n > (uint32_t)TKF_CAP) {
        if (tid == 0) F.fb[y] = 1;
        return;
    }
    int P = 1;
    while (P < (int)n) P <<= 1;
    for (int i = tid; i < P; i += TK_THREADS) sk[i] = i < (int)n ? F.cand[(int64_t)y * TKF_CAP + i] : KEY_NONE;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P; i += TK_THREADS) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = sk[i], b = sk[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { sk[i] = b; sk[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
    // walk the sorted candidates in chunks of TK_THREADS: keep distinct, unmeasured keys, in order
    const uint64_t offset_w = S.offsets[S.w + y];
    out_idx += (int64_t)y * K;
    out_score += (int64_t)y * K;
    int got = 0;
    for (int c0 = 0; c0 < (int)n && got < K; c0 += TK_THREADS) {
        const int i = c0 + tid;
        int f = 0;
        uint64_t v = KEY_NONE;
        if (i < (int)n) {
            v = sk[i];
            f = (v != KEY_NONE && (i == 0 || sk[i - 1] != v)) ? 1 : 0;
            if (f && S.n_measured && in_sorted(S.measured, S.n_measured, offset_w + (v & 0xFFFFFFFFull))) f = 0;
        }
        int incl = f;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int u = __shfl_up_sync(0xFFFFFFFFu, incl, off);
            if (lane >= off) incl += u;
        }
        __syncthreads();
        if (lane == 31) ws[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int x = ws[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(0xFFFFFFFFu, x, off);
                if (lane >= off) x += u;
            }
            ws[lane] = x;
        }
        __syncthreads();
        const int pos = got + incl - f + (warp > 0 ? ws[warp - 1] : 0);
        if (f && pos < K) {
            out_idx[pos] = offset_w + (v & 0xFFFFFFFFull);
            out_score[pos] = fkey_inv((uint32_t)(v >> 32));
        }
        got += ws[31];
        __syncthreads();
    }
    // complete iff K were found, or the candidates were every key of the row
    const bool all = F.need[y] == 0u || F.bstar[y] >= 0x3FFFFFu;
    if (tid == 0) {
        if (got >= K || all) {
            F.fb[y] = 0;
            out_n[y] = got < K ? got : K;
        } else {
            F.fb[y] = 1;
        }
    }
    for (int i = (got < K ? got : K) + tid; i < K && (got >= K || all); i += TK_THREADS) {
        out_idx[i] = 0;
        out_score[i] = 0.f;
    }
}

size_t topk_fast_scratch_bytes(int n_batch)
{
    return ((size_t)n_batch * (TKF_BINS * 4 + 4 + 4 + 4 + 4) + 255) / 256 * 256 + (size_t)n_batch * TKF_CAP * 8;
}

// the SA top-K of every batch row by the threshold fast path; rows it cannot settle are flagged in fb
// (device) and topk_run(..., fb) finishes them
int topk_fast(const TkArgs &a, int n_batch, const uint64_t *offsets, int64_t per, uint8_t *scratch, int32_t *fb,
              cudaStream_t s)
{
    TkSrc S{};
    S.mode = 0;
    S.keys = a.keys;
    S.n = a.n_src;
    S.n_chains = a.n_chains;
    S.chain_w = a.chain_w;
    S.chain_list = a.chain_list;
    S.list_n = a.list_n;
    S.w = a.w;
    S.measured = a.measured;
    S.n_measured = a.n_measured;
    S.list_stride = a.n_chains;
    for (int q = 0; q < MAXW; ++q) S.offsets[q] = offsets ? offsets[q] : a.offset_w;
    TkFast F{};
    F.hist = (uint32_t *)scratch;
    F.cnt = F.hist + (size_t)n_batch * TKF_BINS;
    F.bstar = F.cnt + n_batch;
    F.need = F.bstar + n_batch;
    F.cand = (uint64_t *)(scratch + ((size_t)n_batch * (TKF_BINS * 4 + 4 + 4 + 4 + 4) + 255) / 256 * 256);
    F.fb = fb;
    (void)per;
    F.M = (uint32_t)TKF_M;
    static bool attr = false;
    if (!attr) {
        AT_CUDA_TRY(cudaFuncSetAttribute(tkf_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(TKF_CAP * sizeof(uint64_t))));
        AT_CUDA_TRY(cudaFuncSetAttribute(tkf_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(MAXW * TKF_BINS * sizeof(uint32_t))));
        attr = true;
    }
    ProfScope ps(AT_K_TOPK, s);
    const size_t hsm = (size_t)n_batch * TKF_BINS * sizeof(uint32_t);
    for (int level = 0; level < 2; ++level) {   // 11-bit bins, then 11 more bits inside the crossing bin
        AT_CUDA_TRY(cudaMemsetAsync(F.hist, 0, hsm, s));
        tkf_hist_kernel<<<TKF_GRID, TK_THREADS, hsm, s>>>(S, F, level, n_batch); at::note_launch();
        tkf_thresh_kernel<<<n_batch, TK_THREADS, 0, s>>>(F, level); at::note_launch();
    }
    tkf_compact_kernel<<<TKF_GRID, TK_THREADS, 0, s>>>(S, F, n_batch); at::note_launch();
    tkf_final_kernel<<<n_batch, TK_THREADS, TKF_CAP * sizeof(uint64_t), s>>>(S, F, a.K, a.out_idx, a.out_score,
                                                                               a.out_n); at::note_launch();
    AT_LAUNCH_CHECK("topk fast path");
    return AT_OK;
}

size_t topk_scratch_bytes(int64_t n_src, int K, int n_batch)
{
    const int64_t b1 = (n_src + TK_TILE - 1) / TK_TILE;
    return (size_t)(2 * (b1 + 1) * (int64_t)K) * sizeof(uint64_t) * (size_t)n_batch;
}

// n_batch workloads a.w .. a.w + n_batch - 1 in one launch per pass (blockIdx.y); their outputs are
// consecutive rows of a.out_* (K entries each) and a.out_n[y]
int topk_run(const TkArgs &a, uint64_t *scratch, cudaStream_t s, int n_batch, const uint64_t *offsets,
             const int32_t *fb)
{
    TkSrc S{};
    S.fb = fb;
    S.mode = a.mode;
    S.keys = a.keys;
    S.n = a.n_src;
    S.n_chains = a.n_chains;
    S.chain_w = a.chain_w;
    S.chain_list = a.chain_list;
    S.list_n = a.list_n;
    S.w = a.w;
    S.offset_w = a.offset_w;
    S.l_idx = a.l_idx;
    S.l_score = a.l_score;
    S.l_n = a.l_n;
    S.n_w = a.n_w;
    S.k_in = a.k_in;
    S.measured = a.measured;
    S.n_measured = a.n_measured;
    S.key_stride = 0;
    S.list_stride = a.n_chains;
    for (int q = 0; q < MAXW; ++q) S.offsets[q] = offsets ? offsets[q] : a.offset_w;
    const int K = a.K;
    int64_t blocks = (a.n_src + TK_TILE - 1) / TK_TILE;
    if (blocks < 1) blocks = 1;
    const int64_t stride = (blocks + 1) * K;   // per workload, in each of the two buffers
    uint64_t *bufA = scratch, *bufB = scratch + stride * n_batch;
    ProfScope ps(AT_K_TOPK, s);
    topk_tile_kernel<<<dim3((unsigned)blocks, n_batch), TK_THREADS, 0, s>>>(S, K, bufA, stride); at::note_launch();
    AT_LAUNCH_CHECK("topk_tile_kernel");
    int64_t n = blocks * K;
    while (blocks > 1) {
        TkSrc R = S;
        R.mode = 2;
        R.keys = bufA;
        R.n = n;
        R.key_stride = stride;
        R.chain_list = nullptr;
        R.n_measured = 0;
        R.fb = fb;
        blocks = (n + TK_TILE - 1) / TK_TILE;
        topk_tile_kernel<<<dim3((unsigned)blocks, n_batch), TK_THREADS, 0, s>>>(R, K, bufB, stride); at::note_launch();
        AT_LAUNCH_CHECK("topk_tile_kernel(reduce)");
        n = blocks * K;
        uint64_t *t = bufA; bufA = bufB; bufB = t;
    }
    topk_finish_kernel<<<dim3(1, n_batch), 256, 0, s>>>(bufA, stride, K, S, a.out_idx, a.out_score, a.out_n);
    at::note_launch();
    AT_LAUNCH_CHECK("topk_finish_kernel");
    return AT_OK;
}

}  // namespace at

extern "C" int topk_merge(at_space sp, const uint64_t *d_in_idx, const float *d_in_score, const int32_t *d_in_n,
                          int32_t n_lists, int32_t k_in, const uint64_t *d_measured_sorted, int64_t n_measured,
                          int32_t k_out, uint64_t *d_out_idx, float *d_out_score, int32_t *d_out_n, void *stream)
{
    if (!sp || !d_in_idx || !d_in_score || !d_in_n || !d_out_idx || !d_out_score || !d_out_n)
        return at::fail(AT_EINVAL, "topk_merge: null pointer");
    if (int rc = at::take_range_error(sp)) return rc;
    if (n_lists < 1 || k_in < 1 || k_out < 1 || k_out > 1024 || n_measured < 0)
        return at::fail(AT_EINVAL, "topk_merge: need n_lists, k_in >= 1 and 1 <= k_out <= 1024");
    if (n_measured > 0 && !d_measured_sorted) return at::fail(AT_EINVAL, "topk_merge: null measured list");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_src = (int64_t)n_lists * k_in;
    const int nw = sp->host.n_w;
    int rc = at::scratch_reserve(sp, at::topk_scratch_bytes(n_src, k_out, nw), s);
    if (rc) return rc;
    at::TkArgs a{};   // every workload in one batched pass (blockIdx.y = workload)
    a.mode = 1;
    a.n_src = n_src;
    a.w = 0;
    a.offset_w = sp->host.offset[0];
    a.l_idx = d_in_idx;
    a.l_score = d_in_score;
    a.l_n = d_in_n;
    a.n_w = nw;
    a.k_in = k_in;
    a.measured = d_measured_sorted;
    a.n_measured = n_measured;
    a.K = k_out;
    a.out_idx = d_out_idx;
    a.out_score = d_out_score;
    a.out_n = d_out_n;
    uint64_t offs[at::MAXW];
    for (int q = 0; q < at::MAXW; ++q) offs[q] = q < nw ? sp->host.offset[q] : 0;
    rc = at::topk_run(a, (uint64_t *)sp->d_scratch, s, nw, offs);
    if (rc) return rc;
    return AT_OK;
}
