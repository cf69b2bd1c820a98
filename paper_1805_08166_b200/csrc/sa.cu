// sa.cu -- sa_explore: fused proposal -> features -> GBT -> Metropolis over many chains
// (Alg. 1 P:152-153 "run parallel simulated annealing ... using energy function f-hat";
// P:187 "a batch of parallel Markov chains", persistent states; readings Q20-Q23, Q28).
//
// Block = GRP groups of 32 chains (lane = chain) x SA_NW warps.  Per step, the owner warp of
// each group draws the Philox proposal of its chains and applies the single-knob move to the
// chain's knob vector (kept in registers: no decode after the start state); all warps then
// compute the proposals' 468 features into shared tiles [468][32] (loop extents, context rows,
// relation features: three barrier-separated phases dealt over the warps), walk the ensemble
// (each warp a residue class of trees, gbt.cuh; trees stream in by TMA bulk copies), and the
// owner warps fold the partials in the canonical order, take the Metropolis decisions and record
// the proposals' keys for the distinct top-K.  Chain state never leaves the SM between steps;
// only 8 bytes per chain-step (the visited key) go to HBM.
#include "features.cuh"
#include "gbt.cuh"
#include "topk.cuh"

#include <algorithm>
#include <cstdlib>

namespace at {

constexpr int SA_NW = 16;      // walker warps
constexpr int SA_NWARPS = 17;  // + the tree-stream producer warp (feature-phase items stay with the walkers:
                               // giving the producer some, or an 18th warp, measured no faster)

struct TileSink {
    float *tile;
    int lane;
    __device__ __forceinline__ void put(int f, float v) { tile[f * 32 + lane] = v; }
    __device__ __forceinline__ void put_rel(int f, float v) { tile[f * 32 + lane] = v; }
};

__device__ __forceinline__ void feats_any(const WlDev &W, const uint16_t *fact, const uint32_t *ch, float *tile,
                                          int lane, int part, int nparts)
{
    TileSink sk{tile, lane};
    switch (W.tmpl) {
    case 0: features_one<0>(W, fact, ch, sk, part, nparts, true); break;
    case 1: features_one<1>(W, fact, ch, sk, part, nparts, true); break;
    default: features_one<2>(W, fact, ch, sk, part, nparts, true); break;
    }
}

__device__ __forceinline__ int n_loops(int tmpl) { return tmpl == 0 ? 8 : tmpl == 1 ? 18 : 16; }

// TM >= 0: every workload of the space uses template TM (compile-time: one code path, a smaller
// hot loop); TM = -1: per-lane dispatch (mixed-template unions)
template <int TM>
__device__ __forceinline__ void zero_cols_any(int tmpl, float *tile, int lane)
{
    TileSink sk{tile, lane};
    if (TM >= 0) { features_zero_cols<TM < 0 ? 0 : TM>(sk); return; }
    switch (tmpl) {
    case 0: features_zero_cols<0>(sk); break;
    case 1: features_zero_cols<1>(sk); break;
    default: features_zero_cols<2>(sk); break;
    }
}

template <int TM>
__device__ __forceinline__ void decode_any(const WlDev &W, uint32_t local, uint32_t *ch)
{
    if (TM >= 0) {
        decode_knobs<TM < 0 ? 0 : TM>(W, local, ch);
    } else {
        switch (W.tmpl) {
        case 0: decode_knobs<0>(W, local, ch); break;
        case 1: decode_knobs<1>(W, local, ch); break;
        default: decode_knobs<2>(W, local, ch); break;
        }
    }
#pragma unroll
    for (int j = 0; j < MAXKNOBS; ++j)
        if (j >= W.n_knobs) ch[j] = 0;
}

struct SaParams {
    const SpaceDev *S;
    const uint16_t *fact;
    float base;
    int n_chains, n_steps, init;
    uint64_t seed;
    uint32_t round, chain_base;
    const float *temps;
    const uint16_t *chain_w;
    uint64_t *chain_idx;
    float *chain_E;
    uint32_t *accept_bits;
    float *vis_E;
    uint64_t *vis_idx;
    uint64_t *keys;   // [n_steps+1][n_chains] (step-major: a warp's 32 keys are one coalesced store)
    AcqArgs Q;        // KM > 1: energy = acquisition over Q.K concatenated models
};

// shared-memory layout of sa_kernel: GRP groups of 32 chains
template <int GRP, int KM = 1>
struct SaSmem {
    float tile[GRP][NFEAT * 32];
    float part[GRP][KM > 1 ? KM * 32 * 32 : 1];   // KM = 1: the partials alias tile columns 0..31 (below)
    float fk[GRP][KM > 1 ? KM * 32 : 1];   // per-model energies (KM > 1)
    uint32_t chb[2][GRP][MAXKNOBS][32];   // proposal knob vectors, by step parity (owner-written)
    int32_t pjs[2][GRP][32];              // ... the move that made it (knob, -1: none) and the old value
    uint32_t pvs[2][GRP][32];
    uint16_t extc[2][GRP][MAXLOOPS][32];  // loop extents of the next proposal for both outcomes of the
                                          // current step (0: accepted, 1: rejected), by helper warps
    uint32_t esel[GRP][32];               // which one the owner's decision selected
    uint32_t rnd[GRP][4][32];             // the next step's Philox words, precomputed by a helper warp
    int32_t w[GRP][32];
    uint64_t bar[4 * TS_MAXBUF];          // tree-chunk barriers, then (ring mode) consumption counters; NP
                                          // pipelines: full[2 NP] then empty[2 NP]
};

template <int TM>
__device__ __forceinline__ void sa_row_any(const WlDev &W, const uint16_t *ext, const uint32_t *ch, int k, int lane,
                                           float *tile)
{
    if (TM >= 0) { sa_row_rel<TM < 0 ? 0 : TM>(W, ext, ch, k, lane, tile); return; }
    switch (W.tmpl) {
    case 0: sa_row_rel<0>(W, ext, ch, k, lane, tile); break;
    case 1: sa_row_rel<1>(W, ext, ch, k, lane, tile); break;
    default: sa_row_rel<2>(W, ext, ch, k, lane, tile); break;
    }
}

template <int TM>
__device__ __forceinline__ void sa_extents_any(int tmpl, const uint32_t (&foff)[6], const uint16_t *fact,
                                               const uint32_t *ch, uint16_t *ext)
{
    if (TM >= 0) { sa_extents<TM < 0 ? 0 : TM>(foff, fact, ch, ext); return; }
    switch (tmpl) {
    case 0: sa_extents<0>(foff, fact, ch, ext); break;
    case 1: sa_extents<1>(foff, fact, ch, ext); break;
    default: sa_extents<2>(foff, fact, ch, ext); break;
    }
}

// relation slots of every group back to +0 (before the next rows deposit into them); warps
// g >= GRP only, which are idle while the owner warps propose / decide
template <int GRP>
__device__ __forceinline__ void zero_relation(float (*tile)[NFEAT * 32], int lane, int warp)
{
    if (warp >= SA_NW) return;   // the producer warp
    for (int r = warp - GRP; r < GRP * 120; r += SA_NW - GRP) tile[r / 120][(342 + r % 120) * 32 + lane] = 0.0f;
}

// Block = GRP groups of 32 chains (lane = chain) x SA_NW warps.  Warp g owns group g's chain
// state; every warp takes part in every group's feature phases and tree walk, so each tree byte
// staged in shared memory serves 32 GRP chains.
template <int GRP, int KM, int TM, bool LG = false, int ONLY = 0>
__global__ void __launch_bounds__(SA_NWARPS * 32, 1) sa_kernel(SaParams P, TreeGeo G)
{
    extern __shared__ __align__(128) unsigned char smraw[];
    SaSmem<GRP, KM> &sm = *(SaSmem<GRP, KM> *)smraw;
    uint8_t *bufs = smraw + ((sizeof(SaSmem<GRP, KM>) + 127) / 128) * 128;
    // the energy of group og's chains after a walk: f-hat, or the acquisition over the K models
    auto energy = [&](int og, int lane) -> float {
        if (KM == 1) return gbt_combine(&sm.tile[og][0], lane, P.base);   // partials in tile columns 0..31
        float mu, sd;
        return acquisition(P.Q, &sm.fk[og][lane], 32, mu, sd);
    };
    auto fold_models = [&](int warp, int lane) {   // KM > 1: every warp (g, m) folds model m's partials
        if (KM > 1) {
            if (warp < GRP * P.Q.K) {
                const int g = warp / P.Q.K, m = warp - g * P.Q.K;
                sm.fk[g][m * 32 + lane] = gbt_combine(&sm.part[g][m * 1024], lane, P.Q.base[m]);
            }
            __syncthreads();
        }
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int og = warp < GRP ? warp : 0;                  // the group whose state this warp owns
    const bool owner = warp < GRP;
    const int c = blockIdx.x * 32 * GRP + og * 32 + lane;  // the owner's chain
    const bool live = owner && c < P.n_chains;
    const int64_t per = (int64_t)P.n_steps + 1;
    const uint64_t c_limit = (uint64_t)ts_uses_per_pass(G) * (uint64_t)per;

#ifdef AT_SA_PHASE_TIMING
    if (threadIdx.x < 3 * 17) s_walk_prof[threadIdx.x] = 0ull;
#endif
    ts_start(G, bufs, sm.bar);
    // owner-warp state (registers): knob vector, index and energy of the lane's chain
    uint32_t ch[MAXKNOBS];
    uint64_t idx = 0, idx2 = 0;
    float E = 0.f;
    int w = 0;
    const uint32_t gid = P.chain_base + (uint32_t)c;
    uint32_t accw = 0;
    int pj = -1;
    uint32_t pv = 0;
    uint32_t foff[6] = {0u, 0u, 0u, 0u, 0u, 0u};   // the chain's split-table offsets (fixed workload)
    int tmpl = 0;
    if (owner) {
        if (live && P.chain_w) w = P.chain_w[c];
        if (w >= P.S->n_w) {   // a chain outside the space's workloads: clamped, AT_ERANGE
            flag_range(P.S);
            w = 0;
        }
        const WlDev &W = P.S->w[w];
        if (live) {
            if (P.init) {
                const U4 r = philox(P.seed, gid, 0, P.round, TAG_SA_INIT);
                idx = W.offset + mulhi64((uint64_t)r.x | ((uint64_t)r.y << 32), (uint64_t)W.size);
            } else {
                idx = P.chain_idx[c];
                if (idx < W.offset || idx - W.offset >= (uint64_t)W.size) {   // not a state of workload w: AT_ERANGE
                    flag_range(P.S);
                    idx = W.offset;
                }
            }
        } else {
            idx = W.offset;
        }
        decode_any<TM>(W, (uint32_t)(idx - W.offset), ch);
        // the start state is "step -1's proposal": parity 1, no move; its extents in candidate 0
#pragma unroll
        for (int j = 0; j < MAXKNOBS; ++j) sm.chb[1][og][j][lane] = ch[j];
        sm.pjs[1][og][lane] = -1;
        sm.pvs[1][og][lane] = 0u;
        sm.esel[og][lane] = 0u;
#pragma unroll
        for (int q = 0; q < 6; ++q) foff[q] = W.fact_off[q];
        tmpl = W.tmpl;
        sa_extents_any<TM>(tmpl, foff, P.fact, ch, &sm.extc[0][og][0][lane]);
        sm.w[og][lane] = w;
        zero_cols_any<TM>(W.tmpl, sm.tile[og], lane);
    } else {
        zero_relation<GRP>(sm.tile, lane, warp);
    }
    __syncthreads();
    uint32_t ph[TS_MAXBUF] = {0u, 0u, 0u, 0u};
    uint64_t cs = 0;
    bool no_slots[GRP];
#pragma unroll
    for (int g = 0; g < GRP; ++g) no_slots[g] = false;
#ifdef AT_SA_PHASE_TIMING
    long long t_prop = 0, t_feat = 0, t_walk = 0, t_rows = 0, t0 = clock64();
#endif
    // every warp computes its share of the features of all chains of the block
    auto features_phase = [&](int par) {
        // R) context rows and their relation deposits: items (group, row)
        for (int it = warp; it < GRP * MAXLOOPS && warp < SA_NW; it += SA_NW) {
            const int g = it / MAXLOOPS, k = it - g * MAXLOOPS;
            uint32_t chl[MAXKNOBS];
#pragma unroll
            for (int j = 0; j < MAXKNOBS; ++j) chl[j] = sm.chb[par][g][j][lane];
            sa_row_any<TM>(P.S->w[sm.w[g][lane]], &sm.extc[sm.esel[g][lane]][g][0][lane], chl, k, lane, sm.tile[g]);
        }
        __syncthreads();
#ifdef AT_SA_PHASE_TIMING
        t_rows += clock64() - t0;
#endif
        // T) prefix max of the relation slots: items (group, buffer, pair)
        for (int it = warp; it < GRP * 6 && warp < SA_NW; it += SA_NW) {
            const int g = it / 6, r = it - g * 6;
            relation_prefix(sm.tile[g], lane, r >> 1, r & 1);
        }
        __syncthreads();
    };
    // helper warp GRP + g draws step s's Philox words of group g's chains (off the owner's serial
    // proposal path); the walk's closing barrier publishes them before the owner reads them
    auto draw_next = [&](int s) {
        if (warp >= GRP && warp < 2 * GRP && s < P.n_steps) {
            const int g = warp - GRP;
            const uint32_t gc = P.chain_base + (uint32_t)(blockIdx.x * 32 * GRP + g * 32 + lane);
            const U4 r = philox(P.seed, gc, (uint32_t)s, P.round, TAG_SA_STEP);
            sm.rnd[g][0][lane] = r.x;
            sm.rnd[g][1][lane] = r.y;
            sm.rnd[g][2][lane] = r.z;
            sm.rnd[g][3][lane] = r.w;
        }
    };
    // While the owner warps decide step s (serial, after the walk), helper warps GRP + 2g + b build
    // the loop extents of step s + 1's proposal for group g under both outcomes -- b = 0: the move
    // applied to step s's proposal (accepted), b = 1: to the state before it (rejected) -- so the
    // owner's proposal needs no extents of its own; the proposal barrier publishes them.
    auto precompute = [&](int s_next, int par) {   // par: parity of step s_next - 1's proposal
        const int hw = warp - GRP;
        if (hw >= 0 && hw < 2 * GRP && s_next < P.n_steps) {
            const int g = hw >> 1, b = hw & 1;
            const uint32_t gc = P.chain_base + (uint32_t)(blockIdx.x * 32 * GRP + g * 32 + lane);
            const U4 r = philox(P.seed, gc, (uint32_t)s_next, P.round, TAG_SA_STEP);
            const WlDev &W = P.S->w[sm.w[g][lane]];
            uint32_t x[MAXKNOBS];
#pragma unroll
            for (int j = 0; j < MAXKNOBS; ++j) x[j] = sm.chb[par][g][j][lane];
            const int pjx = sm.pjs[par][g][lane];
            const uint32_t pvx = sm.pvs[par][g][lane];
            if (b == 1)
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == pjx) x[q] = pvx;
            if (W.n_ns > 0) {   // the owner's move, replayed
                const int j = W.ns_list[__umulhi(r.x, W.n_ns)];
                uint32_t v = 0;
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == j) v = x[q];
                uint32_t v2 = __umulhi(r.y, W.radix[j] - 1u);
                if (v2 >= v) v2 += 1;
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == j) x[q] = v2;
            }
            uint32_t fo[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) fo[q] = W.fact_off[q];
            sa_extents_any<TM>(W.tmpl, fo, P.fact, x, &sm.extc[b][g][0][lane]);
        }
    };
    features_phase(1);
    draw_next(0);
    ts_wait_resident(G, sm.bar);
    walk_pass<SA_NW, GRP, KM, false, LG, SA_NW, ONLY>(G, bufs, sm.bar, ph, cs, c_limit, &sm.tile[0][0], NFEAT * 32, lane, warp,
                                              KM == 1 ? &sm.tile[0][0] : &sm.part[0][0], KM == 1 ? NFEAT * 32 : KM * 1024,
                          nullptr, 0, 0, no_slots);
    fold_models(warp, lane);
    if (!owner) zero_relation<GRP>(sm.tile, lane, warp);
    precompute(0, 1);
    if (owner) {
        E = energy(og, lane);
        if (live) {
            P.keys[c] = ((uint64_t)fkey(E) << 32) | (uint64_t)(idx - P.S->w[w].offset);   // step-major: coalesced
            if (P.vis_E) { P.vis_E[(int64_t)c * per] = E; P.vis_idx[(int64_t)c * per] = idx; }
        }
    }

#ifdef AT_SA_PHASE_TIMING
    t_prop = t_feat = t_walk = t_rows = 0;
    t0 = clock64();
#endif
    bool rejected = false;   // the owner's last decision (selects the precomputed extents)
    for (int s = 0; s < P.n_steps; ++s) {
        U4 r;
        const int par = s & 1;
        if (owner) {
            const WlDev &W = P.S->w[w];
            r = U4{sm.rnd[og][0][lane], sm.rnd[og][1][lane], sm.rnd[og][2][lane], sm.rnd[og][3][lane]};   // Philox(gid, s)
            idx2 = idx;
            pj = -1;
            if (W.n_ns > 0) {
                const int j = W.ns_list[__umulhi(r.x, W.n_ns)];
                uint32_t v = 0;
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == j) v = ch[q];
                uint32_t v2 = __umulhi(r.y, W.radix[j] - 1u);
                if (v2 >= v) v2 += 1;
                AT_DCHECK(j < W.n_knobs && v < W.radix[j] && v2 < W.radix[j]);
                idx2 = idx - (uint64_t)v * W.place[j] + (uint64_t)v2 * W.place[j];
                pj = j;
                pv = v;
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == j) ch[q] = v2;
            }
#pragma unroll
            for (int q = 0; q < MAXKNOBS; ++q) sm.chb[par][og][q][lane] = ch[q];
            sm.pjs[par][og][lane] = pj;
            sm.pvs[par][og][lane] = pv;
            sm.esel[og][lane] = rejected ? 1u : 0u;   // the helpers' extents of this proposal
        }
        __syncthreads();
#ifdef AT_SA_PHASE_TIMING
        { long long t = clock64(); t_prop += t - t0; t0 = t; }
#endif
        features_phase(par);
        draw_next(s + 1);
#ifdef AT_SA_PHASE_TIMING
        { long long t = clock64(); t_feat += t - t0; t0 = t; }
#endif
        walk_pass<SA_NW, GRP, KM, false, LG, SA_NW, ONLY>(G, bufs, sm.bar, ph, cs, c_limit, &sm.tile[0][0], NFEAT * 32, lane, warp,
                              KM == 1 ? &sm.tile[0][0] : &sm.part[0][0], KM == 1 ? NFEAT * 32 : KM * 1024, nullptr, 0,
                              0, no_slots);
#ifdef AT_SA_PHASE_TIMING
        { long long t = clock64(); t_walk += t - t0; t0 = t; }
#endif
        fold_models(warp, lane);
        if (!owner) zero_relation<GRP>(sm.tile, lane, warp);
        precompute(s + 1, par);
        if (owner) {
            const float E2 = energy(og, lane);
            const float d = __fsub_rn(E2, E);
            bool acc = d <= 0.0f;
            if (!acc) {
                const float T = __ldg(P.temps + s);
                if (T > 0.0f) {
                    const float u = __fmul_rn(__uint2float_rn(r.z >> 8), __int_as_float(0x33800000));
                    acc = u < exp_det(-__fdiv_rn(d, T));
                }
            }
            if (acc) {
                idx = idx2;
                E = E2;
                accw |= 1u << (s & 31);
            } else if (pj >= 0) {
#pragma unroll
                for (int q = 0; q < MAXKNOBS; ++q) if (q == pj) ch[q] = pv;   // undo the move
            }
            rejected = !acc;
            if (live) {
                const int64_t at = (int64_t)c * per + s + 1;
                P.keys[(int64_t)(s + 1) * P.n_chains + c] = ((uint64_t)fkey(E2) << 32) | (uint64_t)(idx2 - P.S->w[w].offset);
                if (P.vis_E) { P.vis_E[at] = E2; P.vis_idx[at] = idx2; }
                if (P.accept_bits && ((s & 31) == 31 || s == P.n_steps - 1)) {
                    P.accept_bits[(int64_t)c * ((P.n_steps + 31) / 32) + (s >> 5)] = accw;
                }
            }
            if ((s & 31) == 31) accw = 0;
        }
    }
    if (live) {
        P.chain_idx[c] = idx;
        P.chain_E[c] = E;
    }
#ifdef AT_SA_PHASE_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("sa phases (cycles/step, block 0, GRP=%d T=%d NC=%d CH=%d): proposal+accept %lld features %lld (rows %lld) "
               "walk %lld\n", GRP, G.T, G.NC, G.CH, t_prop / max(P.n_steps, 1), t_feat / max(P.n_steps, 1),
               t_rows / max(P.n_steps, 1), t_walk / max(P.n_steps, 1));
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int w = 0; w < 17; ++w)
            printf("  warp %2d per step: tree wait %llu walk %llu barrier+issue %llu\n", w,
                   s_walk_prof[3 * w] / (P.n_steps + 1), s_walk_prof[3 * w + 1] / (P.n_steps + 1),
                   s_walk_prof[3 * w + 2] / (P.n_steps + 1));
#endif
}

template <int GRP, int KM = 1>
size_t sa_smem_bytes(const TreeGeo &G)
{
    return ((sizeof(SaSmem<GRP, KM>) + 127) / 128) * 128 + (size_t)G.NBUF * (size_t)G.chunk_bytes;
}

}  // namespace at

extern "C" int sa_explore(at_space sp, at_gbt g, uint64_t *d_chain_idx, float *d_chain_energy,
                          const uint16_t *d_chain_workload, const uint64_t *d_measured_sorted, int64_t n_measured,
                          const at_sa_opts *o, uint64_t *d_out_idx, float *d_out_score, int32_t *d_out_n,
                          void *stream)
{
    if (!sp || !g || !o) return at::fail(AT_EINVAL, "sa_explore: null handle");
    if (int rc = at::take_range_error(sp)) return rc;
    if (int rc = at::model_error(g)) return rc;
    if (!d_chain_idx || !d_chain_energy || (!o->d_temps && o->n_steps > 0) || !d_out_idx || !d_out_score || !d_out_n)
        return at::fail(AT_EINVAL, "sa_explore: null buffer");
    if (o->n_chains < 1 || o->n_steps < 0 || o->k_out < 1 || o->k_out > 1024 || n_measured < 0)
        return at::fail(AT_EINVAL, "sa_explore: need n_chains >= 1, n_steps >= 0, 1 <= k_out <= 1024");
    if (n_measured > 0 && !d_measured_sorted) return at::fail(AT_EINVAL, "sa_explore: null measured list");
    if (g->n_features != at::NFEAT) return at::fail(AT_EMISMATCH, "sa_explore: model must take 468 features");
    if ((uint64_t)o->chain_id_base + (uint64_t)o->n_chains > 0x100000000ull)
        return at::fail(AT_ERANGE, "sa_explore: global chain ids exceed 2^32");
    if ((o->d_visited_E == nullptr) != (o->d_visited_idx == nullptr))
        return at::fail(AT_EINVAL, "sa_explore: d_visited_E and d_visited_idx go together");
    cudaStream_t s = (cudaStream_t)stream;
    g->last = s;
    const int64_t per = (int64_t)o->n_steps + 1;
    const int64_t n_keys = (int64_t)o->n_chains * per;
    const size_t key_bytes = ((size_t)n_keys * sizeof(uint64_t) + 255) / 256 * 256;
    // chain lists per workload (multi-workload spaces): the top-k then reads only a workload's own keys
    const bool lists = d_chain_workload && sp->host.n_w > 1;
    const size_t list_bytes = lists ? (((size_t)sp->host.n_w * o->n_chains + at::MAXW) * sizeof(int32_t) + 255) / 256 * 256 : 0;
    const int nbt = lists ? sp->host.n_w : 1;
    const size_t tk_bytes = (at::topk_scratch_bytes(n_keys, o->k_out, nbt) + 255) / 256 * 256;
    const size_t fast_bytes = at::topk_fast_scratch_bytes(nbt) + 256;
    int rc = at::scratch_reserve(sp, key_bytes + list_bytes + tk_bytes + fast_bytes, s);
    if (rc) return rc;
    uint64_t *keys = (uint64_t *)sp->d_scratch;
    int32_t *chain_list = lists ? (int32_t *)((char *)sp->d_scratch + key_bytes) : nullptr;
    int32_t *list_n = lists ? chain_list + (size_t)sp->host.n_w * o->n_chains : nullptr;
    uint64_t *tkbuf = (uint64_t *)((char *)sp->d_scratch + key_bytes + list_bytes);
    uint8_t *fastbuf = (uint8_t *)sp->d_scratch + key_bytes + list_bytes + tk_bytes;
    int32_t *fb = (int32_t *)(fastbuf + at::topk_fast_scratch_bytes(nbt));   // [nbt] fall-back flags

    at::SaParams P{};
    P.S = sp->d_space;
    P.fact = sp->d_fact;
    P.base = g->base;
    P.n_chains = o->n_chains;
    P.n_steps = o->n_steps;
    P.init = o->init;
    P.seed = o->seed;
    P.round = o->round;
    P.chain_base = o->chain_id_base;
    P.temps = o->d_temps;
    P.chain_w = d_chain_workload;
    P.chain_idx = d_chain_idx;
    P.chain_E = d_chain_energy;
    P.accept_bits = o->d_accept_bits;
    P.vis_E = o->d_visited_E;
    P.vis_idx = o->d_visited_idx;
    P.keys = keys;
    const at_acq_opts *acq = o->acq;
    if (acq) {
        if (acq->n_models < 1 || acq->n_models > 8 || g->n_trees % acq->n_models != 0)
            return at::fail(AT_EINVAL, "sa_explore: acq needs 1 <= n_models <= 8 dividing n_trees");
        if (acq->kind < AT_ACQ_MEAN || acq->kind > AT_ACQ_EI) return at::fail(AT_EINVAL, "sa_explore: bad acq kind");
        P.Q.K = acq->n_models;
        P.Q.kind = acq->kind;
        P.Q.kappa = acq->kappa;
        P.Q.best = acq->best;
        for (int k = 0; k < 8; ++k) P.Q.base[k] = k < acq->n_models ? acq->model_base[k] : 0.0f;
    }
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        AT_CUDA_TRY(cudaGetDevice(&dev));
        AT_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
#ifdef AT_SA_PHASE_TIMING
    constexpr size_t SMEM_MAX = 226 * 1024;   // room for the static profiling counters
#else
    constexpr size_t SMEM_MAX = 227 * 1024;
#endif
    // the tree buffers take all the shared memory the chain state leaves (bigger chunks: more trees per
    // warp per chunk, more independent walks in flight, fewer chunk hand-offs).  A streamed ensemble
    // uses NBUF buffers; ring mode drops the per-chunk block barrier (gbt.cuh walk_pass)
    static int nbuf_env = -1, ring_env = -1, lg_env = -1, np_env = -1;
    if (nbuf_env < 0) {
        const char *e1 = getenv("AT_SA_NBUF"), *e2 = getenv("AT_SA_RING"), *e3 = getenv("AT_SA_LG");
        const char *e4 = getenv("AT_SA_NP");
        np_env = e4 ? atoi(e4) : 0;
        if (np_env != 2 && np_env != 4) np_env = 0;
        nbuf_env = e1 ? std::max(2, std::min(at::TS_MAXBUF, atoi(e1))) : 2;
        ring_env = e2 ? (atoi(e2) != 0) : 0;
        lg_env = e3 ? (atoi(e3) != 0) : 0;
    }
    auto geo = [&](size_t hdr) {
        at::TreeGeo G0 = at::make_geo(g, (uint32_t)((SMEM_MAX - hdr) / 2));
        if (G0.resident) return G0;
        if (np_env) {
            // NP pipelines of SA_NW / NP warps, each with two slices of SA_NW / NP trees
            const uint32_t per_tree = (uint32_t)((1 << g->depth) - 1) * 8u + (uint32_t)(1 << g->depth) * 4u;
            const int chs = at::SA_NW / np_env;
            if ((size_t)2 * np_env * chs * per_tree <= SMEM_MAX - hdr) {
                at::TreeGeo Gp = at::make_geo(g, (uint32_t)chs * per_tree, false, 2 * np_env, 0);
                Gp.CH = chs;
                Gp.NC = g->t_pad / chs;
                Gp.chunk_bytes = (uint32_t)chs * per_tree;
                Gp.resident = 0;
                Gp.NP = np_env;
                return Gp;
            }
        }
        if (lg_env) {
            // leaves from global memory: the buffers hold nodes only, chunks of a multiple of SA_NW trees
            // (every warp walks the same number of trees per chunk)
            const uint32_t nb = (uint32_t)((1 << g->depth) - 1) * 8u;
            uint32_t per = (uint32_t)((SMEM_MAX - hdr) / nbuf_env) / nb;
            if (per >= (uint32_t)at::SA_NW) per = per / at::SA_NW * at::SA_NW;
            return at::make_geo(g, per * nb, false, nbuf_env, ring_env, 1);
        }
        return at::make_geo(g, (uint32_t)((SMEM_MAX - hdr) / nbuf_env), false, nbuf_env, ring_env);
    };
    const size_t hdr1 = ((sizeof(at::SaSmem<1>) + 127) / 128) * 128;
    at::TreeGeo G1 = geo(hdr1);
    const size_t hdr2 = ((sizeof(at::SaSmem<2>) + 127) / 128) * 128;
    at::TreeGeo G2 = geo(hdr2);
    static int eb_env = -1;
    if (eb_env < 0) {
        const char *e = getenv("AT_SA_EB");
        eb_env = e ? atoi(e) : 1;
    }
    if (eb_env && G2.CH == at::SA_NW && !G2.resident && !G2.ring && G2.NP <= 1 && !G2.leaf_global) G2.eb = 1;
    static int grp_env = -1;
    if (grp_env < 0) {
        const char *e = getenv("AT_SA_GRP");   // 1 / 2 force the group count (measurement knob)
        grp_env = e ? atoi(e) : 0;
    }
    const bool fit2 = !acq && !G1.resident && at::sa_smem_bytes<2>(G2) <= SMEM_MAX;
    // two 32-chain groups per block (every streamed tree byte serves 64 chains) as soon as they still occupy
    // ~85 % of the SMs in one wave: measured on config 3, 8192 chains (128 blocks) run 1.55x faster with two
    // groups than with one (256 blocks), 4096 chains (64 blocks) 1.24x slower
    const bool use2 = grp_env == 2 ? fit2 : grp_env == 1 ? false : fit2 && (int64_t)o->n_chains * 20 >= (int64_t)64 * n_sm * 17;
    if (acq) {   // K models: 32 KB tree buffers leave room for the per-model partials
        G1 = at::make_geo(g, 32 * 1024);
        G1.Tm = g->n_trees / acq->n_models;
    }
    const at::TreeGeo G = use2 ? G2 : G1;
    const size_t smem = acq ? at::sa_smem_bytes<1, 8>(G) : use2 ? at::sa_smem_bytes<2>(G) : at::sa_smem_bytes<1>(G);
    if (smem > SMEM_MAX) return at::fail(AT_EUNSUPPORTED, "sa_explore: shared memory budget exceeded");
    // one template for every workload of the space: the compile-time specialised kernel
    int tm = sp->host.w[0].tmpl;
    for (int q = 1; q < sp->host.n_w; ++q)
        if (sp->host.w[q].tmpl != tm) tm = -1;
    if (acq) tm = -1;
    using KF = void (*)(at::SaParams, at::TreeGeo);
    const KF k1[4] = {at::sa_kernel<1, 1, -1>, at::sa_kernel<1, 1, 0>, at::sa_kernel<1, 1, 1>, at::sa_kernel<1, 1, 2>};
    const KF k2[4] = {at::sa_kernel<2, 1, -1>, at::sa_kernel<2, 1, 0>, at::sa_kernel<2, 1, 1>, at::sa_kernel<2, 1, 2>};
    const KF k1l[4] = {at::sa_kernel<1, 1, -1, true>, at::sa_kernel<1, 1, 0, true>, at::sa_kernel<1, 1, 1, true>,
                       at::sa_kernel<1, 1, 2, true>};
    const KF k2l[4] = {at::sa_kernel<2, 1, -1, true>, at::sa_kernel<2, 1, 0, true>, at::sa_kernel<2, 1, 1, true>,
                       at::sa_kernel<2, 1, 2, true>};
    // the one-tree-per-warp streamed pass (the config-3 geometry): a variant with only that walk compiled in
    const KF k2s[4] = {at::sa_kernel<2, 1, -1, false, 1>, at::sa_kernel<2, 1, 0, false, 1>,
                       at::sa_kernel<2, 1, 1, false, 1>, at::sa_kernel<2, 1, 2, false, 1>};
    // one group on the generic streamed pass (config 2): likewise, only that walk compiled in
    const KF k1g[4] = {at::sa_kernel<1, 1, -1, false, 3>, at::sa_kernel<1, 1, 0, false, 3>,
                       at::sa_kernel<1, 1, 1, false, 3>, at::sa_kernel<1, 1, 2, false, 3>};
    const bool lg = !acq && G.leaf_global;
    static int so_env = -1;
    if (so_env < 0) {
        const char *e = getenv("AT_SA_SO");   // "0": the generic kernel (measurement knob)
        so_env = e ? atoi(e) : 1;
    }
    const bool so = so_env && !acq && use2 && !lg && G.CH == at::SA_NW && !G.resident && !G.ring && G.NP <= 1 &&
                    G.D >= 6 && G.D <= 8;
    const bool gen1 = so_env && !acq && !use2 && !lg && !G.resident && !G.ring && G.NP <= 1;
    const KF kern = acq ? at::sa_kernel<1, 8, -1> : so ? k2s[tm + 1] : gen1 ? k1g[tm + 1]
                  : use2 ? (lg ? k2l : k2)[tm + 1] : (lg ? k1l : k1)[tm + 1];
    static size_t attr[25] = {0};
    const int ai = acq ? 16 : so ? 17 + tm + 1 : gen1 ? 21 + tm + 1 : (lg ? 8 : 0) + (use2 ? 4 : 0) + tm + 1;
    if (smem > attr[ai]) {
        AT_CUDA_TRY(cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[ai] = smem;
    }
    {
        at::ProfScope ps(AT_K_SA, s);
        const int cpb = use2 ? 64 : 32;
        const unsigned blocks = (unsigned)((o->n_chains + cpb - 1) / cpb);
        kern<<<blocks, at::SA_NWARPS * 32, smem, s>>>(P, G);   // 16 walkers + the producer
        at::note_launch();
        AT_LAUNCH_CHECK("sa_kernel");
    }
    if (lists) {
        AT_CUDA_TRY(cudaMemsetAsync(list_n, 0, at::MAXW * sizeof(int32_t), s));
        at::topk_chain_lists(d_chain_workload, o->n_chains, sp->host.n_w, chain_list, list_n, s);
        AT_LAUNCH_CHECK("chain lists");
    }
    // one batched top-k over all workloads (chain lists), or one pass per workload
    const int nb = lists ? sp->host.n_w : 1;
    for (int w = 0; w < sp->host.n_w; w += nb) {
        at::TkArgs a{};
        a.mode = 0;
        a.chain_list = lists ? chain_list : nullptr;
        a.list_n = list_n;
        a.keys = keys;
        a.n_src = n_keys;
        a.n_chains = o->n_chains;
        a.chain_w = d_chain_workload;
        a.w = w;
        a.offset_w = sp->host.offset[w];
        a.measured = d_measured_sorted;
        a.n_measured = n_measured;
        a.K = o->k_out;
        a.out_idx = d_out_idx + (int64_t)w * o->k_out;
        a.out_score = d_out_score + (int64_t)w * o->k_out;
        a.out_n = d_out_n + w;
        if (!d_chain_workload && w > 0) {
            // no chain belongs to this workload: empty list
            a.n_src = 0;
        }
        uint64_t offs[at::MAXW];
        for (int q = 0; q < at::MAXW; ++q) offs[q] = q < sp->host.n_w ? sp->host.offset[q] : 0;
        // the threshold fast path settles (almost) every workload; the exact tile reduction then runs only
        // for the rows it flagged (AT_TOPK_FAST=0: the tile reduction alone)
        static int fast_env = -1;
        if (fast_env < 0) {
            const char *e = getenv("AT_TOPK_FAST");
            fast_env = e ? atoi(e) : 1;
        }
        if (fast_env) {
            rc = at::topk_fast(a, nb, offs, per, fastbuf, fb, s);
            if (rc) return rc;
        }
        rc = at::topk_run(a, tkbuf, s, nb, offs, fast_env ? fb : nullptr);
        if (rc) return rc;
    }
    return AT_OK;
}
