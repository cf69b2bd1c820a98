// gbt.cuh -- device-side GBT walk + canonical reduction (reading Q19), shared by gbt_predict
// and sa_explore.
//
// Trees reach shared memory by TMA bulk copies (cp.async.bulk, completion on an mbarrier)
// in chunks of CH trees (nodes [CH][2^D-1] uint2 {feature, threshold bits}, then leaves
// [CH][2^D] f32), double-buffered: while the block walks chunk c, chunk c+1 is in flight
// and chunk c+2 is issued as soon as every warp has left c's buffer.  An ensemble that
// fits in the two buffers is loaded once and stays resident.
//
// A block owns 32 candidates (lane = candidate) whose features sit in shared memory as
// tile[f * 32 + lane] (bank = lane for every f: conflict-free gathers whatever node each
// lane is at).  Its NW warps split the trees by residue class: warp w walks the trees
// t = w (mod NW); the NQ = 32/NW partial sums p[q], q = t mod 32, stay in registers and
// receive leaves in ascending t, exactly the canonical order.  Walks of the NQ trees of a
// 32-tree round advance level by level together (NQ independent dependency chains).
#pragma once
#include "at_common.cuh"
#include "tma.cuh"

namespace at {

struct TreeGeo {
    const uint8_t *nodes;   // [T_pad][ni] uint2 {feature, threshold bits} (nbytes 8) or rank words (nbytes 4)
    int nbytes;             // bytes per internal node
    const float *leaf;      // [T_pad][nl]
    int T, T_pad, D, ni, nl;
    int CH;                 // trees per chunk (even: 16-B aligned bulk copies)
    int NC;                 // chunks per pass
    uint32_t chunk_bytes;   // CH * (ni * nbytes + nl * 4)
    int resident;           // NC <= NBUF: loaded once, never re-streamed
    int Tm;                 // trees per model (KM > 1: K equal models concatenated, gbt_predict_acq)
    int NBUF;               // chunk buffers (2: double buffering; up to TS_MAXBUF in ring mode)
    int ring;               // 0: a block barrier after every chunk; 1: no block barrier -- per-buffer
                            // consumption counters, the last warp done with a chunk refills its buffer
    int leaf_global;        // 1: chunks carry the nodes only; a walk's leaf is read from global memory
                            // (L2) and added one batch later (walk_batch<..., LG>), so the tree buffers
                            // hold 1.5x the trees of a depth-8 ensemble
    int eb;                 // 1 (walk_stream_one only): no chunk barrier -- walkers wait on the chunk's full
                            // mbarrier and count out on its empty mbarrier; the producer refills after it
    int NP;                 // > 1: NP independent tree pipelines (walk_pass): warp group p of NW / NP warps
                            // streams its own slices of CH = NW / NP trees through its own two buffers,
                            // with full / empty mbarriers and no block barrier; NC counts slices
};

// stream uses per pass (the unit of the stream counter c): chunks, or each pipeline's slices
__host__ __device__ inline int ts_uses_per_pass(const TreeGeo &G) { return G.NP > 1 ? G.NC / G.NP : G.NC; }

// pipeline q's use v of the stream: slice (v mod per) NP + q of pass v / per into slot 2q + (v & 1)
__device__ __forceinline__ void ts_issue_slice(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, int q, uint64_t v)
{
    const uint32_t per = (uint32_t)(G.NC / G.NP);
    const int s = (int)((uint32_t)v % per) * G.NP + q;
    const int slot = 2 * q + (int)(v & 1);
    const int t0 = s * G.CH;
    const uint32_t nb = (uint32_t)G.CH * G.ni * (uint32_t)G.nbytes, lb = (uint32_t)G.CH * G.nl * 4u;
    uint8_t *dst = bufs + (size_t)slot * G.chunk_bytes;
    mbar_arrive_expect_tx(&bar[slot], nb + lb);
    bulk_g2s(dst, G.nodes + (int64_t)t0 * G.ni * G.nbytes, nb, &bar[slot]);
    bulk_g2s(dst + (size_t)G.CH * G.ni * G.nbytes, G.leaf + (int64_t)t0 * G.nl, lb, &bar[slot]);
}
constexpr int TS_MAXBUF = 4;
#ifndef AT_SA_SPEC
#define AT_SA_SPEC 1   // speculative levels of the eb walk: 1 = the root's children + the leaf pair (measured best)
#endif
static_assert(AT_SA_SPEC >= 1, "the eb walk's root step always loads the root's children");

constexpr uint32_t TREE_BUF_BYTES = 48 * 1024;   // default per buffer (two buffers)
#ifdef AT_SA_PHASE_TIMING
__shared__ unsigned long long s_walk_prof[3 * 17];   // instrumented builds only (tools/sa_phases.py)
#endif
TreeGeo make_geo(const at_gbt_s *g, uint32_t buf_bytes = TREE_BUF_BYTES, bool rank = false, int nbuf = 2, int ring = 0,
                 int leaf_global = 0);

// leaves of the last walked batch, in flight from global memory (LG mode): added to the partial sums
// when the next batch is done, before its own leaves -- ascending t per residue class, as in Q19
template <int GRP, int NBMAX>
struct LeafPend {
    float v[GRP][NBMAX];
    int j[NBMAX];
    int n;
};

__device__ __forceinline__ void ts_issue(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint64_t c)
{
    const int k = (int)((uint32_t)c % (uint32_t)G.NC);     // (32-bit: a 64-bit modulo is ~100 cycles)
    const int b = (int)((uint32_t)c % (uint32_t)G.NBUF);
    const int t0 = k * G.CH;
    const int nt = min(G.CH, G.T_pad - t0);
    const uint32_t nb = (uint32_t)nt * G.ni * (uint32_t)G.nbytes, lb = (uint32_t)nt * G.nl * 4u;
    uint8_t *dst = bufs + (size_t)b * G.chunk_bytes;
#ifdef AT_SA_NOSTREAM
    // experiment only (tools): after the first buffers, complete the chunk without copying -- the walk
    // then reuses stale trees, which isolates the cost of the L2 -> shared stream
    if (c >= (uint64_t)G.NBUF) { mbar_arrive(&bar[b]); return; }
#endif
    if (G.leaf_global) {
        mbar_arrive_expect_tx(&bar[b], nb);
        bulk_g2s(dst, G.nodes + (int64_t)t0 * G.ni * G.nbytes, nb, &bar[b]);
        return;
    }
    mbar_arrive_expect_tx(&bar[b], nb + lb);
    bulk_g2s(dst, G.nodes + (int64_t)t0 * G.ni * G.nbytes, nb, &bar[b]);
    bulk_g2s(dst + (size_t)G.CH * G.ni * G.nbytes, G.leaf + (int64_t)t0 * G.nl, lb, &bar[b]);
}

// thread 0: initialise the NBUF barriers (and, ring mode, the consumption counters that follow them
// in `bar`) and start the first NBUF chunks of the stream
__device__ __forceinline__ void ts_start(const TreeGeo &G, uint8_t *bufs, uint64_t *bar)
{
    if (threadIdx.x == 0) {
        if (G.NP > 1) {   // full[2 NP] (one arrival + tx), then empty[2 NP] (one arrival per walker warp)
            for (int b = 0; b < 2 * G.NP; ++b) {
                mbar_init(&bar[b], 1);
                mbar_init(&bar[2 * G.NP + b], 16 / G.NP);
            }
            fence_proxy_async();
            for (int q = 0; q < G.NP; ++q) {
                ts_issue_slice(G, bufs, bar, q, 0);
                ts_issue_slice(G, bufs, bar, q, 1);
            }
            return;
        }
        for (int b = 0; b < G.NBUF; ++b) {
            mbar_init(&bar[b], 1);
            if (G.ring) ((unsigned *)(bar + G.NBUF))[b] = 0u;
            if (G.eb) mbar_init(&bar[G.NBUF + b], 16);   // empty: one arrival per walker warp
        }
        fence_proxy_async();
        for (int b = 0; b < G.NBUF && b < G.NC; ++b) ts_issue(G, bufs, bar, (uint64_t)b);
    }
}

// A batch of NB trees t = t0, t0 + NW, ... (all owned by this warp: t = warp mod NW) walked for
// GRP candidate groups at once: NB * GRP independent dependency chains.  RK: rank form -- 4-byte
// nodes {k | tile byte offset of the feature << 16}, tiles of u16 feature ranks in pairs,
// x < theta <=> rank < k.
template <int NW, int GRP, int NB, int KM, bool RK = false, bool LG = false, int NBP = 1>
__device__ __forceinline__ void walk_batch(const TreeGeo &G, const uint8_t *buf, int c0, int t0, const void *tile,
                                           int gstride, int lane, float (&p)[GRP][KM][32 / NW],
                                           uint8_t *__restrict__ slots, int64_t slot_ld, int64_t cand0,
                                           const bool (&cand_ok)[GRP], LeafPend<GRP, NBP> &pend)
{
    constexpr int NQ = 32 / NW;
    constexpr uint32_t NBY = RK ? 4u : 8u;   // bytes per node
    const float *leaves = (const float *)(buf + (size_t)G.CH * G.ni * NBY);
    const int D = G.D, ni = G.ni, nl = G.nl;
    const uint32_t tree_bytes = (uint32_t)ni * NBY;
    // a = shared address of the current node = tb + NBY h (h: 1-based heap index, tb = tree base -
    // NBY); the left child 2h sits at 2a - tb, the right one 2h + 1 at 2a - tb + NBY, so one select
    // of a precomputed addend and one 3-input add advance a walk: LDS.64, IMAD, LDS, FSETP, SEL, IADD3
    uint32_t add_l[NB], add_r[NB], a[GRP][NB];
#pragma unroll
    for (int jj = 0; jj < NB; ++jj) {
        const uint32_t tb = (uint32_t)__cvta_generic_to_shared(buf) + (uint32_t)(t0 + jj * NW - c0) * tree_bytes - NBY;
        add_l[jj] = 0u - tb;
        add_r[jj] = NBY - tb;
#pragma unroll
        for (int g = 0; g < GRP; ++g) a[g][jj] = tb + NBY;
    }
    for (int d = 0; d < D; ++d) {
#pragma unroll
        for (int g = 0; g < GRP; ++g) {
            if (RK) {
                // u32 tile of rank pairs: feature f of candidate `lane` at + (f / 2) * 128 + (f % 2) * 2
                // (bank = lane whatever f); the node's high half is that byte offset, the low half k
                const uint32_t tile_lane =
                    (uint32_t)__cvta_generic_to_shared((const uint32_t *)tile + g * gstride + lane);
#pragma unroll
                for (int jj = 0; jj < NB; ++jj) {
                    uint32_t nd, x;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nd) : "r"(a[g][jj]));
                    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(tile_lane + (nd >> 16)));
                    a[g][jj] = 2u * a[g][jj] + (x < (nd & 0xFFFFu) ? add_l[jj] : add_r[jj]);
                }
            } else {
                const uint32_t tile_lane =
                    (uint32_t)__cvta_generic_to_shared((const float *)tile + g * gstride + lane);   // f at + f * 128
#pragma unroll
                for (int jj = 0; jj < NB; ++jj) {
                    uint32_t nf, nt;
                    float x;
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nf), "=r"(nt) : "r"(a[g][jj]));
                    AT_DCHECK(nf < (uint32_t)(gstride / 32));   // a feature row of the tile
                    AT_DCHECK(((a[g][jj] + add_l[jj]) >> 3) >= 1u && ((a[g][jj] + add_l[jj]) >> 3) <= (uint32_t)ni);   // heap index
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile_lane + (nf << 7)));
                    const uint32_t al = 2u * a[g][jj] + add_l[jj];
                    a[g][jj] = x < __uint_as_float(nt) ? al : al + NBY;
                }
            }
        }
    }
    if constexpr (LG) {
        // the previous batch's leaves (loaded one batch ago) go first, then this batch's leaf loads are
        // issued straight into the pending registers
#pragma unroll
        for (int jj = 0; jj < NBP; ++jj)
            if (jj < pend.n)
#pragma unroll
                for (int g = 0; g < GRP; ++g)
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (q == pend.j[jj]) p[g][0][q] = __fadd_rn(p[g][0][q], pend.v[g][jj]);
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) {
            const int t = t0 + jj * NW;
            pend.j[jj] = (t & 31) / NW;
#pragma unroll
            for (int g = 0; g < GRP; ++g) {
                const int slot = (int)((a[g][jj] + add_l[jj]) >> (RK ? 2 : 3)) - nl;
                AT_DCHECK(slot >= 0 && slot < nl);
                pend.v[g][jj] = __ldg(G.leaf + (int64_t)t * nl + slot);
            }
        }
        pend.n = NB;
    } else {
        // leaves in ascending t: tree t adds to its residue class q = t mod 32, slot (q - warp) / NW = q / NW;
        // with KM models of Tm trees, tree t = km Tm + u adds to model km's class u mod 32 (all trees of
        // one (model, class) pair share t mod NW, so one warp owns it and sums it in ascending u)
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) {
            const int t = t0 + jj * NW;
            int km = 0, u = t;
            if (KM > 1) { km = t / G.Tm; u = t - km * G.Tm; }
            const int j = (u & 31) / NW;
#pragma unroll
            for (int g = 0; g < GRP; ++g) {
                const int slot = (int)((a[g][jj] + add_l[jj]) >> (RK ? 2 : 3)) - nl;   // h = (a - tb) / NBY in [2^D, 2^(D+1))
                AT_DCHECK(slot >= 0 && slot < nl);
                AT_DCHECK(t - c0 >= 0 && t - c0 < G.CH);
                const float lv = leaves[(t - c0) * nl + slot];
#pragma unroll
                for (int m = 0; m < KM; ++m)
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (m == km && q == j) p[g][m][q] = __fadd_rn(p[g][m][q], lv);
                if (slots && cand_ok[g]) slots[(int64_t)t * slot_ld + cand0 + 32 * g] = (uint8_t)slot;
            }
        }
    }
}

// One pass over a streamed ensemble whose chunks hold exactly NW trees (one per walker warp: tree
// NW k + warp of chunk k), fp32 nodes, compile-time depth D, with a producer warp PW: the SA kernel's
// depth-6..8 walk.  Everything that does not change from chunk to chunk -- the warp's tree base in
// either buffer, its leaf row, the lane's tile address, the depth dispatch -- is computed once per
// pass, so a chunk starts walking right after the barrier (the per-chunk setup of the generic
// walk_chunk was ~25 % of the kernel's stall samples).  Sums exactly as walk_batch<NB = 1> does: tree
// t adds its leaf to class t mod 32 in ascending t.
template <int NW, int GRP, int D, int PW>
__device__ __forceinline__ void walk_stream_one(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint32_t *ph,
                                                uint64_t &c, uint64_t c_limit, const float *tile, int gstride,
                                                int lane, int warp, float (&p)[GRP][1][32 / NW])
{
    constexpr int NQ = 32 / NW;
    constexpr uint32_t ni = (1u << D) - 1u, nl = 1u << D;
    const bool walker = warp < PW;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bufs);
    const uint32_t tbw = sb + (uint32_t)warp * ni * 8u - 8u;                       // + buffer offset
    const uint32_t lfw = sb + (uint32_t)G.CH * ni * 8u + (uint32_t)warp * nl * 4u;  // + buffer offset
    const uint32_t tile0 = (uint32_t)__cvta_generic_to_shared(tile + lane);
    const uint32_t gbytes = (uint32_t)gstride * 4u;
    const int T = G.T, NC = G.NC;
    const uint32_t cbytes = G.chunk_bytes;
    // 32-bit stream counters (c_limit < 2^32) and running per-chunk values: no 64-bit or multiply in the
    // chunk loop's critical path
    uint32_t cc = (uint32_t)c;
    const uint32_t climit = (uint32_t)c_limit;
    uint32_t boff = (cc & 1u) ? cbytes : 0u;
    int t = warp;
    if (G.eb) {
        // no chunk barrier: walkers wait on the chunk's full barrier and count out on its empty barrier;
        // the producer refills a buffer as soon as all walkers left it
        for (int k = 0; k < NC; ++k, ++cc, t += NW, boff ^= cbytes) {
            const int b = (int)(cc & 1u);
            const uint32_t par = (cc >> 1) & 1u;
            if (walker) {
                mbar_wait(&bar[b], par);
                if (t < T) {
                    // Speculative descent: on the top SPEC levels a node's two children (adjacent in the
                    // heap) are loaded beside its feature value, so the dependent chain per level is one
                    // shared load instead of two; the last level loads its two leaves (one 8-B pair)
                    // beside the feature.  Same comparisons, same leaves: bit-identical to the plain walk.
                    constexpr int SPEC = D - 1 < AT_SA_SPEC ? D - 1 : AT_SA_SPEC;
                    const uint32_t tb = tbw + boff;
                    const uint32_t add_l = 0u - tb;   // (the right child is the left one + 8 bytes)
                    uint32_t a[GRP], cf[GRP], ct[GRP];   // current node: address, feature, threshold bits
                    {   // the root and its two children: one load each serves every group
                        uint32_t rf, rt, lf, lt, qf, qt;
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(rf), "=r"(rt) : "r"(tb + 8u));
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lf), "=r"(lt) : "r"(tb + 16u));
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(qf), "=r"(qt) : "r"(tb + 24u));
#pragma unroll
                        for (int g = 0; g < GRP; ++g) {
                            float x;
                            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (rf << 7)));
                            const bool c = x < __uint_as_float(rt);
                            a[g] = c ? tb + 16u : tb + 24u;
                            cf[g] = c ? lf : qf;
                            ct[g] = c ? lt : qt;
                        }
                    }
#pragma unroll
                    for (int d = 1; d < SPEC; ++d) {
#pragma unroll
                        for (int g = 0; g < GRP; ++g) {
                            const uint32_t la = 2u * a[g] + add_l;
                            uint32_t lf, lt, qf, qt;
                            float x;
                            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (cf[g] << 7)));
                            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lf), "=r"(lt) : "r"(la));
                            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(qf), "=r"(qt) : "r"(la + 8u));
                            const bool c = x < __uint_as_float(ct[g]);
                            a[g] = c ? la : la + 8u;
                            cf[g] = c ? lf : qf;
                            ct[g] = c ? lt : qt;
                        }
                    }
                    // a[g] is a level-SPEC node with its data in (cf, ct)
                    if constexpr (SPEC < D - 1) {
#pragma unroll
                        for (int g = 0; g < GRP; ++g) {
                            float x;
                            const uint32_t al = 2u * a[g] + add_l;   // both children's addresses off the chain
                            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (cf[g] << 7)));
                            a[g] = x < __uint_as_float(ct[g]) ? al : al + 8u;
                        }
#pragma unroll
                        for (int d = SPEC + 1; d < D - 1; ++d) {
#pragma unroll
                            for (int g = 0; g < GRP; ++g) {
                                uint32_t nf, nt;
                                float x;
                                const uint32_t al = 2u * a[g] + add_l;
                                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nf), "=r"(nt) : "r"(a[g]));
                                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (nf << 7)));
                                a[g] = x < __uint_as_float(nt) ? al : al + 8u;
                            }
                        }
#pragma unroll
                        for (int g = 0; g < GRP; ++g)
                            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cf[g]), "=r"(ct[g]) : "r"(a[g]));
                    }
                    // last level: its feature value and its two leaves (slots 2 idx + 2 - 2^D, + 1) together
                    const int j = (t & 31) / NW;
#pragma unroll
                    for (int g = 0; g < GRP; ++g) {
                        const uint32_t slot = ((a[g] + add_l) >> 2) - nl;
                        float x, lL, lR;
                        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (cf[g] << 7)));
                        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(lL), "=f"(lR) : "r"(lfw + boff + slot * 4u));
                        const float lv = x < __uint_as_float(ct[g]) ? lL : lR;
#pragma unroll
                        for (int q = 0; q < NQ; ++q)
                            if (q == j) p[g][0][q] = __fadd_rn(p[g][0][q], lv);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar[2 + b]);
            } else if (warp == PW && lane == 0) {
                mbar_wait(&bar[2 + b], par);   // every walker left chunk cc
                if (cc + 2u < climit) {
                    fence_proxy_async();
                    ts_issue(G, bufs, bar, (uint64_t)cc + 2u);
                }
            }
        }
        c = cc;
        return;
    }
    for (int k = 0; k < NC; ++k, ++cc, t += NW, boff ^= cbytes) {
        if (cc == 0u) {   // the kernel's first chunk; later ones are waited for by the producer (below)
            mbar_wait(&bar[0], ph[0]);
            ph[0] ^= 1u;
        }
        if (walker && t < T) {
            const uint32_t tb = tbw + boff;
            const uint32_t add_l = 0u - tb, add_r = 8u - tb;
            uint32_t a[GRP];
            {   // the root: one node load serves every group
                uint32_t nf, nt;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nf), "=r"(nt) : "r"(tb + 8u));
                AT_DCHECK(nf < (uint32_t)(gstride / 32));
#pragma unroll
                for (int g = 0; g < GRP; ++g) {
                    float x;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (nf << 7)));
                    a[g] = 2u * (tb + 8u) + (x < __uint_as_float(nt) ? add_l : add_r);
                }
            }
#pragma unroll
            for (int d = 1; d < D; ++d) {
#pragma unroll
                for (int g = 0; g < GRP; ++g) {
                    uint32_t nf, nt;
                    float x;
                    const uint32_t al = 2u * a[g] + add_l;   // both children's addresses off the chain
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nf), "=r"(nt) : "r"(a[g]));
                    AT_DCHECK(nf < (uint32_t)(gstride / 32));
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile0 + (uint32_t)g * gbytes + (nf << 7)));
                    a[g] = x < __uint_as_float(nt) ? al : al + 8u;
                }
            }
            const int j = (t & 31) / NW;
#pragma unroll
            for (int g = 0; g < GRP; ++g) {
                const uint32_t slot = ((a[g] + add_l) >> 3) - nl;
                AT_DCHECK(slot < nl);
                float lv;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lv) : "r"(lfw + boff + slot * 4u));
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (q == j) p[g][0][q] = __fadd_rn(p[g][0][q], lv);
            }
        } else if (warp == PW && cc + 1u < climit) {
            // the producer waits for the NEXT chunk before the block barrier, so the barrier publishes it
            const int b1 = (int)((cc + 1u) & 1u);
            mbar_wait(&bar[b1], ph[b1]);
            ph[b1] ^= 1u;
        }
        __syncthreads();   // every warp is done with this chunk's buffer
        if (warp == PW && lane == 0 && cc + 2u < climit) {
            fence_proxy_async();
            ts_issue(G, bufs, bar, (uint64_t)cc + 2u);
        }
    }
    c = cc;
}

// x < (nd & 0xFFFF) for u16 ranks, as one fp16 compare of the low halves: ranks and node ranks are at
// most 257 (positive fp16 subnormals, ordered like their integers; the compare keeps subnormals) and a
// NaN feature's rank 0xFFFF is an fp16 NaN, which compares false -- as 0xFFFF < k does.  Returns
// lt ? al : al + step without a separate mask of nd.
__device__ __forceinline__ uint32_t rank_step(uint32_t x, uint32_t nd, uint32_t al, uint32_t step)
{
    uint32_t r;
    asm("{\n.reg .b16 xl, xh, kl, kh;\n.reg .pred p;\nmov.b32 {xl, xh}, %1;\nmov.b32 {kl, kh}, %2;\n"
        "setp.lt.f16 p, xl, kl;\nadd.u32 %0, %3, %4;\n@p mov.u32 %0, %3;\n}"
        : "=r"(r)
        : "r"(x), "r"(nd), "r"(al), "r"(step));
    return r;
}

// The rank-form counterpart for gbt_predict's streamed depth-6..8 ensembles: chunks of TPW NW trees,
// TPW trees per walker warp (tree NW (TPW k + jj) + warp, jj < TPW), walked for GRP candidate groups
// at once (TPW GRP independent chains), 4-byte nodes {k | tile byte offset << 16} against u16
// feature ranks (x < theta <=> rank < k).  Per-pass constants hoisted as in walk_stream_one; leaves
// added in ascending t per residue class (jj ascending = t ascending).
template <int NW, int GRP, int D, int PW, int TPW>
__device__ __forceinline__ void walk_stream_rank(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint32_t *ph,
                                                 uint64_t &c, uint64_t c_limit, const uint32_t *tile, int gstride,
                                                 int lane, int warp, float (&p)[GRP][1][32 / NW])
{
    constexpr int NQ = 32 / NW;
    constexpr uint32_t ni = (1u << D) - 1u, nl = 1u << D;
    const bool walker = warp < PW;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bufs);
    const uint32_t tbw = sb + (uint32_t)warp * ni * 4u - 4u;                       // + buffer + jj NW trees
    const uint32_t lfw = sb + (uint32_t)G.CH * ni * 4u + (uint32_t)warp * nl * 4u;  // + buffer + jj NW leaf rows
    const uint32_t tile0 = (uint32_t)__cvta_generic_to_shared(tile + lane);
    const uint32_t gbytes = (uint32_t)gstride * 4u;
    const int T = G.T, NC = G.NC;
    const uint32_t cbytes = G.chunk_bytes;
    uint32_t cc = (uint32_t)c;
    const uint32_t climit = (uint32_t)c_limit;
    uint32_t boff = (cc & 1u) ? cbytes : 0u;
    int t = warp;
    for (int k = 0; k < NC; ++k, ++cc, t += TPW * NW, boff ^= cbytes) {
        if (cc == 0u) {
            mbar_wait(&bar[0], ph[0]);
            ph[0] ^= 1u;
        }
        if (walker && t < T) {
            uint32_t a[TPW][GRP], add_l[TPW];   // (right child = left + 4 bytes)
            const bool two = TPW > 1 && t + NW < T;   // warp-uniform: the chunk's second tree exists
#pragma unroll
            for (int jj = 0; jj < TPW; ++jj) {
                const uint32_t tb = tbw + boff + (uint32_t)(jj * NW) * ni * 4u;
                add_l[jj] = 0u - tb;
                if (jj > 0 && !two) break;
                uint32_t nd;   // the root: one node load serves every group
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nd) : "r"(tb + 4u));
                const uint32_t al = 2u * (tb + 4u) + add_l[jj];
#pragma unroll
                for (int g = 0; g < GRP; ++g) {
                    uint32_t x;
                    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(tile0 + (uint32_t)g * gbytes + (nd >> 16)));
                    a[jj][g] = rank_step(x, nd, al, 4u);
                }
            }
#pragma unroll
            for (int d = 1; d < D; ++d) {
#pragma unroll
                for (int jj = 0; jj < TPW; ++jj) {
                    if (jj > 0 && !two) break;
#pragma unroll
                    for (int g = 0; g < GRP; ++g) {
                        uint32_t nd, x;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nd) : "r"(a[jj][g]));
                        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(x) : "r"(tile0 + (uint32_t)g * gbytes + (nd >> 16)));
                        const uint32_t al = 2u * a[jj][g] + add_l[jj];
                        a[jj][g] = rank_step(x, nd, al, 4u);
                    }
                }
            }
#pragma unroll
            for (int jj = 0; jj < TPW; ++jj) {
                if (jj > 0 && !two) break;
                const int j = ((t + jj * NW) & 31) / NW;
#pragma unroll
                for (int g = 0; g < GRP; ++g) {
                    const uint32_t slot = ((a[jj][g] + add_l[jj]) >> 2) - nl;
                    AT_DCHECK(slot < nl);
                    float lv;
                    asm volatile("ld.shared.f32 %0, [%1];"
                                 : "=f"(lv)
                                 : "r"(lfw + boff + (uint32_t)(jj * NW) * nl * 4u + slot * 4u));
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (q == j) p[g][0][q] = __fadd_rn(p[g][0][q], lv);
                }
            }
        } else if (warp == PW && cc + 1u < climit) {
            const int b1 = (int)((cc + 1u) & 1u);
            mbar_wait(&bar[b1], ph[b1]);
            ph[b1] ^= 1u;
        }
        __syncthreads();
        if (warp == PW && lane == 0 && cc + 2u < climit) {
            fence_proxy_async();
            ts_issue(G, bufs, bar, (uint64_t)cc + 2u);
        }
    }
    c = cc;
}

// Walk one staged chunk [c0, c1): every warp takes the trees of its residue classes (t = warp mod NW)
// in ascending order, in batches of up to 4 / GRP trees; no walk slot is spent on an absent tree,
// whatever the chunk size.  GRP candidate groups of 32 (group g's tile at tile + g * gstride floats)
// share every staged tree byte.
template <int GRP, int KM>
constexpr int walk_nbmax() { return GRP == 1 ? (KM == 1 ? 6 : 4) : (GRP == 2 && KM == 1 ? 4 : 2); }

template <int NW, int GRP, int KM, bool RK = false, bool LG = false>
__device__ __forceinline__ void walk_chunk(const TreeGeo &G, const uint8_t *buf, int k, const void *tile, int gstride,
                                           int lane, int warp, float (&p)[GRP][KM][32 / NW], uint8_t *__restrict__ slots,
                                           int64_t slot_ld, int64_t cand0, const bool (&cand_ok)[GRP],
                                           LeafPend<GRP, walk_nbmax<GRP, KM>()> &pend)
{
    constexpr int NBMAX = walk_nbmax<GRP, KM>();
    const int c0 = k * G.CH;
    const int c1 = min(c0 + G.CH, G.T);
    int t0 = c0 + ((warp - c0) % NW + NW) % NW;
    for (; t0 + (NBMAX - 1) * NW < c1; t0 += NBMAX * NW)
        walk_batch<NW, GRP, NBMAX, KM, RK, LG, NBMAX>(G, buf, c0, t0, tile, gstride, lane, p, slots, slot_ld, cand0, cand_ok,
                                                      pend);
    int rest = t0 < c1 ? (c1 - 1 - t0) / NW + 1 : 0;   // warp-uniform, < NBMAX
    if (NBMAX > 4 && rest >= 4) {
        walk_batch<NW, GRP, 4, KM, RK, LG, NBMAX>(G, buf, c0, t0, tile, gstride, lane, p, slots, slot_ld, cand0, cand_ok,
                                                      pend);
        t0 += 4 * NW;
        rest -= 4;
    }
    if (NBMAX >= 4 && rest == 3)
        walk_batch<NW, GRP, 3, KM, RK, LG, NBMAX>(G, buf, c0, t0, tile, gstride, lane, p, slots, slot_ld, cand0, cand_ok,
                                                      pend);
    else if (rest >= 2)
        walk_batch<NW, GRP, 2, KM, RK, LG, NBMAX>(G, buf, c0, t0, tile, gstride, lane, p, slots, slot_ld, cand0, cand_ok,
                                                      pend);
    else if (rest == 1)
        walk_batch<NW, GRP, 1, KM, RK, LG, NBMAX>(G, buf, c0, t0, tile, gstride, lane, p, slots, slot_ld, cand0, cand_ok,
                                                      pend);
}

// One full pass over the ensemble.  `c` is the block-wide stream counter (identical in every
// thread); `c_limit` the total number of chunks the kernel will consume.  Ends with group g's
// partials in part[g * pstride + q * 32 + lane] (KM models: part[g * pstride + (m 32 + q) 32 + lane])
// and a __syncthreads.
// PW >= 0: warp PW is a producer only -- it walks nothing and issues the tree-chunk copies (the
// issuing work, a proxy fence and two bulk copies, then never delays a walking warp)
// ONLY = 1 / 2: the caller guarantees the stream_one (sa_kernel) / stream_rank (gbt_predict rank form)
// geometry and only that walk is compiled in, so the hot loop is register-allocated and scheduled on its own
template <int NW, int GRP, int KM = 1, bool RK = false, bool LG = false, int PW = -1, int ONLY = 0>
__device__ __forceinline__ void walk_pass(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint32_t *ph, uint64_t &c,
                                          uint64_t c_limit, const void *tile, int gstride, int lane, int warp,
                                          float *part, int pstride, uint8_t *__restrict__ slots, int64_t slot_ld,
                                          int64_t cand0, const bool (&cand_ok)[GRP])
{
    constexpr int NQ = 32 / NW;
    float p[GRP][KM][NQ];
#pragma unroll
    for (int g = 0; g < GRP; ++g)
#pragma unroll
        for (int m = 0; m < KM; ++m)
#pragma unroll
            for (int j = 0; j < NQ; ++j) p[g][m][j] = 0.0f;
    LeafPend<GRP, walk_nbmax<GRP, KM>()> pend;
    pend.n = 0;
    const bool walker = PW < 0 || warp < PW;
    // the SA kernel's streamed chunks of one tree per walker warp (two chain groups, depth 6..8)
    // gbt_predict's streamed rank-form depth-7/8 chunks of NW or 2 NW trees
    const bool stream_rank = PW >= 0 && KM == 1 && RK && !LG && !G.resident && !G.ring && G.NP <= 1 &&
                             (G.CH == NW || G.CH == 2 * NW) && slots == nullptr && G.D >= 7 && G.D <= 8;
    const bool stream_one = PW >= 0 && GRP == 2 && KM == 1 && !RK && !LG && !G.resident && !G.ring && G.NP <= 1 &&
                            G.CH == NW && slots == nullptr && G.D >= 6 && G.D <= 8;
    // the generic streamed pass: a block barrier after every chunk (ONLY = 3 compiles this one alone)
    auto generic_pass = [&]() {
        for (int k = 0; k < G.NC; ++k, ++c) {
            const int b = (int)(c & 1);
#ifdef AT_SA_PHASE_TIMING
            long long q0 = clock64();
#endif
            if (PW < 0 || c == 0) {   // with a producer warp only the kernel's first chunk is waited for here
                mbar_wait(&bar[b], ph[b]);
                ph[b] ^= 1u;
            }
#ifdef AT_SA_PHASE_TIMING
            long long q1 = clock64();
#endif
            if (walker) {
                walk_chunk<NW, GRP, KM, RK, LG>(G, bufs + (size_t)b * G.chunk_bytes, k, tile, gstride, lane, warp, p,
                                                slots, slot_ld, cand0, cand_ok, pend);
            } else if (warp == PW && c + 1 < c_limit) {
                // the producer waits for the NEXT chunk before the block barrier, so the barrier itself
                // publishes it: the walkers start it without an mbarrier wait of their own
                const int b1 = (int)((c + 1) & 1);
                mbar_wait(&bar[b1], ph[b1]);
                ph[b1] ^= 1u;
            }
#ifdef AT_SA_PHASE_TIMING
            long long q2 = clock64();
#endif
            __syncthreads();   // every warp is done with buffer b
#ifdef AT_SA_PHASE_TIMING
            if (lane == 0 && warp < 17) {
                const long long q3 = clock64();
                s_walk_prof[3 * warp] += q1 - q0;
                s_walk_prof[3 * warp + 1] += q2 - q1;
                s_walk_prof[3 * warp + 2] += q3 - q2;
            }
#endif
            if ((PW < 0 ? threadIdx.x == 0 : (warp == PW && lane == 0)) && c + 2 < c_limit) {
                fence_proxy_async();
                ts_issue(G, bufs, bar, c + 2);
            }
        }
    };
    if constexpr (ONLY == 1) {
        static_assert(PW >= 0 && GRP == 2 && KM == 1 && !RK && !LG, "ONLY = 1: the stream_one geometry");
        const float *tf = (const float *)tile;
        if (G.D == 8)
            walk_stream_one<NW, GRP, 8, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
        else if (G.D == 7)
            walk_stream_one<NW, GRP, 7, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
        else
            walk_stream_one<NW, GRP, 6, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
    } else if constexpr (ONLY == 3) {
        generic_pass();
    } else if constexpr (ONLY == 2) {
        static_assert(PW >= 0 && KM == 1 && RK && !LG, "ONLY = 2: the stream_rank geometry");
        const uint32_t *tu = (const uint32_t *)tile;
        const int tpw = G.CH / NW;
        if (G.D == 8 && tpw == 2)
            walk_stream_rank<NW, GRP, 8, PW, 2>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
        else if (G.D == 8)
            walk_stream_rank<NW, GRP, 8, PW, 1>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
        else if (G.D == 7 && tpw == 2)
            walk_stream_rank<NW, GRP, 7, PW, 2>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
        else
            walk_stream_rank<NW, GRP, 7, PW, 1>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
    } else if (PW >= 0 && G.NP > 1) {
        // NP independent pipelines, no block barrier: warp group p (NW / NP warps) walks its slices -- each
        // warp one tree per slice -- waiting on the slot's full barrier and counting out on its empty
        // barrier; lane q of the producer warp refills pipeline q's slot as soon as its walkers are out.
        // The groups drift apart, so one group's fill / drain overlaps another's steady walk.
        const int per = G.NC / G.NP;
        if (walker) {
            const int pp = warp / (NW / G.NP);
            for (int kk = 0; kk < per; ++kk, ++c) {
                const int slot = 2 * pp + (int)(c & 1);
                mbar_wait(&bar[slot], (uint32_t)((c >> 1) & 1));
                walk_chunk<NW, GRP, KM, RK, LG>(G, bufs + (size_t)slot * G.chunk_bytes, kk * G.NP + pp, tile, gstride,
                                                lane, warp, p, slots, slot_ld, cand0, cand_ok, pend);
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar[2 * G.NP + slot]);
            }
        } else {
            if (warp == PW && lane < G.NP) {
                uint64_t u = c;
                for (int kk = 0; kk < per; ++kk, ++u) {
                    const int slot = 2 * lane + (int)(u & 1);
                    mbar_wait(&bar[2 * G.NP + slot], (uint32_t)((u >> 1) & 1));
                    if (u + 2 < c_limit) {
                        fence_proxy_async();
                        ts_issue_slice(G, bufs, bar, lane, u + 2);
                    }
                }
            }
            __syncwarp();
            c += per;
        }
    } else if (G.resident) {
        for (int k = 0; k < G.NC && walker; ++k)
            walk_chunk<NW, GRP, KM, RK, LG>(G, bufs + (size_t)k * G.chunk_bytes, k, tile, gstride, lane, warp, p, slots, slot_ld,
                                cand0, cand_ok, pend);
    } else if (G.ring) {
        // no block barrier per chunk: every warp waits for each chunk's data (so its phase bits stay
        // exact), walks the trees of its residue class in it, and counts itself out; the last of the NW
        // warps to leave chunk c refills that buffer with chunk c + NBUF.  Warps drift by up to NBUF - 1
        // chunks, so one slow warp no longer stalls the other NW - 1 at every chunk.
        unsigned *cnt = (unsigned *)(bar + G.NBUF);
        if (!walker) {
            // producer: chunk c's buffer is refilled with chunk c + NBUF once all NW walkers counted out
            if (lane == 0)
                for (int k = 0; k < G.NC; ++k, ++c) {
                    const int b = (int)((uint32_t)c % (uint32_t)G.NBUF);
                    const unsigned want = ((uint32_t)c / (uint32_t)G.NBUF + 1u) * (unsigned)NW;
                    while (*(volatile unsigned *)&cnt[b] < want) {
                    }
                    if (c + G.NBUF < c_limit) {
                        fence_proxy_async();
                        ts_issue(G, bufs, bar, c + G.NBUF);
                    }
                }
            else
                c += G.NC;
            c = __shfl_sync(0xFFFFFFFFu, c, 0);
        } else {
            for (int k = 0; k < G.NC; ++k, ++c) {
                const int b = (int)((uint32_t)c % (uint32_t)G.NBUF);
                mbar_wait(&bar[b], ph[b]);
                ph[b] ^= 1u;
                walk_chunk<NW, GRP, KM, RK, LG>(G, bufs + (size_t)b * G.chunk_bytes, k, tile, gstride, lane, warp, p, slots,
                                                slot_ld, cand0, cand_ok, pend);
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();   // this warp's reads of buffer b precede the refill
                    if (PW >= 0) {
                        atomicAdd(&cnt[b], 1u);
                    } else {
                        const unsigned old = atomicAdd(&cnt[b], 1u);
                        if (old % NW == NW - 1 && c + G.NBUF < c_limit) {
                            fence_proxy_async();
                            ts_issue(G, bufs, bar, c + G.NBUF);
                        }
                    }
                }
            }
        }
    } else if (stream_rank) {
        if constexpr (PW >= 0 && KM == 1 && RK && !LG) {
            const uint32_t *tu = (const uint32_t *)tile;
            const int tpw = G.CH / NW;
            if (G.D == 8 && tpw == 2)
                walk_stream_rank<NW, GRP, 8, PW, 2>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
            else if (G.D == 8)
                walk_stream_rank<NW, GRP, 8, PW, 1>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
            else if (G.D == 7 && tpw == 2)
                walk_stream_rank<NW, GRP, 7, PW, 2>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
            else
                walk_stream_rank<NW, GRP, 7, PW, 1>(G, bufs, bar, ph, c, c_limit, tu, gstride, lane, warp, p);
        }
    } else if (stream_one) {
        if constexpr (PW >= 0 && GRP == 2 && KM == 1 && !RK && !LG) {
            const float *tf = (const float *)tile;
            if (G.D == 8)
                walk_stream_one<NW, GRP, 8, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
            else if (G.D == 7)
                walk_stream_one<NW, GRP, 7, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
            else
                walk_stream_one<NW, GRP, 6, PW>(G, bufs, bar, ph, c, c_limit, tf, gstride, lane, warp, p);
        }
    } else {
        generic_pass();
    }
    if (LG) {   // the last batch's leaves
#pragma unroll
        for (int jj = 0; jj < walk_nbmax<GRP, KM>(); ++jj)
            if (jj < pend.n)
#pragma unroll
                for (int g = 0; g < GRP; ++g)
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (q == pend.j[jj]) p[g][0][q] = __fadd_rn(p[g][0][q], pend.v[g][jj]);
    }
    // a resident pass has no per-chunk barrier: every warp must be done reading the tile before the
    // partials are written (sa_kernel keeps them in the tile's first columns)
    if (G.resident || G.NP > 1 || G.eb) __syncthreads();
#pragma unroll
    for (int g = 0; g < GRP && walker; ++g)
#pragma unroll
        for (int m = 0; m < KM; ++m) {
            // the warp's classes of model m: q = j NW + r, r = (warp - m Tm) mod NW
            const int r = KM == 1 ? warp : ((warp - (m * G.Tm) % NW) % NW + NW) % NW;
#pragma unroll
            for (int j = 0; j < NQ; ++j) part[g * pstride + (m * 32 + (r + j * NW)) * 32 + lane] = p[g][m][j];
        }
    __syncthreads();
}

// resident ensembles: wait once for the initial load
__device__ __forceinline__ void ts_wait_resident(const TreeGeo &G, uint64_t *bar)
{
    if (G.resident)
        for (int b = 0; b < G.NC; ++b) mbar_wait(&bar[b], 0);
}

// K bootstrap models scored at once (gbt_predict_acq): per-model canonical sums, then the acquisition
struct AcqArgs {
    int K, kind;
    float kappa, best;
    float base[8];
    float *mean, *std;
};

// Q43, the oracle's sequence of fp32 RN operations (exp = exp_det): EI below `best` of a minimised cost
__device__ __forceinline__ float expected_improvement(float mu, float sd, float best)
{
    const float d = __fsub_rn(best, mu);
    if (!(sd > 0.0f)) return d > 0.0f ? d : 0.0f;
    const float z = __fdiv_rn(d, sd);
    const float x = __fmul_rn(fabsf(z), 0.70710677f);
    const float t = __fdiv_rn(1.0f, __fadd_rn(1.0f, __fmul_rn(0.3275911f, x)));
    float poly = 1.061405429f;
    poly = __fadd_rn(__fmul_rn(poly, t), -1.453152027f);
    poly = __fadd_rn(__fmul_rn(poly, t), 1.421413741f);
    poly = __fadd_rn(__fmul_rn(poly, t), -0.284496736f);
    poly = __fadd_rn(__fmul_rn(poly, t), 0.254829592f);
    poly = __fmul_rn(poly, t);
    const float ec = __fmul_rn(poly, exp_det(-__fmul_rn(x, x)));
    const float Phi = z >= 0.0f ? __fsub_rn(1.0f, __fmul_rn(0.5f, ec)) : __fmul_rn(0.5f, ec);
    const float phi = __fmul_rn(0.3989423f, exp_det(__fmul_rn(__fmul_rn(-0.5f, z), z)));
    return __fadd_rn(__fmul_rn(d, Phi), __fmul_rn(sd, phi));
}

// Q41/Q42: fp64 mean / population std in model order; mean, UCB (mu - kappa sigma) or -EI
__device__ __forceinline__ float acquisition(const AcqArgs &Q, const float *f, int stride, float &mean, float &sd)
{
    double mu = 0.0, v = 0.0;
    for (int k = 0; k < Q.K; ++k) mu = __dadd_rn(mu, (double)f[k * stride]);
    mu = __ddiv_rn(mu, (double)Q.K);
    for (int k = 0; k < Q.K; ++k) {
        const double e = __dsub_rn((double)f[k * stride], mu);
        v = __dadd_rn(v, __dmul_rn(e, e));
    }
    const double s = __dsqrt_rn(__ddiv_rn(v, (double)Q.K));
    mean = (float)mu;
    sd = (float)s;
    if (Q.kind == 1) return (float)__dsub_rn(mu, __dmul_rn((double)Q.kappa, s));
    if (Q.kind == 2) return -expected_improvement(mean, sd, Q.best);
    return mean;
}

// canonical combination of the 32 partials of candidate `lane` (call from one warp)
__device__ __forceinline__ float gbt_combine(const float *part, int lane, float base)
{
    float p[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) p[q] = part[q * 32 + lane];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            if ((q & off) == 0) {
                const float s = __fadd_rn(p[q], p[q | off]);
                p[q] = s;
                p[q | off] = s;
            }
        }
    }
    return __fadd_rn(p[0], base);
}

}  // namespace at
