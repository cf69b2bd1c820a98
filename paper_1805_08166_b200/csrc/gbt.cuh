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
    const uint2 *nodes;     // [T_pad][ni]
    const float *leaf;      // [T_pad][nl]
    int T, T_pad, D, ni, nl;
    int CH;                 // trees per chunk (even: 16-B aligned bulk copies)
    int NC;                 // chunks per pass
    uint32_t chunk_bytes;   // CH * (ni * 8 + nl * 4)
    int resident;           // NC <= 2: loaded once, never re-streamed
};

constexpr uint32_t TREE_BUF_BYTES = 48 * 1024;   // default per buffer (two buffers)
TreeGeo make_geo(const at_gbt_s *g, uint32_t buf_bytes = TREE_BUF_BYTES);

__device__ __forceinline__ void ts_issue(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint64_t c)
{
    const int k = (int)(c % (uint64_t)G.NC);
    const int b = (int)(c & 1);
    const int t0 = k * G.CH;
    const int nt = min(G.CH, G.T_pad - t0);
    const uint32_t nb = (uint32_t)nt * G.ni * 8u, lb = (uint32_t)nt * G.nl * 4u;
    uint8_t *dst = bufs + (size_t)b * G.chunk_bytes;
    mbar_arrive_expect_tx(&bar[b], nb + lb);
    bulk_g2s(dst, G.nodes + (int64_t)t0 * G.ni, nb, &bar[b]);
    bulk_g2s(dst + (size_t)G.CH * G.ni * 8, G.leaf + (int64_t)t0 * G.nl, lb, &bar[b]);
}

// thread 0: initialise both barriers and start the first two chunks of the stream
__device__ __forceinline__ void ts_start(const TreeGeo &G, uint8_t *bufs, uint64_t *bar)
{
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_proxy_async();
        ts_issue(G, bufs, bar, 0);
        if (G.NC > 1) ts_issue(G, bufs, bar, 1);
    }
}

// GRP candidate groups of 32 (group g's tile at tile + g * gstride floats) walk the same trees:
// every tree byte staged in shared memory serves 32 * GRP candidates.
template <int NW, int GRP>
__device__ __forceinline__ void walk_chunk(const TreeGeo &G, const uint8_t *buf, int k, const float *tile, int gstride,
                                           int lane, int warp, float (&p)[GRP][32 / NW], uint8_t *__restrict__ slots,
                                           int64_t slot_ld, int64_t cand0, const bool (&cand_ok)[GRP])
{
    constexpr int NQ = 32 / NW;
    constexpr int R = GRP == 1 ? 2 : 1;  // 32-tree rounds walked together: R * NQ * GRP independent walks
    constexpr int NJ = R * NQ;
    const float *leaves = (const float *)(buf + (size_t)G.CH * G.ni * 8);
    const int c0 = k * G.CH;
    const int c1 = min(c0 + G.CH, G.T);
    const int D = G.D, ni = G.ni, nl = G.nl;
    const uint32_t tree_bytes = (uint32_t)ni * 8u;
    for (int b64 = c0 & ~31; b64 < c1; b64 += 32 * R) {
        const uint8_t *tb[NJ];
        uint32_t off[GRP][NJ];   // byte offset of the current node: node i at 8 i, children at 2 off + 8 / + 16
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int t = b64 + 32 * (jj / NQ) + warp + (jj % NQ) * NW;
            const int lt = (t >= c0 && t < c1) ? t - c0 : 0;   // absent trees walk tree 0, result unused
            tb[jj] = buf + (uint32_t)lt * tree_bytes;
#pragma unroll
            for (int g = 0; g < GRP; ++g) off[g][jj] = 0;
        }
        for (int d = 0; d < D; ++d) {
#pragma unroll
            for (int g = 0; g < GRP; ++g) {
                const uint8_t *tile_lane = (const uint8_t *)(tile + g * gstride + lane);   // feature f at + f * 128
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) {
                    const uint2 nd = *(const uint2 *)(tb[jj] + off[g][jj]);
                    const float x = *(const float *)(tile_lane + (nd.x << 7));
                    off[g][jj] = 2u * off[g][jj] + (x < __uint_as_float(nd.y) ? 8u : 16u);
                }
            }
        }
        // leaves in ascending t within each residue class (round 0 before round 1)
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int t = b64 + 32 * (jj / NQ) + warp + (jj % NQ) * NW;
            if (t >= c0 && t < c1) {
#pragma unroll
                for (int g = 0; g < GRP; ++g) {
                    const int slot = (int)(off[g][jj] >> 3) - ni;
                    p[g][jj % NQ] = __fadd_rn(p[g][jj % NQ], leaves[(t - c0) * nl + slot]);
                    if (slots && cand_ok[g]) slots[(int64_t)t * slot_ld + cand0 + 32 * g] = (uint8_t)slot;
                }
            }
        }
    }
}

// One full pass over the ensemble.  `c` is the block-wide stream counter (identical in every
// thread); `c_limit` the total number of chunks the kernel will consume.  Ends with group g's
// partials in part[g * 1024 + q * 32 + lane] and a __syncthreads.
template <int NW, int GRP>
__device__ __forceinline__ void walk_pass(const TreeGeo &G, uint8_t *bufs, uint64_t *bar, uint32_t *ph, uint64_t &c,
                                          uint64_t c_limit, const float *tile, int gstride, int lane, int warp,
                                          float *part, uint8_t *__restrict__ slots, int64_t slot_ld, int64_t cand0,
                                          const bool (&cand_ok)[GRP])
{
    constexpr int NQ = 32 / NW;
    float p[GRP][NQ];
#pragma unroll
    for (int g = 0; g < GRP; ++g)
#pragma unroll
        for (int j = 0; j < NQ; ++j) p[g][j] = 0.0f;
    if (G.resident) {
        for (int k = 0; k < G.NC; ++k)
            walk_chunk<NW, GRP>(G, bufs + (size_t)k * G.chunk_bytes, k, tile, gstride, lane, warp, p, slots, slot_ld,
                                cand0, cand_ok);
    } else {
        for (int k = 0; k < G.NC; ++k, ++c) {
            const int b = (int)(c & 1);
            mbar_wait(&bar[b], ph[b]);
            ph[b] ^= 1u;
            walk_chunk<NW, GRP>(G, bufs + (size_t)b * G.chunk_bytes, k, tile, gstride, lane, warp, p, slots, slot_ld,
                                cand0, cand_ok);
            __syncthreads();   // every warp is done with buffer b
            if (threadIdx.x == 0 && c + 2 < c_limit) {
                fence_proxy_async();
                ts_issue(G, bufs, bar, c + 2);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < GRP; ++g)
#pragma unroll
        for (int j = 0; j < NQ; ++j) part[g * 1024 + (warp + j * NW) * 32 + lane] = p[g][j];
    __syncthreads();
}

// resident ensembles: wait once for the initial load
__device__ __forceinline__ void ts_wait_resident(const TreeGeo &G, uint64_t *bar)
{
    if (G.resident) {
        mbar_wait(&bar[0], 0);
        if (G.NC > 1) mbar_wait(&bar[1], 0);
    }
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
