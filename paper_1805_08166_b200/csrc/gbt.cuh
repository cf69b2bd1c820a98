// gbt.cuh -- device-side GBT walk + canonical reduction (reading Q19), shared by
// gbt_predict and sa_explore.
//
// Layout: a block owns a tile of 32 candidates (lane = candidate) whose features sit
// in shared memory as tile[f * 32 + lane] (bank = lane for every f: conflict-free
// gathers whatever node each lane is at).  The block's NW warps split the trees by
// residue class: warp w owns q = w, w + NW, ... (q = t mod 32), walks those NQ = 32/NW
// trees of every 32-tree round together (NQ independent walks = ILP) and keeps the
// partial sums p[q] in registers, adding leaves in ascending t exactly as the
// canonical order prescribes.  The 32 partials of a candidate are then combined by
// the xor butterfly (off = 16 ... 1) and base is added.
#pragma once
#include "at_common.cuh"

namespace at {

template <int NW>
__device__ __forceinline__ void gbt_walk_partials(const uint2 *__restrict__ nodes, const float *__restrict__ leaf,
                                                  int T, int D, const float *tile, int lane, int warp,
                                                  float *part /* [32][32] smem */, uint8_t *__restrict__ slots,
                                                  int64_t slot_ld, int64_t cand, bool cand_ok)
{
    constexpr int NQ = 32 / NW;
    const int ni = (1 << D) - 1;
    float p[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) p[j] = 0.0f;
    for (int t0 = 0; t0 < T; t0 += 32) {
        int node[NQ];
        const uint2 *tn[NQ];
        bool ok[NQ];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            const int t = t0 + warp + j * NW;
            ok[j] = t < T;
            tn[j] = nodes + (int64_t)(ok[j] ? t : 0) * ni;
            node[j] = 0;
        }
        for (int d = 0; d < D; ++d) {
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                const uint2 nd = __ldg(tn[j] + node[j]);
                const float x = tile[nd.x * 32 + lane];
                node[j] = 2 * node[j] + 2 - (x < __uint_as_float(nd.y) ? 1 : 0);
            }
        }
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
            if (ok[j]) {
                const int t = t0 + warp + j * NW;
                const int slot = node[j] - ni;
                p[j] = __fadd_rn(p[j], __ldg(leaf + (int64_t)t * (ni + 1) + slot));
                if (slots && cand_ok) slots[(int64_t)t * slot_ld + cand] = (uint8_t)slot;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) part[(warp + j * NW) * 32 + lane] = p[j];
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
