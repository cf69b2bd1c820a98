// features.cuh -- knob decode + closed-form lowering + loop-context / relation features
// for one candidate, as a device function shared by features_extract and sa_explore.
//
// Paper: x = g(e, s); loop context per loop (Appendix table): length,
// one-hot annotation, top-down (product of outer lengths), bottom-up (this loop and
// inner), per buffer touch count ("number of touched elements"), reuse ratio
// (bottom-up / touch), stride (coefficient of the loop variable);
// relation features R_t = max_{k : touch_b(k) < 2^t} Z_k,i.
//
// GPU design (differs from the oracle's literal enumeration): one pass from the
// innermost loop outward keeps the active extent product A_a of every axis; then
//   touch of a dimension indexed by one axis       = A_a
//   touch of a dimension indexed by y*S + ry       = min(A_y A_ry, (A_y - 1) S + A_ry)
// (the active levels of every split chain are a suffix of the nest, so each chain
// covers a contiguous range), the stride of loop k is coef_k x rowstride where
// coef_k = A_axis before loop k is folded in, and the relation max over the
// qualifying loops {k : touch_b(k) < 2^t} -- an inner suffix, because touch only
// grows outward -- is emitted for each t the moment the pass reaches the first loop
// whose touch reaches 2^t.  All integers are u32 (space_create guarantees no overflow);
// the float conversions and the reuse division are single IEEE RN operations.
#pragma once
#include "at_common.cuh"

namespace at {

// lexicographic permutations of 3 items: item at slot q of permutation p
// (0,1,2) (0,2,1) (1,0,2) (1,2,0) (2,0,1) (2,1,0), packed 2 bits per slot
__host__ __device__ __forceinline__ uint32_t perm3(uint32_t p, uint32_t q)
{
    const uint32_t t = (p == 0) ? 0x24u : (p == 1) ? 0x18u : (p == 2) ? 0x21u : (p == 3) ? 0x09u : (p == 4) ? 0x12u : 0x06u;
    return (t >> (2 * q)) & 3u;
}

template <int TMPL> struct Tmpl;
template <> struct Tmpl<0> { static constexpr int NK = 4, NL = 8, NA = 3; };
template <> struct Tmpl<1> { static constexpr int NK = 9, NL = 18, NA = 6; };
template <> struct Tmpl<2> { static constexpr int NK = 8, NL = 16, NA = 5; };

__device__ __forceinline__ uint32_t comp_touch(uint32_t Y, uint32_t R, uint32_t S)
{
    uint32_t a = Y * R, b = (Y - 1u) * S + R;
    return a < b ? a : b;
}

// decode local flat index (knob 0 fastest)
template <int TMPL>
__device__ __forceinline__ void decode_knobs(const WlDev &W, uint32_t local, uint32_t *ch)
{
#pragma unroll
    for (int j = 0; j < Tmpl<TMPL>::NK; ++j) {
        uint32_t r = W.radix[j];
        uint32_t q = local / r;
        ch[j] = local - q * r;
        local = q;
    }
}

// Compute the 468 features of the loop nest given by knob choices `ch`.
// Sink: put(int f, float v) / put_rel(int f, float v).
// Work split (part, nparts): nparts == 1 computes everything; otherwise part b < 3 owns the
// relation features (and footprint) of buffer b, and the loop rows are dealt round-robin to
// parts 3 .. nparts-1 (to parts 0 .. nparts-1 when nparts < 4).  The cheap running products
// are recomputed by every part; the expensive per-row work and the stores are not.
__host__ __device__ __forceinline__ int row_owner(int k, int nparts)
{
    return nparts >= 4 ? 3 + k % (nparts - 3) : k % nparts;
}

template <int TMPL, class Sink>
__device__ __forceinline__ void features_one(const WlDev &W, const uint16_t *__restrict__ fact,
                                             const uint32_t *ch, Sink &sk, int part = 0, int nparts = 1,
                                             bool rows_only = false)
{
    constexpr int NL = Tmpl<TMPL>::NL;
    constexpr int NA = Tmpl<TMPL>::NA;
    uint32_t ext[NL];
    int axis_[NL];
    int level_[NL];
    uint32_t unroll_max, vec;
    // ---- lowering (DESIGN Q3 templates): loop extents, axes, levels of the nest, outer -> inner
    if (TMPL == 0) {
        // i0 j0 k0 i1 j1 k1 i2 j2
        uint32_t Fi[3], Fj[3], Fk[2];
        const uint16_t *ti = fact + W.fact_off[0] + ch[0] * 3;
        const uint16_t *tj = fact + W.fact_off[1] + ch[1] * 3;
        const uint16_t *tk = fact + W.fact_off[2] + ch[2] * 2;
#pragma unroll
        for (int l = 0; l < 3; ++l) { Fi[l] = __ldg(ti + l); Fj[l] = __ldg(tj + l); }
        Fk[0] = __ldg(tk); Fk[1] = __ldg(tk + 1);
        const int ax[8] = {0, 1, 2, 0, 1, 2, 0, 1};
        const int lv[8] = {0, 0, 0, 1, 1, 1, 2, 2};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            axis_[k] = ax[k];
            level_[k] = lv[k];
            ext[k] = ax[k] == 0 ? Fi[lv[k]] : ax[k] == 1 ? Fj[lv[k]] : Fk[lv[k]];
        }
        unroll_max = W.unroll_vals[ch[3]];
        vec = 0;
    } else {
        constexpr int NSPLIT = (TMPL == 1) ? 6 : 5;
        uint32_t F[NSPLIT][4];
#pragma unroll
        for (int a = 0; a < NSPLIT; ++a) {
            const int L = (a < 3) ? 4 : 2;
            const uint16_t *t = fact + W.fact_off[a] + ch[a] * L;
#pragma unroll
            for (int l = 0; l < 4; ++l) F[a][l] = (l < L) ? (uint32_t)__ldg(t + l) : 1u;
        }
        const uint32_t p = ch[NSPLIT];
        unroll_max = W.unroll_vals[ch[NSPLIT + 1]];
        vec = ch[NSPLIT + 2];
#pragma unroll
        for (int k = 0; k < 9; ++k) { axis_[k] = k % 3; level_[k] = k / 3; }
        if (TMPL == 1) {
            // f0 y0 x0 f1 y1 x1 f2 y2 x2 | perm(rc0 ry0 rx0) | rc1 ry1 rx1 | f3 y3 x3
#pragma unroll
            for (int q = 0; q < 3; ++q) { axis_[9 + q] = 3 + (int)perm3(p, q); level_[9 + q] = 0; }
#pragma unroll
            for (int q = 0; q < 3; ++q) { axis_[12 + q] = 3 + q; level_[12 + q] = 1; }
#pragma unroll
            for (int q = 0; q < 3; ++q) { axis_[15 + q] = q; level_[15 + q] = 3; }
        } else {
            // c0 y0 x0 c1 y1 x1 c2 y2 x2 | ry0 rx0 ry1 rx1 | perm(c3 y3 x3)
            axis_[9] = 3; level_[9] = 0; axis_[10] = 4; level_[10] = 0;
            axis_[11] = 3; level_[11] = 1; axis_[12] = 4; level_[12] = 1;
#pragma unroll
            for (int q = 0; q < 3; ++q) { axis_[13 + q] = (int)perm3(p, q); level_[13 + q] = 3; }
        }
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            uint32_t e = 1;
#pragma unroll
            for (int a = 0; a < NSPLIT; ++a)
#pragma unroll
                for (int l = 0; l < 4; ++l)
                    if (axis_[k] == a && level_[k] == l) e = F[a][l];
            ext[k] = e;
        }
    }

    // ---- top-down prefix products
    uint32_t td[NL];
    td[0] = 1;
#pragma unroll
    for (int k = 1; k < NL; ++k) td[k] = td[k - 1] * ext[k - 1];

    // ---- inner -> outer pass
    uint32_t A[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) A[a] = 1;
    uint32_t bu = 1;
    float smax_r[3], smax_t[3];
    int tnext[3];
    bool has[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) { smax_r[b] = 0.f; smax_t[b] = 0.f; tnext[b] = 1; has[b] = false; }
    const uint32_t S = W.S;

#pragma unroll
    for (int k = NL - 1; k >= 0; --k) {
        const int a = axis_[k];
        uint32_t coef = 1;
#pragma unroll
        for (int q = 0; q < NA; ++q) if (a == q) coef = A[q];
#pragma unroll
        for (int q = 0; q < NA; ++q) if (a == q) A[q] *= ext[k];
        bu *= ext[k];
        const bool own_row = nparts == 1 || part == (rows_only ? k % nparts : row_owner(k, nparts));
        bool own_rel[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) own_rel[b] = !rows_only && (nparts == 1 || part == b % nparts);
        if (!own_row && !own_rel[0] && !own_rel[1] && !own_rel[2]) continue;
        uint32_t T[3];
        uint32_t st[3];
        if (TMPL == 0) {
            T[0] = A[0] * A[1];                // C[i][j]
            T[1] = A[2] * A[0];                // A[k][i]
            T[2] = A[2] * A[1];                // B[k][j]
            st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : 0u;
            st[1] = (a == 2) ? coef * W.str_in[0] : (a == 0) ? coef * W.str_in[1] : 0u;
            st[2] = (a == 2) ? coef * W.str_ker[0] : (a == 1) ? coef * W.str_ker[1] : 0u;
        } else if (TMPL == 1) {
            T[0] = A[0] * A[1] * A[2];                                             // Out[f][y][x]
            T[1] = A[3] * comp_touch(A[1], A[4], S) * comp_touch(A[2], A[5], S);   // Data[rc][yS+ry][xS+rx]
            T[2] = A[0] * A[3] * A[4] * A[5];                                      // Ker[f][rc][ry][rx]
            st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
            st[1] = (a == 3) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 4) ? coef * W.str_in[1]
                  : (a == 2) ? coef * S * W.str_in[2] : (a == 5) ? coef * W.str_in[2] : 0u;
            st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2]
                  : (a == 5) ? coef * W.str_ker[3] : 0u;
        } else {
            T[0] = A[0] * A[1] * A[2];                                             // Out[c][y][x]
            T[1] = A[0] * comp_touch(A[1], A[3], S) * comp_touch(A[2], A[4], S);   // Data[c][yS+ry][xS+rx]
            T[2] = A[0] * A[3] * A[4];                                             // Ker[c][ry][rx]
            st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
            st[1] = (a == 0) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 3) ? coef * W.str_in[1]
                  : (a == 2) ? coef * S * W.str_in[2] : (a == 4) ? coef * W.str_in[2] : 0u;
            st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2] : 0u;
        }
        // annotation: 0 serial 1 unroll 2 vectorize 3 parallel 4 blockIdx 5 vthread 6 threadIdx
        int ann;
        if (TMPL != 0 && k < 9) {
            ann = 4 + level_[k];
        } else {
            ann = (bu <= unroll_max) ? 1 : 0;
            if (k == NL - 1 && vec) ann = 2;
        }
        const float fbu = __uint2float_rn(bu);
        float reuse[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) reuse[b] = __fdiv_rn(fbu, __uint2float_rn(T[b]));
        const float ftd = __uint2float_rn(td[k]);
        // relation emission (before loop k joins the qualifying suffix)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            if (!own_rel[b]) continue;
            while (tnext[b] <= 20 && (T[b] >> tnext[b]) != 0u) {
                sk.put_rel(342 + 40 * b + tnext[b] - 1, has[b] ? smax_r[b] : 0.f);
                sk.put_rel(362 + 40 * b + tnext[b] - 1, has[b] ? smax_t[b] : 0.f);
                ++tnext[b];
            }
            smax_r[b] = has[b] ? fmaxf(smax_r[b], reuse[b]) : reuse[b];
            smax_t[b] = has[b] ? fmaxf(smax_t[b], ftd) : ftd;
            has[b] = true;
        }
        if (!own_row) continue;
        // the 19 context columns of row k
        const int base = 19 * k;
        sk.put(base + 0, __uint2float_rn(ext[k]));
#pragma unroll
        for (int q = 0; q < 7; ++q) sk.put(base + 1 + q, ann == q ? 1.0f : 0.0f);
        sk.put(base + 8, ftd);
        sk.put(base + 9, fbu);
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            sk.put(base + 10 + 3 * b, __uint2float_rn(T[b]));
            sk.put(base + 11 + 3 * b, reuse[b]);
            sk.put(base + 12 + 3 * b, __uint2float_rn(st[b]));
        }
        if (k == 0) {
            // scalars: total iterations and footprints touch(b, 0)
            sk.put(462, fbu);
#pragma unroll
            for (int b = 0; b < 3; ++b) sk.put(463 + b, __uint2float_rn(T[b]));
        }
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        if (rows_only || !(nparts == 1 || part == b % nparts)) continue;
        while (tnext[b] <= 20) {
            sk.put_rel(342 + 40 * b + tnext[b] - 1, smax_r[b]);
            sk.put_rel(362 + 40 * b + tnext[b] - 1, smax_t[b]);
            ++tnext[b];
        }
    }
}

// ------------------------------------------------------------------------------------------
// Block-cooperative variant used by sa_kernel (32 chains per block, lane = chain): the work of
// one candidate is spread over the block's warps in three phases separated by barriers:
//   L) loop extents: warp w lowers loops k = w, w + NW, ... for all 32 chains (one factor load
//      each) into shared arrays ext[k][lane], axis[k][lane];
//   R) context rows: warp w owns rows k = w (mod NW) and rebuilds that row's active products
//      from the shared extents (inner loops' extents, top-down prefix) -- the same integer
//      formulas as features_one;
//   T) relation features from the finished rows (relation_from_tile).
struct SaLowering {
    uint32_t ext[MAXLOOPS][32];
    uint8_t axis[MAXLOOPS][32];
    uint32_t unroll_max[32];
    uint8_t vec[32];
};

// (axis, level) of loop k of template TMPL with reorder knob p (DESIGN Q3 nest orders)
template <int TMPL>
__device__ __forceinline__ void loop_axis_level(int k, uint32_t p, int &axis, int &level)
{
    if (TMPL == 0) {
        axis = k % 3;                         // i0 j0 k0 i1 j1 k1 i2 j2
        level = k / 3;
    } else if (k < 9) {
        axis = k % 3;                         // spatial levels 0..2
        level = k / 3;
    } else if (TMPL == 1) {
        if (k < 12) { axis = 3 + (int)perm3(p, k - 9); level = 0; }   // perm(rc0 ry0 rx0)
        else if (k < 15) { axis = 3 + (k - 12); level = 1; }          // rc1 ry1 rx1
        else { axis = k - 15; level = 3; }                            // f3 y3 x3
    } else {
        if (k < 13) { axis = 3 + ((k - 9) & 1); level = (k - 9) >> 1; }   // ry0 rx0 ry1 rx1
        else { axis = (int)perm3(p, k - 13); level = 3; }                  // perm(c3 y3 x3)
    }
}

template <int TMPL>
__device__ __forceinline__ void sa_lower_loop(const WlDev &W, const uint16_t *__restrict__ fact, const uint32_t *ch,
                                              int k, int lane, SaLowering &L)
{
    constexpr int NL = Tmpl<TMPL>::NL;
    if (k >= NL) return;
    const uint32_t p = TMPL == 1 ? ch[6] : TMPL == 2 ? ch[5] : 0u;
    int axis, level;
    loop_axis_level<TMPL>(k, p, axis, level);
    const int Lv = TMPL == 0 ? (axis == 2 ? 2 : 3) : (axis < 3 ? 4 : 2);
    uint32_t cha = 0;
#pragma unroll
    for (int q = 0; q < 6; ++q) if (q == axis) cha = ch[q];
    L.ext[k][lane] = __ldg(fact + W.fact_off[axis] + cha * (uint32_t)Lv + level);
    L.axis[k][lane] = (uint8_t)axis;
    if (k == 0) {
        L.unroll_max[lane] = W.unroll_vals[TMPL == 0 ? ch[3] : TMPL == 1 ? ch[7] : ch[6]];
        L.vec[lane] = (uint8_t)(TMPL == 0 ? 0u : TMPL == 1 ? ch[8] : ch[7]);
    }
}

template <int TMPL, class Sink>
__device__ __forceinline__ void sa_row(const WlDev &W, const SaLowering &L, int k, int lane, uint32_t p, Sink &sk)
{
    constexpr int NL = Tmpl<TMPL>::NL;
    constexpr int NA = Tmpl<TMPL>::NA;
    if (k >= NL) return;
    // all extents of this chain at once (independent loads), then predicated products:
    // A_a and bottom-up over the loops inside k, top-down over the loops outside k
    // The axis of loop l is a compile-time constant except for the three reordered loops
    // (T_CONV 9..11 over {3,4,5}, T_DW 13..15 over {0,1,2}), whose axis perm3 of knob p picks.
    uint32_t ev[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) ev[l] = L.ext[l][lane];
    uint32_t A[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) A[q] = 1;
    uint32_t bu = 1, td = 1;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        const uint32_t m = l > k ? ev[l] : 1u;
        if (TMPL == 1 && l >= 9 && l < 12) {
            const uint32_t al = perm3(p, l - 9);
#pragma unroll
            for (int q = 0; q < 3; ++q) A[3 + q] = al == (uint32_t)q ? A[3 + q] * m : A[3 + q];
        } else if (TMPL == 2 && l >= 13 && l < 16) {
            const uint32_t al = perm3(p, l - 13);
#pragma unroll
            for (int q = 0; q < 3; ++q) A[q] = al == (uint32_t)q ? A[q] * m : A[q];
        } else {
            int al, lv;
            loop_axis_level<TMPL>(l, p, al, lv);
            A[al] *= m;
        }
        bu *= m;
        td = l < k ? td * ev[l] : td;
    }
    uint32_t ek = 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) if (l == k) ek = ev[l];
    int a, level;
    loop_axis_level<TMPL>(k, p, a, level);
    uint32_t coef = 1;
#pragma unroll
    for (int q = 0; q < NA; ++q) if (a == q) coef = A[q];
#pragma unroll
    for (int q = 0; q < NA; ++q) if (a == q) A[q] *= ek;
    bu *= ek;
    const uint32_t S = W.S;
    uint32_t T[3], st[3];
    if (TMPL == 0) {
        T[0] = A[0] * A[1];
        T[1] = A[2] * A[0];
        T[2] = A[2] * A[1];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : 0u;
        st[1] = (a == 2) ? coef * W.str_in[0] : (a == 0) ? coef * W.str_in[1] : 0u;
        st[2] = (a == 2) ? coef * W.str_ker[0] : (a == 1) ? coef * W.str_ker[1] : 0u;
    } else if (TMPL == 1) {
        T[0] = A[0] * A[1] * A[2];
        T[1] = A[3] * comp_touch(A[1], A[4], S) * comp_touch(A[2], A[5], S);
        T[2] = A[0] * A[3] * A[4] * A[5];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
        st[1] = (a == 3) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 4) ? coef * W.str_in[1]
              : (a == 2) ? coef * S * W.str_in[2] : (a == 5) ? coef * W.str_in[2] : 0u;
        st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2]
              : (a == 5) ? coef * W.str_ker[3] : 0u;
    } else {
        T[0] = A[0] * A[1] * A[2];
        T[1] = A[0] * comp_touch(A[1], A[3], S) * comp_touch(A[2], A[4], S);
        T[2] = A[0] * A[3] * A[4];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
        st[1] = (a == 0) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 3) ? coef * W.str_in[1]
              : (a == 2) ? coef * S * W.str_in[2] : (a == 4) ? coef * W.str_in[2] : 0u;
        st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2] : 0u;
    }
    int ann;
    if (TMPL != 0 && k < 9) {
        ann = 4 + level;
    } else {
        ann = (bu <= L.unroll_max[lane]) ? 1 : 0;
        if (k == NL - 1 && L.vec[lane]) ann = 2;
    }
    const float fbu = __uint2float_rn(bu);
    const int base = 19 * k;
    sk.put(base + 0, __uint2float_rn(ek));
#pragma unroll
    for (int q = 0; q < 7; ++q) sk.put(base + 1 + q, ann == q ? 1.0f : 0.0f);
    sk.put(base + 8, __uint2float_rn(td));
    sk.put(base + 9, fbu);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        sk.put(base + 10 + 3 * b, __uint2float_rn(T[b]));
        sk.put(base + 11 + 3 * b, __fdiv_rn(fbu, __uint2float_rn(T[b])));
        sk.put(base + 12 + 3 * b, __uint2float_rn(st[b]));
    }
    if (k == 0) {
        sk.put(462, fbu);
#pragma unroll
        for (int b = 0; b < 3; ++b) sk.put(463 + b, __uint2float_rn(T[b]));
    }
}

// sa_kernel's fused row item: the extents of every loop (kept in shared memory by the owner warp,
// sa_extents, after each move), then row k exactly as sa_row, and the
// row's relation contributions deposited at once: row k qualifies for threshold 2^t iff
// T_k < 2^t, i.e. iff t >= bitlen(T_k), so it raises slot max(1, bitlen(T_k)) of R[b][p] to its
// Z (shared atomic max on the fp32 bits: every Z is > 0, and the slots start at +0); a prefix
// max over t (relation_prefix) then gives R_t = max_{k : T_k < 2^t} Z_k, 0 for an empty set.
// the extents of every loop of template TMPL for knob vector ch (one factor-table load per loop)
template <int TMPL>
__device__ __forceinline__ void sa_extents(const uint32_t (&foff)[6], const uint16_t *__restrict__ fact,
                                           const uint32_t *ch, uint16_t *ext /* [MAXLOOPS][32] at the lane */)
{
    constexpr int NL = Tmpl<TMPL>::NL;
    const uint32_t p = TMPL == 1 ? ch[6] : TMPL == 2 ? ch[5] : 0u;
    uint32_t ev[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        int axis, level;
        loop_axis_level<TMPL>(l, p, axis, level);
        const int Lv = TMPL == 0 ? (axis == 2 ? 2 : 3) : (axis < 3 ? 4 : 2);
        uint32_t cha = 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) if (q == axis) cha = ch[q];
        uint32_t fo = 0;   // the split table of this axis (register copy: no dependent global load)
#pragma unroll
        for (int q = 0; q < 6; ++q) if (q == axis) fo = foff[q];
        ev[l] = __ldg(fact + fo + cha * (uint32_t)Lv + level);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) ext[l * 32] = (uint16_t)ev[l];   // factors are u16 (space tables)
}

template <int TMPL>
__device__ __forceinline__ void sa_row_rel(const WlDev &W, const uint16_t *ext /* [l * 32] at the lane */,
                                           const uint32_t *ch, int k, int lane, float *tile)
{
    constexpr int NL = Tmpl<TMPL>::NL;
    constexpr int NA = Tmpl<TMPL>::NA;
    if (k >= NL) return;
    const uint32_t p = TMPL == 1 ? ch[6] : TMPL == 2 ? ch[5] : 0u;
    uint32_t ev[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) ev[l] = ext[l * 32];
    const uint32_t unroll_max = W.unroll_vals[TMPL == 0 ? ch[3] : TMPL == 1 ? ch[7] : ch[6]];
    const uint32_t vec = TMPL == 0 ? 0u : TMPL == 1 ? ch[8] : ch[7];
    uint32_t A[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) A[q] = 1;
    uint32_t bu = 1, td = 1;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        const uint32_t m = l > k ? ev[l] : 1u;
        if (TMPL == 1 && l >= 9 && l < 12) {
            const uint32_t al = perm3(p, l - 9);
#pragma unroll
            for (int q = 0; q < 3; ++q) A[3 + q] = al == (uint32_t)q ? A[3 + q] * m : A[3 + q];
        } else if (TMPL == 2 && l >= 13 && l < 16) {
            const uint32_t al = perm3(p, l - 13);
#pragma unroll
            for (int q = 0; q < 3; ++q) A[q] = al == (uint32_t)q ? A[q] * m : A[q];
        } else {
            int al, lv;
            loop_axis_level<TMPL>(l, p, al, lv);
            A[al] *= m;
        }
        bu *= m;
        td = l < k ? td * ev[l] : td;
    }
    uint32_t ek = 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) if (l == k) ek = ev[l];
    int a, level;
    loop_axis_level<TMPL>(k, p, a, level);
    uint32_t coef = 1;
#pragma unroll
    for (int q = 0; q < NA; ++q) if (a == q) coef = A[q];
#pragma unroll
    for (int q = 0; q < NA; ++q) if (a == q) A[q] *= ek;
    bu *= ek;
    const uint32_t S = W.S;
    uint32_t T[3], st[3];
    if (TMPL == 0) {
        T[0] = A[0] * A[1];
        T[1] = A[2] * A[0];
        T[2] = A[2] * A[1];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : 0u;
        st[1] = (a == 2) ? coef * W.str_in[0] : (a == 0) ? coef * W.str_in[1] : 0u;
        st[2] = (a == 2) ? coef * W.str_ker[0] : (a == 1) ? coef * W.str_ker[1] : 0u;
    } else if (TMPL == 1) {
        T[0] = A[0] * A[1] * A[2];
        T[1] = A[3] * comp_touch(A[1], A[4], S) * comp_touch(A[2], A[5], S);
        T[2] = A[0] * A[3] * A[4] * A[5];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
        st[1] = (a == 3) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 4) ? coef * W.str_in[1]
              : (a == 2) ? coef * S * W.str_in[2] : (a == 5) ? coef * W.str_in[2] : 0u;
        st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2]
              : (a == 5) ? coef * W.str_ker[3] : 0u;
    } else {
        T[0] = A[0] * A[1] * A[2];
        T[1] = A[0] * comp_touch(A[1], A[3], S) * comp_touch(A[2], A[4], S);
        T[2] = A[0] * A[3] * A[4];
        st[0] = (a == 0) ? coef * W.str_out[0] : (a == 1) ? coef * W.str_out[1] : (a == 2) ? coef * W.str_out[2] : 0u;
        st[1] = (a == 0) ? coef * W.str_in[0] : (a == 1) ? coef * S * W.str_in[1] : (a == 3) ? coef * W.str_in[1]
              : (a == 2) ? coef * S * W.str_in[2] : (a == 4) ? coef * W.str_in[2] : 0u;
        st[2] = (a == 0) ? coef * W.str_ker[0] : (a == 3) ? coef * W.str_ker[1] : (a == 4) ? coef * W.str_ker[2] : 0u;
    }
    int ann;
    if (TMPL != 0 && k < 9) {
        ann = 4 + level;
    } else {
        ann = (bu <= unroll_max) ? 1 : 0;
        if (k == NL - 1 && vec) ann = 2;
    }
    float *col = tile + lane;   // feature f at col[f * 32]
    const float fbu = __uint2float_rn(bu), ftd = __uint2float_rn(td);
    const int base = 19 * k;
    col[(base + 0) * 32] = __uint2float_rn(ek);
#pragma unroll
    for (int q = 0; q < 7; ++q) col[(base + 1 + q) * 32] = ann == q ? 1.0f : 0.0f;
    col[(base + 8) * 32] = ftd;
    col[(base + 9) * 32] = fbu;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const float reuse = __fdiv_rn(fbu, __uint2float_rn(T[b]));
        col[(base + 10 + 3 * b) * 32] = __uint2float_rn(T[b]);
        col[(base + 11 + 3 * b) * 32] = reuse;
        col[(base + 12 + 3 * b) * 32] = __uint2float_rn(st[b]);
        const int e = 32 - __clz((int)T[b]);   // bitlen(T) >= 1
        if (e <= 20) {
            unsigned *R = (unsigned *)(col + (342 + 40 * b + (e - 1)) * 32);
            atomicMax(R, __float_as_uint(reuse));
            atomicMax(R + 20 * 32, __float_as_uint(ftd));
        }
    }
    if (k == 0) {
        col[462 * 32] = fbu;
#pragma unroll
        for (int b = 0; b < 3; ++b) col[(463 + b) * 32] = __uint2float_rn(T[b]);
    }
}

// prefix max over t of the deposited relation slots R[b][p][t] (sa_row_rel)
__device__ __forceinline__ void relation_prefix(float *tile, int lane, int b, int p)
{
    float *R = tile + (342 + 40 * b + 20 * p) * 32 + lane;
    float m = 0.0f;
#pragma unroll
    for (int t = 0; t < 20; ++t) {
        m = fmaxf(m, R[t * 32]);
        R[t * 32] = m;
    }
}

// Relation features of buffer b, pair p (0: reuse, 1: top-down) from context rows already in a
// smem tile [f][32] (rows-only pass).  Row k qualifies for threshold 2^t iff T_k < 2^t, i.e. iff
// t >= bitlen(T_k) (T_k >= 1), so R_t = max(0, max_{k : bitlen(T_k) <= t} Z_k): each row deposits
// its Z at slot max(1, bitlen(T_k)) (a per-lane max in the output rows themselves), then a prefix
// max over t finishes.  bitlen is read from the exponent of the fp32 touch value: exact for
// T < 2^24, and any larger T has bitlen > 20 either way.  Every Z is > 0 (reuse > 0, top-down
// >= 1), so the empty-set value 0 is the max's identity.
__device__ __forceinline__ void relation_from_tile(float *tile, int lane, int NL, int b, int p)
{
    const int colT = 10 + 3 * b, colZ = p == 0 ? 11 + 3 * b : 8;
    float *R = tile + (342 + 40 * b + 20 * p) * 32 + lane;   // R[(t - 1) * 32], t = 1..20
#pragma unroll
    for (int t = 0; t < 20; ++t) R[t * 32] = 0.0f;
    for (int k = 0; k < NL; ++k) {
        const float T = tile[(19 * k + colT) * 32 + lane];
        const float z = tile[(19 * k + colZ) * 32 + lane];
        const int e = (int)((__float_as_uint(T) >> 23) & 0xFF) - 126;   // bitlen(T) for T >= 1
        if (e <= 20) {
            float *slot = R + (e < 1 ? 0 : e - 1) * 32;
            *slot = fmaxf(*slot, z);
        }
    }
    float m = 0.0f;
#pragma unroll
    for (int t = 0; t < 20; ++t) {
        m = fmaxf(m, R[t * 32]);
        R[t * 32] = m;
    }
}

// columns that are zero for every candidate of a template (absent loop rows + padding)
template <int TMPL, class Sink>
__device__ __forceinline__ void features_zero_cols(Sink &sk)
{
    constexpr int NL = Tmpl<TMPL>::NL;
#pragma unroll 4
    for (int f = 19 * NL; f < 342; ++f) sk.put(f, 0.0f);
    sk.put(466, 0.0f);
    sk.put(467, 0.0f);
}

}  // namespace at
