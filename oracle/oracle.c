/*
 * oracle.c -- plain, slow CPU oracle for the AutoTVM hot path (arXiv 1805.08166).
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -ffp-contract=off -fno-fast-math -o liboracle.so oracle.c -lm
 * (no FMA contraction, no flush-to-zero: every fp32 / fp64 operation is one IEEE RN op,
 * written in the order DESIGN.md fixes.)
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { TAG_SA_INIT = 0, TAG_SA_STEP = 1, TAG_EPS = 2, TAG_GROUP_PERM = 3, TAG_BOOT = 6 };

static float f_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }

/* ======================================================================
 * RNG: Philox4x32-10 (Salmon et al. 2011, Random123), Q28.  Counter
 * (id, step_or_attempt, round, tag), key (seed_lo, seed_hi).
 * ==================================================================== */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox(uint64_t seed, uint32_t id, uint32_t step, uint32_t round, uint32_t tag, uint32_t out[4])
{
    uint32_t ctr[4] = { id, step, round, tag };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    or_philox4x32_10(ctr, key, out);
}

/* floor(a * b / 2^64): uniform draw of a u64 onto [0, b) (Q28) */
uint64_t or_mulhi64(uint64_t a, uint64_t b)
{
    unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
    return (uint64_t)(p >> 64);
}

/* ======================================================================
 * exp_det (Q22): the one transcendental both sides must agree on bit for
 * bit (Metropolis acceptance; rank-loss sigmoid, Eq. 2).
 * All ops are single fp32 RN operations; fmaf is the correctly rounded fma.
 * ==================================================================== */
float or_exp_det(float a)
{
    if (a < -87.0f) return 0.0f;
    if (a > 88.0f) return INFINITY;
    const float log2e = f_from_bits(0x3FB8AA3Bu);
    const float ln2_hi = f_from_bits(0x3F317200u);
    const float ln2_lo = f_from_bits(0x35BFBE8Eu);
    float t = a * log2e;
    float n = rintf(t);                       /* round half to even */
    float r = fmaf(-n, ln2_hi, a);
    r = fmaf(-n, ln2_lo, r);
    float p = f_from_bits(0x39500D01u);       /* 1/5040 */
    p = fmaf(p, r, f_from_bits(0x3AB60B61u)); /* 1/720 */
    p = fmaf(p, r, f_from_bits(0x3C088889u)); /* 1/120 */
    p = fmaf(p, r, f_from_bits(0x3D2AAAABu)); /* 1/24 */
    p = fmaf(p, r, f_from_bits(0x3E2AAAABu)); /* 1/6 */
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    int e = (int)n;                           /* e in [-126, 127] on the domain above */
    float scale = f_from_bits((uint32_t)(e + 127) << 23);
    return p * scale;
}

/* exp_det of the fp32 values whose bits are first_bits, first_bits + 1, ... (u32 wrap), n of them */
void or_exp_det_range(uint32_t first_bits, int64_t n, float *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = or_exp_det(f_from_bits(first_bits + (uint32_t)i));
}

/* ======================================================================
 * Schedule space S_e ("multi-level tiling on each loop axis, loop
 * ordering ... unrolling and vectorization"; templates Q3, knob order O2).
 * ==================================================================== */

/* all ordered L-tuples of positive integers with product n, lexicographically
 * ascending (outermost factor first), by nested ascending-divisor loops. */
static void fact_rec(int64_t n, int L, int depth, int *cur, int *out, int *cnt)
{
    if (depth == L - 1) {
        cur[depth] = (int)n;
        if (out) memcpy(out + (size_t)(*cnt) * L, cur, sizeof(int) * L);
        (*cnt)++;
        return;
    }
    for (int64_t d = 1; d <= n; ++d) {
        if (n % d == 0) {
            cur[depth] = (int)d;
            fact_rec(n / d, L, depth + 1, cur, out, cnt);
        }
    }
}

uint64_t or_count_factorizations(int64_t n, int L)
{
    int cur[8];
    int cnt = 0;
    fact_rec(n, L, 0, cur, NULL, &cnt);
    return (uint64_t)cnt;
}

static int add_split(or_space *sp, int axis)
{
    int j = sp->n_knobs++;
    int L = sp->axis_levels[axis];
    int cur[8], cnt = 0;
    fact_rec(sp->axis_ext[axis], L, 0, cur, NULL, &cnt);
    sp->fact[j] = (int *)malloc(sizeof(int) * (size_t)cnt * L);
    if (!sp->fact[j]) return -1;
    int c2 = 0;
    fact_rec(sp->axis_ext[axis], L, 0, cur, sp->fact[j], &c2);
    sp->knob_kind[j] = 0;
    sp->knob_axis[j] = axis;
    sp->radix[j] = cnt;
    return 0;
}

static void add_simple(or_space *sp, int kind, int radix)
{
    int j = sp->n_knobs++;
    sp->knob_kind[j] = kind;
    sp->knob_axis[j] = -1;
    sp->radix[j] = radix;
    sp->fact[j] = NULL;
}

static void set_dim1(or_space *sp, int b, int d, int64_t shape, int axis)
{
    sp->shape[b][d] = shape;
    sp->n_terms[b][d] = 1;
    sp->term_axis[b][d][0] = axis;
    sp->term_mult[b][d][0] = 1;
}

static void set_dim2(or_space *sp, int b, int d, int64_t shape, int axis0, int64_t mult0, int axis1)
{
    sp->shape[b][d] = shape;
    sp->n_terms[b][d] = 2;
    sp->term_axis[b][d][0] = axis0;
    sp->term_mult[b][d][0] = mult0;
    sp->term_axis[b][d][1] = axis1;
    sp->term_mult[b][d][1] = 1;
}

static int space_create1(const or_workload *w, or_space *sp)
{
    memset(sp, 0, sizeof(*sp));
    sp->wl = *w;
    if (w->kind == 0) {
        /* T_MM: C[i][j] = sum_k A[k][i] B[k][j] (Q1); axes i, j (3 levels), k (2 levels) */
        if (w->n < 1 || w->m < 1 || w->k < 1) return -1;
        sp->tmpl = 0;
        sp->n_axes = 3;
        sp->axis_ext[0] = w->n; sp->axis_levels[0] = 3;
        sp->axis_ext[1] = w->m; sp->axis_levels[1] = 3;
        sp->axis_ext[2] = w->k; sp->axis_levels[2] = 2;
        if (add_split(sp, 0) || add_split(sp, 1) || add_split(sp, 2)) return -1;
        add_simple(sp, 2, 5);
        int uv[5] = { 1, 2, 4, 8, 16 };
        memcpy(sp->unroll_vals, uv, sizeof uv);
        /* b0 = C[n][m], b1 = A[k][n], b2 = B[k][m] */
        sp->n_dims[0] = 2; set_dim1(sp, 0, 0, w->n, 0); set_dim1(sp, 0, 1, w->m, 1);
        sp->n_dims[1] = 2; set_dim1(sp, 1, 0, w->k, 2); set_dim1(sp, 1, 1, w->n, 0);
        sp->n_dims[2] = 2; set_dim1(sp, 2, 0, w->k, 2); set_dim1(sp, 2, 1, w->m, 1);
    } else if (w->kind == 1 || w->kind == 2) {
        if (w->h < 1 || w->w < 1 || w->ic < 1 || w->ksize < 1 || w->stride < 1 || w->pad < 0) return -1;
        if (w->kind == 1 && w->oc < 1) return -1;
        int64_t hp = (int64_t)w->h + 2 * w->pad, wp = (int64_t)w->w + 2 * w->pad;
        if (hp < w->ksize || wp < w->ksize) return -1;
        int64_t oh = (hp - w->ksize) / w->stride + 1;
        int64_t ow = (wp - w->ksize) / w->stride + 1;
        int64_t S = w->stride, K = w->ksize;
        int uv[5] = { 0, 512, 1500, 0, 0 };
        memcpy(sp->unroll_vals, uv, sizeof uv);
        if (w->kind == 1) {
            /* T_CONV: Out[f][y][x] = sum Data[rc][y*S+ry][x*S+rx] * Ker[f][rc][ry][rx] (O1) */
            sp->tmpl = 1;
            sp->n_axes = 6;
            int64_t ext[6] = { w->oc, oh, ow, w->ic, K, K };
            int lev[6] = { 4, 4, 4, 2, 2, 2 };
            for (int a = 0; a < 6; ++a) { sp->axis_ext[a] = ext[a]; sp->axis_levels[a] = lev[a]; }
            for (int a = 0; a < 6; ++a) if (add_split(sp, a)) return -1;
            add_simple(sp, 1, 6);
            add_simple(sp, 2, 3);
            add_simple(sp, 3, 2);
            sp->n_dims[0] = 3;
            set_dim1(sp, 0, 0, w->oc, 0); set_dim1(sp, 0, 1, oh, 1); set_dim1(sp, 0, 2, ow, 2);
            sp->n_dims[1] = 3;
            set_dim1(sp, 1, 0, w->ic, 3); set_dim2(sp, 1, 1, hp, 1, S, 4); set_dim2(sp, 1, 2, wp, 2, S, 5);
            sp->n_dims[2] = 4;
            set_dim1(sp, 2, 0, w->oc, 0); set_dim1(sp, 2, 1, w->ic, 3);
            set_dim1(sp, 2, 2, K, 4); set_dim1(sp, 2, 3, K, 5);
        } else {
            /* T_DW: Out[c][y][x] = sum Data[c][y*S+ry][x*S+rx] * Ker[c][ry][rx] (Q30) */
            sp->tmpl = 2;
            sp->n_axes = 5;
            int64_t ext[5] = { w->ic, oh, ow, K, K };
            int lev[5] = { 4, 4, 4, 2, 2 };
            for (int a = 0; a < 5; ++a) { sp->axis_ext[a] = ext[a]; sp->axis_levels[a] = lev[a]; }
            for (int a = 0; a < 5; ++a) if (add_split(sp, a)) return -1;
            add_simple(sp, 1, 6);
            add_simple(sp, 2, 3);
            add_simple(sp, 3, 2);
            sp->n_dims[0] = 3;
            set_dim1(sp, 0, 0, w->ic, 0); set_dim1(sp, 0, 1, oh, 1); set_dim1(sp, 0, 2, ow, 2);
            sp->n_dims[1] = 3;
            set_dim1(sp, 1, 0, w->ic, 0); set_dim2(sp, 1, 1, hp, 1, S, 3); set_dim2(sp, 1, 2, wp, 2, S, 4);
            sp->n_dims[2] = 3;
            set_dim1(sp, 2, 0, w->ic, 0); set_dim1(sp, 2, 1, K, 3); set_dim1(sp, 2, 2, K, 4);
        }
    } else {
        return -1;
    }
    /* row-major strides over the (padded) shape (Q7) */
    for (int b = 0; b < 3; ++b) {
        int64_t s = 1;
        for (int d = sp->n_dims[b] - 1; d >= 0; --d) { sp->rowstride[b][d] = s; s *= sp->shape[b][d]; }
    }
    /* |S_e| = prod_j r_j; flat idx = c_0 + r_0 (c_1 + r_1 (c_2 + ...)) (O2) */
    uint64_t place = 1;
    for (int j = 0; j < sp->n_knobs; ++j) { sp->place[j] = place; place *= (uint64_t)sp->radix[j]; }
    sp->size = place;
    return 0;
}

int or_space_set_create(const or_workload *w, int n, or_space_set *out)
{
    memset(out, 0, sizeof(*out));
    if (n < 1 || n > OR_MAXW) return -1;
    out->n = n;
    out->offset[0] = 0;
    for (int i = 0; i < n; ++i) {
        if (space_create1(&w[i], &out->sp[i])) { or_space_set_free(out); return -1; }
        out->offset[i + 1] = out->offset[i] + out->sp[i].size;
    }
    return 0;
}

void or_space_set_free(or_space_set *s)
{
    for (int i = 0; i < OR_MAXW; ++i)
        for (int j = 0; j < OR_MAXKNOBS; ++j) { free(s->sp[i].fact[j]); s->sp[i].fact[j] = NULL; }
}

int or_space_set_find(const or_space_set *s, uint64_t gidx)
{
    for (int i = 0; i < s->n; ++i)
        if (gidx >= s->offset[i] && gidx < s->offset[i + 1]) return i;
    return -1;
}

void or_decode(const or_space *sp, uint64_t idx, int *choices)
{
    for (int j = 0; j < sp->n_knobs; ++j) {
        choices[j] = (int)(idx % (uint64_t)sp->radix[j]);
        idx /= (uint64_t)sp->radix[j];
    }
}

uint64_t or_encode(const or_space *sp, const int *choices)
{
    uint64_t idx = 0;
    for (int j = sp->n_knobs - 1; j >= 0; --j) idx = idx * (uint64_t)sp->radix[j] + (uint64_t)choices[j];
    return idx;
}

/* ======================================================================
 * Lowering x = g(e, s) into an explicit loop nest (O3).
 * ==================================================================== */
static void push_loop(const or_space *sp, const int *choices, or_nest *ns, int axis, int level)
{
    /* factor tuple of the split knob owning this axis */
    int j = -1;
    for (int q = 0; q < sp->n_knobs; ++q)
        if (sp->knob_kind[q] == 0 && sp->knob_axis[q] == axis) j = q;
    int L = sp->axis_levels[axis];
    const int *f = sp->fact[j] + (size_t)choices[j] * L;
    int k = ns->n++;
    ns->axis[k] = axis;
    ns->level[k] = level;
    ns->ext[k] = f[level];
    /* v = sum_l v_l * prod_{l' > l} f_l' */
    int64_t c = 1;
    for (int l = level + 1; l < L; ++l) c *= f[l];
    ns->coef[k] = c;
    ns->ann[k] = 0;
}

void or_lower(const or_space *sp, const int *choices, or_nest *ns)
{
    memset(ns, 0, sizeof(*ns));
    /* lexicographic permutations of three items */
    static const int perms[6][3] = { {0,1,2}, {0,2,1}, {1,0,2}, {1,2,0}, {2,0,1}, {2,1,0} };
    int unroll_max = 0, vectorize = 0;
    if (sp->tmpl == 0) {
        /* i0 j0 k0 i1 j1 k1 i2 j2 */
        push_loop(sp, choices, ns, 0, 0); push_loop(sp, choices, ns, 1, 0); push_loop(sp, choices, ns, 2, 0);
        push_loop(sp, choices, ns, 0, 1); push_loop(sp, choices, ns, 1, 1); push_loop(sp, choices, ns, 2, 1);
        push_loop(sp, choices, ns, 0, 2); push_loop(sp, choices, ns, 1, 2);
        unroll_max = sp->unroll_vals[choices[3]];
    } else if (sp->tmpl == 1) {
        /* f0 y0 x0 . f1 y1 x1 . f2 y2 x2 . perm(rc0 ry0 rx0) . rc1 ry1 rx1 . f3 y3 x3 */
        for (int l = 0; l < 3; ++l)
            for (int a = 0; a < 3; ++a) push_loop(sp, choices, ns, a, l);
        const int *p = perms[choices[6]];
        for (int q = 0; q < 3; ++q) push_loop(sp, choices, ns, 3 + p[q], 0);
        for (int a = 3; a < 6; ++a) push_loop(sp, choices, ns, a, 1);
        for (int a = 0; a < 3; ++a) push_loop(sp, choices, ns, a, 3);
        unroll_max = sp->unroll_vals[choices[7]];
        vectorize = choices[8];
    } else {
        /* c0 y0 x0 . c1 y1 x1 . c2 y2 x2 . ry0 rx0 . ry1 rx1 . perm(c3 y3 x3) */
        for (int l = 0; l < 3; ++l)
            for (int a = 0; a < 3; ++a) push_loop(sp, choices, ns, a, l);
        push_loop(sp, choices, ns, 3, 0); push_loop(sp, choices, ns, 4, 0);
        push_loop(sp, choices, ns, 3, 1); push_loop(sp, choices, ns, 4, 1);
        const int *p = perms[choices[5]];
        for (int q = 0; q < 3; ++q) push_loop(sp, choices, ns, p[q], 3);
        unroll_max = sp->unroll_vals[choices[6]];
        vectorize = choices[7];
    }
    /* annotations (O3): GPU templates bind spatial level 0/1/2 to blockIdx/vthread/threadIdx;
     * serial loops with bottom_up <= unroll_max get unroll; vectorize marks the last loop. */
    for (int k = 0; k < ns->n; ++k) {
        int bound = 0;
        if (sp->tmpl != 0 && ns->axis[k] < 3 && ns->level[k] < 3) {
            ns->ann[k] = 4 + ns->level[k];
            bound = 1;
        }
        if (!bound) {
            int64_t bu = 1;
            for (int l = k; l < ns->n; ++l) bu *= ns->ext[l];
            ns->ann[k] = (bu <= unroll_max) ? 1 : 0;
        }
    }
    if (vectorize) ns->ann[ns->n - 1] = 2;
}

/* coefficient of loop k's variable in dimension d of buffer b, 0 if absent */
static int64_t dim_coef(const or_space *sp, const or_nest *ns, int b, int d, int k)
{
    int64_t c = 0;
    for (int t = 0; t < sp->n_terms[b][d]; ++t)
        if (sp->term_axis[b][d][t] == ns->axis[k]) c += sp->term_mult[b][d][t] * ns->coef[k];
    return c;
}

/* touch count ("the number of touched elements", Q5): distinct elements of
 * buffer b touched when loops l < k are fixed and loops l >= k run over their
 * ranges.  Every loop variable enters at most one dimension of a buffer, so the
 * touched set is the Cartesian product of per-dimension value sets; each set is
 * enumerated literally over the loops of that dimension. */
uint64_t or_touch(const or_space *sp, const or_nest *ns, int b, int k)
{
    uint64_t prod = 1;
    for (int d = 0; d < sp->n_dims[b]; ++d) {
        int64_t ext[OR_MAXLOOPS], cf[OR_MAXLOOPS];
        int nl = 0;
        for (int l = k; l < ns->n; ++l) {
            int64_t c = dim_coef(sp, ns, b, d, l);
            if (c != 0) { ext[nl] = ns->ext[l]; cf[nl] = c; ++nl; }
        }
        int64_t shape = sp->shape[b][d];
        unsigned char *seen = (unsigned char *)calloc((size_t)shape, 1);
        int64_t v[OR_MAXLOOPS];
        for (int i = 0; i < nl; ++i) v[i] = 0;
        uint64_t count = 0;
        for (;;) {
            int64_t val = 0;
            for (int i = 0; i < nl; ++i) val += cf[i] * v[i];
            if (!seen[val]) { seen[val] = 1; ++count; }
            int i = nl - 1;
            while (i >= 0) { if (++v[i] < ext[i]) break; v[i] = 0; --i; }
            if (i < 0) break;
        }
        free(seen);
        prod *= count;
    }
    return prod;
}

/* brute force over the whole flat buffer (pins or_touch on tiny nests) */
uint64_t or_touch_bruteforce(const or_space *sp, const or_nest *ns, int b, int k)
{
    int64_t total = 1;
    for (int d = 0; d < sp->n_dims[b]; ++d) total *= sp->shape[b][d];
    unsigned char *seen = (unsigned char *)calloc((size_t)total, 1);
    int64_t v[OR_MAXLOOPS];
    for (int l = 0; l < ns->n; ++l) v[l] = 0;
    uint64_t count = 0;
    for (;;) {
        int64_t flat = 0;
        for (int d = 0; d < sp->n_dims[b]; ++d) {
            int64_t ix = 0;
            for (int l = k; l < ns->n; ++l) ix += dim_coef(sp, ns, b, d, l) * v[l];
            flat += ix * sp->rowstride[b][d];
        }
        if (!seen[flat]) { seen[flat] = 1; ++count; }
        int l = ns->n - 1;
        while (l >= k) { if (++v[l] < ns->ext[l]) break; v[l] = 0; --l; }
        if (l < k) break;
    }
    free(seen);
    return count;
}

/* loop context (Appendix table; Q5-Q9) */
void or_context(const or_space *sp, const or_nest *ns, or_loopctx *rows)
{
    for (int k = 0; k < ns->n; ++k) {
        or_loopctx *r = &rows[k];
        r->length = ns->ext[k];
        r->ann = ns->ann[k];
        r->top_down = 1;
        for (int l = 0; l < k; ++l) r->top_down *= ns->ext[l];      /* product of outer loop lengths */
        r->bottom_up = 1;
        for (int l = k; l < ns->n; ++l) r->bottom_up *= ns->ext[l]; /* this loop and inner loops (Q9) */
        for (int b = 0; b < 3; ++b) {
            r->touch[b] = or_touch(sp, ns, b, k);
            r->reuse[b] = (float)r->bottom_up / (float)r->touch[b];  /* P:636, Q6 */
            int64_t s = 0;
            for (int d = 0; d < sp->n_dims[b]; ++d) s += dim_coef(sp, ns, b, d, k) * sp->rowstride[b][d];
            r->stride[b] = s;                                         /* P:637, Q7 */
        }
    }
}

/* feature vector (Appendix A layout): 18 rows x 19, relation 120, scalars 4, pad 2 */
void or_features_nest(const or_space *sp, const or_nest *ns, float *out)
{
    or_loopctx rows[OR_MAXLOOPS];
    or_context(sp, ns, rows);
    for (int i = 0; i < OR_NFEAT; ++i) out[i] = 0.0f;
    for (int k = 0; k < ns->n; ++k) {
        float *z = out + 19 * k;
        z[0] = (float)rows[k].length;
        z[1 + rows[k].ann] = 1.0f;
        z[8] = (float)rows[k].top_down;
        z[9] = (float)rows[k].bottom_up;
        for (int b = 0; b < 3; ++b) {
            z[10 + 3 * b] = (float)rows[k].touch[b];
            z[11 + 3 * b] = rows[k].reuse[b];
            z[12 + 3 * b] = (float)rows[k].stride[b];
        }
    }
    /* context relation features R_t^{(ij)} = max_{k : Z_kj < beta_t} Z_ki (Q10-Q12):
     * j = touch count of buffer b, i in {reuse ratio of b, top-down}, beta_t = 2^t, t = 1..20;
     * the comparison uses the exact integer touch count; empty set -> 0. */
    for (int b = 0; b < 3; ++b) {
        for (int p = 0; p < 2; ++p) {
            for (int t = 1; t <= 20; ++t) {
                int found = 0;
                float best = 0.0f;
                for (int k = 0; k < ns->n; ++k) {
                    if (rows[k].touch[b] < ((uint64_t)1 << t)) {
                        float zi = (p == 0) ? rows[k].reuse[b] : (float)rows[k].top_down;
                        if (!found || zi > best) { best = zi; found = 1; }
                    }
                }
                out[342 + 40 * b + 20 * p + (t - 1)] = found ? best : 0.0f;
            }
        }
    }
    int64_t total = 1;
    for (int k = 0; k < ns->n; ++k) total *= ns->ext[k];
    out[462] = (float)total;
    for (int b = 0; b < 3; ++b) out[463 + b] = (float)or_touch(sp, ns, b, 0);
}

int or_features(const or_space_set *s, const uint64_t *idx, int64_t n, float *out)
{
    int choices[OR_MAXKNOBS];
    or_nest ns;
    for (int64_t i = 0; i < n; ++i) {
        int w = or_space_set_find(s, idx[i]);
        if (w < 0) return -2;
        or_decode(&s->sp[w], idx[i] - s->offset[w], choices);
        or_lower(&s->sp[w], choices, &ns);
        or_features_nest(&s->sp[w], &ns, out + (size_t)i * OR_NFEAT);
    }
    return 0;
}

/* ======================================================================
 * GBT inference (Q18 walk rule, Q19 summation order)
 * ==================================================================== */
float or_gbt_score(const or_gbt *m, const float *x, uint8_t *slots)
{
    int64_t n_int = ((int64_t)1 << m->depth) - 1;
    int64_t n_leaf = (int64_t)1 << m->depth;
    float p[32];
    for (int q = 0; q < 32; ++q) p[q] = 0.0f;
    for (int t = 0; t < m->n_trees; ++t) {
        int64_t node = 0;
        for (int d = 0; d < m->depth; ++d) {
            uint16_t f = m->feat[(size_t)t * n_int + node];
            float th = m->thresh[(size_t)t * n_int + node];
            node = (x[f] < th) ? 2 * node + 1 : 2 * node + 2;   /* go left iff x < theta */
        }
        int64_t slot = node - n_int;
        if (slots) slots[t] = (uint8_t)slot;
        p[t % 32] = p[t % 32] + m->leaf[(size_t)t * n_leaf + slot];
    }
    for (int off = 16; off >= 1; off /= 2) {
        float q[32];
        for (int i = 0; i < 32; ++i) q[i] = p[i] + p[i ^ off];
        memcpy(p, q, sizeof p);
    }
    return p[0] + m->base;
}

int or_gbt_predict(const or_gbt *m, const float *X, int64_t n, int F, float *score, uint8_t *slots)
{
    uint8_t *tmp = slots ? (uint8_t *)malloc((size_t)m->n_trees) : NULL;
    for (int64_t i = 0; i < n; ++i) {
        score[i] = or_gbt_score(m, X + (size_t)i * F, tmp);
        if (slots) for (int t = 0; t < m->n_trees; ++t) slots[(size_t)t * n + i] = tmp[t];
    }
    free(tmp);
    return 0;
}

/* SA energy of configuration gidx: f-hat(g(e, s)); with K bootstrap models, the acquisition of
 * their scores (K = 1 with kind 0 is exactly f-hat) */
typedef struct { const or_gbt *models; int K, kind; float kappa, best; } or_energy;

float or_acquisition(int kind, int K, const float *f, float kappa, float best, float *mean_out, float *std_out);

static float energy_idx(const or_space_set *s, const or_energy *en, uint64_t gidx)
{
    float x[OR_NFEAT], f[64];
    or_features(s, &gidx, 1, x);
    if (en->K == 1 && en->kind == 0) return or_gbt_score(&en->models[0], x, NULL);
    for (int k = 0; k < en->K; ++k) f[k] = or_gbt_score(&en->models[k], x, NULL);
    return or_acquisition(en->kind, en->K, f, en->kappa, en->best, NULL, NULL);
}

/* ======================================================================
 * Parallel simulated annealing (Alg. 1; O9, Q20-Q23)
 * ==================================================================== */
static int sa_explore_energy(const or_space_set *s, const or_energy *en,
                             int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                             uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                             int init, uint64_t *chain_idx, float *chain_energy,
                             uint32_t *accept_bits, float *visited_E, uint64_t *visited_idx);

int or_sa_explore(const or_space_set *s, const or_gbt *m,
                  int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                  uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                  int init, uint64_t *chain_idx, float *chain_energy,
                  uint32_t *accept_bits, float *visited_E, uint64_t *visited_idx)
{
    or_energy en = {m, 1, 0, 0.0f, 0.0f};
    return sa_explore_energy(s, &en, n_chains, n_steps, seed, round, chain_id_base, temps, chain_workload, init,
                             chain_idx, chain_energy, accept_bits, visited_E, visited_idx);
}

int or_sa_explore_acq(const or_space_set *s, const or_gbt *models, int K, int kind, float kappa, float best,
                      int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                      uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                      int init, uint64_t *chain_idx, float *chain_energy,
                      uint32_t *accept_bits, float *visited_E, uint64_t *visited_idx)
{
    if (K < 1 || K > 64) return -3;
    or_energy en = {models, K, kind, kappa, best};
    return sa_explore_energy(s, &en, n_chains, n_steps, seed, round, chain_id_base, temps, chain_workload, init,
                             chain_idx, chain_energy, accept_bits, visited_E, visited_idx);
}

static int sa_explore_energy(const or_space_set *s, const or_energy *en,
                             int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                             uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                             int init, uint64_t *chain_idx, float *chain_energy,
                             uint32_t *accept_bits, float *visited_E, uint64_t *visited_idx)
{
    int n_words = (n_steps + 31) / 32;
    for (int32_t c = 0; c < n_chains; ++c) {
        uint32_t g = chain_id_base + (uint32_t)c;
        int w = chain_workload ? chain_workload[c] : 0;
        if (w < 0 || w >= s->n) return -1;
        const or_space *sp = &s->sp[w];
        uint32_t r[4];
        uint64_t idx;
        if (init) {
            philox(seed, g, 0, round, TAG_SA_INIT, r);
            uint64_t u = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
            idx = s->offset[w] + or_mulhi64(u, sp->size);
        } else {
            idx = chain_idx[c];
            if (idx < s->offset[w] || idx >= s->offset[w + 1]) return -2;
        }
        float E = energy_idx(s, en, idx);   /* energies recomputed under the current f-hat */
        visited_E[(size_t)c * (n_steps + 1)] = E;
        visited_idx[(size_t)c * (n_steps + 1)] = idx;
        if (accept_bits) for (int q = 0; q < n_words; ++q) accept_bits[(size_t)c * n_words + q] = 0;
        /* the non-singleton knobs in knob order */
        int ns_list[OR_MAXKNOBS], n_ns = 0;
        for (int j = 0; j < sp->n_knobs; ++j) if (sp->radix[j] > 1) ns_list[n_ns++] = j;
        for (int32_t st = 0; st < n_steps; ++st) {
            philox(seed, g, (uint32_t)st, round, TAG_SA_STEP, r);
            uint64_t idx2 = idx;
            if (n_ns > 0) {
                int j = ns_list[(uint32_t)(((uint64_t)r[0] * (uint64_t)n_ns) >> 32)];
                int choices[OR_MAXKNOBS];
                or_decode(sp, idx - s->offset[w], choices);
                int v = choices[j];
                int v2 = (int)(((uint64_t)r[1] * (uint64_t)(sp->radix[j] - 1)) >> 32);
                if (v2 >= v) v2 += 1;
                choices[j] = v2;
                idx2 = s->offset[w] + or_encode(sp, choices);
            }
            float E2 = energy_idx(s, en, idx2);
            float d = E2 - E;
            int accept = 0;
            if (d <= 0.0f) {
                accept = 1;
            } else if (temps[st] > 0.0f) {
                float u = (float)(r[2] >> 8) * f_from_bits(0x33800000u);   /* 2^-24 */
                float a = -(d / temps[st]);
                if (u < or_exp_det(a)) accept = 1;
            }
            if (accept) {
                idx = idx2;
                E = E2;
                if (accept_bits) accept_bits[(size_t)c * n_words + st / 32] |= (1u << (st % 32));
            }
            visited_E[(size_t)c * (n_steps + 1) + st + 1] = E2;
            visited_idx[(size_t)c * (n_steps + 1) + st + 1] = idx2;
        }
        chain_idx[c] = idx;
        chain_energy[c] = E;
    }
    return 0;
}

static int in_sorted(const uint64_t *a, int64_t n, uint64_t v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == v;
}

typedef struct { float E; uint64_t idx; } or_key;

static int key_cmp(const void *a, const void *b)
{
    const or_key *x = (const or_key *)a, *y = (const or_key *)b;
    if (x->E < y->E) return -1;
    if (x->E > y->E) return 1;
    if (x->idx < y->idx) return -1;
    if (x->idx > y->idx) return 1;
    return 0;
}

/* O10: visited minus measured, unique by idx, sorted by (E asc, idx asc), first K per workload */
int or_topk_distinct(const or_space_set *s, const float *E, const uint64_t *idx, int64_t n,
                     const uint64_t *measured_sorted, int64_t n_measured, int32_t K,
                     uint64_t *out_idx, float *out_E, int32_t *out_n)
{
    for (int w = 0; w < s->n; ++w) {
        or_key *keys = (or_key *)malloc(sizeof(or_key) * (size_t)(n > 0 ? n : 1));
        int64_t nk = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (idx[i] < s->offset[w] || idx[i] >= s->offset[w + 1]) continue;
            if (in_sorted(measured_sorted, n_measured, idx[i])) continue;
            keys[nk].E = E[i];
            keys[nk].idx = idx[i];
            ++nk;
        }
        qsort(keys, (size_t)nk, sizeof(or_key), key_cmp);
        int32_t cnt = 0;
        for (int64_t i = 0; i < nk && cnt < K; ++i) {
            int dup = 0;
            for (int32_t q = 0; q < cnt; ++q) if (out_idx[(size_t)w * K + q] == keys[i].idx) dup = 1;
            if (dup) continue;
            out_idx[(size_t)w * K + cnt] = keys[i].idx;
            out_E[(size_t)w * K + cnt] = keys[i].E;
            ++cnt;
        }
        out_n[w] = cnt;
        free(keys);
    }
    return 0;
}

/* ======================================================================
 * Diversity-aware selection (Eq. 3) + epsilon-greedy (O11, Q24-Q27)
 * ==================================================================== */
int or_select(const or_space_set *s, int w, const uint64_t *pool_idx, const float *pool_E, int64_t n_pool,
              const uint64_t *measured_sorted, int64_t n_measured, int32_t b, float eps, float alpha,
              uint64_t seed, uint32_t round, uint64_t *out_idx, int32_t *out_n)
{
    if (w < 0 || w >= s->n || b < 0) return -1;
    const or_space *sp = &s->sp[w];
    /* Q26: ceil of the fp32 product eps * b (RN), so eps = 0.05f, b = 20 gives 1, not 2 */
    float eb = eps * (float)b;
    int32_t n_rand = (int32_t)ceilf(eb);
    if (n_rand > b) n_rand = b;
    int32_t n_g = b - n_rand;
    int32_t cnt = 0;
    /* standardized scores, fp64, sequential in pool order */
    double mu = 0.0, var = 0.0, sigma;
    for (int64_t i = 0; i < n_pool; ++i) mu += (double)pool_E[i];
    if (n_pool > 0) mu /= (double)n_pool;
    for (int64_t i = 0; i < n_pool; ++i) { double dd = (double)pool_E[i] - mu; var += dd * dd; }
    if (n_pool > 0) var /= (double)n_pool;
    sigma = sqrt(var);
    if (sigma == 0.0) sigma = 1.0;
    int *chosen = (int *)calloc((size_t)(n_pool > 0 ? n_pool : 1), sizeof(int));
    int *ch = (int *)malloc(sizeof(int) * (size_t)(n_pool > 0 ? n_pool : 1) * OR_MAXKNOBS);
    for (int64_t i = 0; i < n_pool; ++i) or_decode(sp, pool_idx[i] - s->offset[w], ch + i * OR_MAXKNOBS);
    /* greedy maximisation of L(S) = -sum z(s) + alpha * sum_j |U_{s in S} {s_j}| */
    while (cnt < n_g && cnt < n_pool) {
        int64_t best = -1;
        double best_gain = 0.0, best_z = 0.0;
        for (int64_t i = 0; i < n_pool; ++i) {
            if (chosen[i]) continue;
            int newcov = 0;
            for (int j = 0; j < sp->n_knobs; ++j) {
                int covered = 0;
                for (int64_t q = 0; q < n_pool; ++q)
                    if (chosen[q] && ch[q * OR_MAXKNOBS + j] == ch[i * OR_MAXKNOBS + j]) covered = 1;
                if (!covered) ++newcov;
            }
            double z = ((double)pool_E[i] - mu) / sigma;
            double gain = (-z) + (double)alpha * (double)newcov;
            int better = 0;
            if (best < 0) better = 1;
            else if (gain > best_gain) better = 1;
            else if (gain == best_gain && z < best_z) better = 1;
            else if (gain == best_gain && z == best_z && pool_idx[i] < pool_idx[best]) better = 1;
            if (better) { best = i; best_gain = gain; best_z = z; }
        }
        chosen[best] = 1;
        out_idx[cnt++] = pool_idx[best];
    }
    free(chosen);
    free(ch);
    /* random picks uniformly from S_e, never measured, never already selected (Q25) */
    uint64_t lo = s->offset[w], size = sp->size;
    uint64_t n_meas_w = 0;
    for (int64_t i = 0; i < n_measured; ++i) if (measured_sorted[i] >= lo && measured_sorted[i] < lo + size) ++n_meas_w;
    for (int32_t p = 0; cnt < b; ++p) {
        if (size - n_meas_w - (uint64_t)cnt == 0) break;   /* exhausted space */
        uint64_t cand = 0;
        int ok = 0;
        for (uint32_t a = 0; a < 1024 && !ok; ++a) {
            uint32_t r[4];
            philox(seed, (uint32_t)p, a, round, TAG_EPS, r);
            uint64_t u = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
            cand = lo + or_mulhi64(u, size);
            int taken = in_sorted(measured_sorted, n_measured, cand);
            for (int32_t q = 0; q < cnt && !taken; ++q) if (out_idx[q] == cand) taken = 1;
            if (!taken) ok = 1;
        }
        while (!ok) {   /* after 1024 rejections: scan upward from the last draw */
            cand = lo + ((cand - lo + 1) % size);
            int taken = in_sorted(measured_sorted, n_measured, cand);
            for (int32_t q = 0; q < cnt && !taken; ++q) if (out_idx[q] == cand) taken = 1;
            if (!taken) ok = 1;
        }
        out_idx[cnt++] = cand;
    }
    *out_n = cnt;
    return 0;
}

/* ======================================================================
 * Histogram GBT refit under the rank loss (Eq. 2; Alg. 1; O12, Q16-Q17, Q34-Q37)
 * ==================================================================== */
static int flt_cmp(const void *a, const void *b)
{
    float x = *(const float *)a, y = *(const float *)b;
    return (x < y) ? -1 : (x > y) ? 1 : 0;
}

/* cuts per feature (Q36): U <= max_bins unique values -> cuts = u_2..u_U;
 * otherwise the order statistics sorted[floor((q+1) n / max_bins)], q = 0..max_bins-2,
 * without duplicates and without the minimum.  bin(x) = #cuts <= x. */
int or_fit_cuts(const float *X, int64_t n, int F, int max_bins, float *cuts, int32_t *ncuts)
{
    float *col = (float *)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (int f = 0; f < F; ++f) {
        for (int64_t i = 0; i < n; ++i) col[i] = X[(size_t)i * F + f];
        qsort(col, (size_t)n, sizeof(float), flt_cmp);
        int64_t U = 0;
        for (int64_t i = 0; i < n; ++i) if (i == 0 || col[i] != col[i - 1]) ++U;
        float *c = cuts + (size_t)f * (max_bins - 1);
        int32_t nc = 0;
        if (U <= max_bins) {
            for (int64_t i = 1; i < n; ++i) if (col[i] != col[i - 1]) c[nc++] = col[i];
        } else {
            for (int q = 0; q < max_bins - 1; ++q) {
                float v = col[((int64_t)(q + 1) * n) / max_bins];
                if (v == col[0]) continue;
                if (nc > 0 && c[nc - 1] == v) continue;
                c[nc++] = v;
            }
        }
        ncuts[f] = nc;
    }
    free(col);
    return 0;
}

static int bin_of(const float *c, int32_t nc, float x)
{
    int b = 0;
    for (int32_t q = 0; q < nc; ++q) if (c[q] <= x) ++b;
    return b;
}

/* group permutation (Q17): inside each workload run (samples in ascending index
 * order, rank r), position pos = pi_t(r), a 4-round Feistel network on 2h bits
 * with Philox round functions, cycle-walked onto [0, n_w). */
static uint64_t feistel(uint64_t x, int h, uint64_t seed, uint32_t tree, uint32_t wkey)
{
    uint64_t mask = ((uint64_t)1 << h) - 1;
    uint64_t L = x >> h, R = x & mask;
    for (uint32_t r = 0; r < 4; ++r) {
        uint32_t o[4];
        philox(seed, (uint32_t)R, tree, (wkey << 2) | r, TAG_GROUP_PERM, o);
        uint64_t F = (uint64_t)o[0] & mask;
        uint64_t nL = R, nR = L ^ F;
        L = nL; R = nR;
    }
    return (L << h) | R;
}

int or_group_positions(const uint16_t *gkey, int64_t n, uint64_t seed, int32_t tree, int64_t *pos)
{
    unsigned char *present = (unsigned char *)calloc(65536, 1);
    for (int64_t i = 0; i < n; ++i) present[gkey[i]] = 1;
    for (uint32_t w = 0; w < 65536; ++w) {
        if (!present[w]) continue;
        int64_t nw = 0;
        for (int64_t i = 0; i < n; ++i) if (gkey[i] == w) ++nw;
        int bits = 0;
        while (((uint64_t)1 << bits) < (uint64_t)nw) ++bits;   /* 2^bits >= nw */
        int h = (bits + 1) / 2;
        if (h < 1) h = 1;
        int64_t r = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (gkey[i] != w) continue;
            uint64_t y = feistel((uint64_t)r, h, seed, (uint32_t)tree, w);
            while (y >= (uint64_t)nw) y = feistel(y, h, seed, (uint32_t)tree, w);
            pos[i] = (int64_t)y;
            ++r;
        }
    }
    free(present);
    return 0;
}

typedef struct { uint16_t w; int64_t pos; int64_t i; } or_member;

static int member_cmp(const void *a, const void *b)
{
    const or_member *x = (const or_member *)a, *y = (const or_member *)b;
    if (x->w != y->w) return x->w < y->w ? -1 : 1;
    if (x->pos != y->pos) return x->pos < y->pos ? -1 : 1;
    return 0;
}

/* Eq. 2 gradients, both orders of every pair within a group (Q17):
 * for c_i > c_j: rho = sigma(f_j - f_i) = 1 / (1 + exp_det(-(f_j - f_i)));
 * dl/df_i = -rho, dl/df_j = +rho, curvature rho (1 - rho); quantised to 2^-32. */
int or_pair_gradients(const float *cost, const float *pred, const uint16_t *gkey, int64_t n,
                      uint64_t seed, int32_t tree, int32_t group_size, int64_t *g, int64_t *h)
{
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    or_member *mem = (or_member *)malloc(sizeof(or_member) * (size_t)(n > 0 ? n : 1));
    or_group_positions(gkey, n, seed, tree, pos);
    for (int64_t i = 0; i < n; ++i) { g[i] = 0; h[i] = 0; mem[i].w = gkey[i]; mem[i].pos = pos[i]; mem[i].i = i; }
    qsort(mem, (size_t)n, sizeof(or_member), member_cmp);   /* groups: runs of (w, pos / group_size) */
    for (int64_t a = 0; a < n; ++a) {
        for (int64_t b = a + 1; b < n; ++b) {
            if (mem[b].w != mem[a].w || mem[b].pos / group_size != mem[a].pos / group_size) break;
            int64_t i = mem[a].i, j = mem[b].i;
            if (cost[i] == cost[j]) continue;        /* sign(c_i - c_j) = 0 contributes nothing */
            if (cost[i] < cost[j]) { int64_t tmp = i; i = j; j = tmp; }   /* now c_i > c_j */
            float d = pred[j] - pred[i];
            float e = or_exp_det(-d);
            float rho = 1.0f / (1.0f + e);
            float hh = rho * (1.0f - rho);
            int64_t q = llrint((double)rho * 4294967296.0);
            int64_t qh = llrint((double)hh * 4294967296.0);
            /* the ordered pairs (i, j) and (j, i) of Eq. 2 carry the same term */
            g[i] -= 2 * q;
            g[j] += 2 * q;
            h[i] += 2 * qh;
            h[j] += 2 * qh;
        }
    }
    free(pos);
    free(mem);
    return 0;
}

/* Regression loss of P:175, sum_i (f_i - c_i)^2 taken literally: dl/df_i = 2 (f_i - c_i),
 * d2l/df_i^2 = 2, in the same 2^-32 fixed point as the rank-loss terms. */
int or_reg_gradients(const float *cost, const float *pred, int64_t n, int64_t *g, int64_t *h)
{
    for (int64_t i = 0; i < n; ++i) {
        double r = (double)pred[i] - (double)cost[i];
        g[i] = llrint(2.0 * r * 4294967296.0);
        h[i] = 2 * (int64_t)4294967296LL;
    }
    return 0;
}

double or_rank_loss(const float *cost, const float *pred, int64_t n)
{
    double L = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (i == j) continue;
            double sg = (cost[i] > cost[j]) ? 1.0 : (cost[i] < cost[j]) ? -1.0 : 0.0;
            L += log1p(exp(-sg * ((double)pred[i] - (double)pred[j])));
        }
    return L;
}

int or_fit_hist(const float *X, int64_t n, int F, const float *cost, const uint16_t *gkey,
                const or_fit_opts *o, uint16_t *feat, float *thresh, float *leaf,
                float *pred_out, int64_t *hist0_out)
{
    if (n <= 0) return -7;
    const int D = o->depth, B = o->max_bins;
    const int64_t n_int = ((int64_t)1 << D) - 1, n_leaf = (int64_t)1 << D;
    const double S = 1.0 / 4294967296.0;   /* 2^-32 */
    const double lam = (double)o->lambda, mcw = (double)o->min_child_weight, eta = (double)o->eta;
    float *cuts = (float *)malloc(sizeof(float) * (size_t)F * (B - 1));
    int32_t *ncuts = (int32_t *)malloc(sizeof(int32_t) * (size_t)F);
    or_fit_cuts(X, n, F, B, cuts, ncuts);
    int *bins = (int *)malloc(sizeof(int) * (size_t)n * F);
    for (int64_t i = 0; i < n; ++i)
        for (int f = 0; f < F; ++f)
            bins[(size_t)i * F + f] = bin_of(cuts + (size_t)f * (B - 1), ncuts[f], X[(size_t)i * F + f]);
    float *pred = (float *)malloc(sizeof(float) * (size_t)n);
    /* base score 0 (Q35), or the caller's margin: f = f_global + f_local fits f_local on top of
     * f_global's predictions (Eq. 4) */
    for (int64_t i = 0; i < n; ++i) pred[i] = o->base_margin ? o->base_margin[i] : 0.0f;
    int64_t *g = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *h = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *node = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *hg = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_leaf * B);
    int64_t *hh = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_leaf * B);
    int64_t *Gn = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_leaf);
    int64_t *Hn = (int64_t *)malloc(sizeof(int64_t) * (size_t)n_leaf);
    int *bf = (int *)malloc(sizeof(int) * (size_t)n_leaf);
    int *bs = (int *)malloc(sizeof(int) * (size_t)n_leaf);
    double *bg = (double *)malloc(sizeof(double) * (size_t)n_leaf);
    char *dead = (char *)malloc((size_t)(n_int + n_leaf));

    for (int t = 0; t < o->n_trees; ++t) {
        if (o->objective == 1) or_reg_gradients(cost, pred, n, g, h);
        else or_pair_gradients(cost, pred, gkey, n, o->seed, t, o->group_size, g, h);
        for (int64_t i = 0; i < n; ++i) node[i] = 0;
        memset(dead, 0, (size_t)(n_int + n_leaf));
        uint16_t *tf = feat + (size_t)t * n_int;
        float *tt = thresh + (size_t)t * n_int;
        for (int d = 0; d < D; ++d) {
            const int64_t first = ((int64_t)1 << d) - 1, nn = (int64_t)1 << d;
            for (int64_t q = 0; q < nn; ++q) { bf[q] = -1; bs[q] = 0; bg[q] = 0.0; Gn[q] = 0; Hn[q] = 0; }
            for (int64_t i = 0; i < n; ++i) { Gn[node[i] - first] += g[i]; Hn[node[i] - first] += h[i]; }
            for (int f = 0; f < F; ++f) {
                /* histogram of (g, h) over the bins of feature f, one per node of this level */
                for (int64_t q = 0; q < nn * B; ++q) { hg[q] = 0; hh[q] = 0; }
                for (int64_t i = 0; i < n; ++i) {
                    int64_t q = (node[i] - first) * B + bins[(size_t)i * F + f];
                    hg[q] += g[i];
                    hh[q] += h[i];
                }
                if (t == 0 && d == 0 && hist0_out)
                    for (int q = 0; q < B; ++q) {
                        hist0_out[((size_t)f * B + q) * 2] = hg[q];
                        hist0_out[((size_t)f * B + q) * 2 + 1] = hh[q];
                    }
                for (int64_t q = 0; q < nn; ++q) {
                    if (dead[first + q]) continue;
                    double G = (double)Gn[q] * S, H = (double)Hn[q] * S;
                    int64_t GLi = 0, HLi = 0;
                    for (int s = 1; s <= ncuts[f]; ++s) {
                        GLi += hg[q * B + s - 1];
                        HLi += hh[q * B + s - 1];
                        double GL = (double)GLi * S, HL = (double)HLi * S;
                        double GR = (double)(Gn[q] - GLi) * S, HR = (double)(Hn[q] - HLi) * S;
                        if (HL < mcw || HR < mcw) continue;
                        double gain = (GL * GL / (HL + lam) + GR * GR / (HR + lam)) - G * G / (H + lam);
                        if (!(gain > 0.0)) continue;
                        /* max gain; ties -> lower feature, then lower split (ascending scan, strict >) */
                        if (bf[q] < 0 || gain > bg[q]) { bf[q] = f; bs[q] = s; bg[q] = gain; }
                    }
                }
            }
            for (int64_t q = 0; q < nn; ++q) {
                int64_t nd = first + q;
                if (bf[q] < 0) {
                    /* no valid split: pass-through node, every sample goes left (Q18) */
                    tf[nd] = 0;
                    tt[nd] = INFINITY;
                    dead[2 * nd + 1] = 1;
                    dead[2 * nd + 2] = 1;
                } else {
                    tf[nd] = (uint16_t)bf[q];
                    tt[nd] = cuts[(size_t)bf[q] * (B - 1) + bs[q] - 1];
                }
            }
            for (int64_t i = 0; i < n; ++i) {
                int64_t q = node[i] - first;
                if (bf[q] < 0) node[i] = 2 * node[i] + 1;
                else node[i] = (bins[(size_t)i * F + bf[q]] < bs[q]) ? 2 * node[i] + 1 : 2 * node[i] + 2;
            }
        }
        /* leaves w = -eta G / (H + lambda) (eta folded in, Q35); then f_i += w in tree order (Q37) */
        float *tl = leaf + (size_t)t * n_leaf;
        for (int64_t l = 0; l < n_leaf; ++l) { Gn[l] = 0; Hn[l] = 0; }
        for (int64_t i = 0; i < n; ++i) { Gn[node[i] - n_int] += g[i]; Hn[node[i] - n_int] += h[i]; }
        for (int64_t l = 0; l < n_leaf; ++l) {
            double G = (double)Gn[l] * S, H = (double)Hn[l] * S;
            tl[l] = (float)(-(eta * (G / (H + lam))));
        }
        for (int64_t i = 0; i < n; ++i) pred[i] = pred[i] + tl[node[i] - n_int];
    }
    if (pred_out) memcpy(pred_out, pred, sizeof(float) * (size_t)n);
    free(cuts); free(ncuts); free(bins); free(pred); free(g); free(h); free(node);
    free(hg); free(hh); free(dead); free(Gn); free(Hn); free(bf); free(bs); free(bg);
    return 0;
}

/* ======================================================================
 * Transfer learning, Eq. 4: one ensemble holding the global model's trees, then
 * the local model's; a shallower tree is padded to the common depth with pass-through nodes.
 * ==================================================================== */
static void copy_padded(const or_gbt *m, int t, int D, uint16_t *feat, float *thresh, float *leaf)
{
    const int64_t ni = ((int64_t)1 << m->depth) - 1, nl = (int64_t)1 << m->depth;
    const int64_t NI = ((int64_t)1 << D) - 1, NL = (int64_t)1 << D;
    for (int64_t k = 0; k < NI; ++k) { feat[k] = 0; thresh[k] = INFINITY; }
    for (int64_t l = 0; l < NL; ++l) leaf[l] = 0.0f;
    /* heap node k of depth d keeps index k: the top levels coincide */
    for (int64_t k = 0; k < ni; ++k) { feat[k] = m->feat[(size_t)t * ni + k]; thresh[k] = m->thresh[(size_t)t * ni + k]; }
    /* old leaf slot s is heap node ni + s; below it every node goes left, so it ends at the
     * leftmost descendant (ni + s + 1) * 2^(D - d) - 1, i.e. slot s << (D - d) */
    for (int64_t s = 0; s < nl; ++s) leaf[s << (D - m->depth)] = m->leaf[(size_t)t * nl + s];
}

int or_gbt_concat(const or_gbt *a, const or_gbt *b, uint16_t *feat, float *thresh, float *leaf, float *base)
{
    const int D = a->depth > b->depth ? a->depth : b->depth;
    const int64_t NI = ((int64_t)1 << D) - 1, NL = (int64_t)1 << D;
    for (int t = 0; t < a->n_trees; ++t)
        copy_padded(a, t, D, feat + (size_t)t * NI, thresh + (size_t)t * NI, leaf + (size_t)t * NL);
    for (int t = 0; t < b->n_trees; ++t) {
        const size_t u = (size_t)(a->n_trees + t);
        copy_padded(b, t, D, feat + u * NI, thresh + u * NI, leaf + u * NL);
    }
    *base = a->base + b->base;
    return 0;
}

/* ======================================================================
 * Uncertainty estimate by bootstrapping, EI / UCB acquisition (readings Q40-Q43)
 * ==================================================================== */
/* Q40: model k's training multiset: draw r = 0..n-1 picks sample (u * n) >> 32 with
 * u = word 0 of Philox(r, k, round, TAG_BOOT) (uniform, with replacement). */
int or_bootstrap_indices(int64_t n, int32_t model, uint64_t seed, uint32_t round, int64_t *idx)
{
    for (int64_t r = 0; r < n; ++r) {
        uint32_t o[4];
        philox(seed, (uint32_t)r, (uint32_t)model, round, TAG_BOOT, o);
        idx[r] = (int64_t)(((uint64_t)o[0] * (uint64_t)n) >> 32);
    }
    return 0;
}

/* Q43: expected improvement below the incumbent `best` for a minimised cost, in fp32 with one
 * RN operation per step: EI = d Phi(z) + sigma phi(z), d = best - mu, z = d / sigma; sigma = 0
 * gives max(d, 0).  Phi(z) = 1 - erfc(z / sqrt 2) / 2 (z >= 0), erfc(x / sqrt 2)/2 (z < 0), with
 * Abramowitz-Stegun 7.1.26 for erfc(x) = t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) exp(-x^2),
 * t = 1 / (1 + p x) (|error| <= 1.5e-7), phi(z) = exp(-z^2 / 2) / sqrt(2 pi); exp = exp_det. */
float or_expected_improvement(float mu, float sd, float best)
{
    float d = best - mu;
    if (!(sd > 0.0f)) return d > 0.0f ? d : 0.0f;
    float z = d / sd;
    float x = fabsf(z) * 0.70710677f;                     /* |z| / sqrt 2 */
    float t = 1.0f / (1.0f + 0.3275911f * x);
    float poly = 1.061405429f;
    poly = poly * t + -1.453152027f;
    poly = poly * t + 1.421413741f;
    poly = poly * t + -0.284496736f;
    poly = poly * t + 0.254829592f;
    poly = poly * t;
    float ec = poly * or_exp_det(-(x * x));               /* erfc(x) */
    float Phi = z >= 0.0f ? 1.0f - 0.5f * ec : 0.5f * ec;
    float phi = 0.3989423f * or_exp_det((-0.5f * z) * z);
    return d * Phi + sd * phi;
}

/* Q41/Q42: over the K models' scores f[k]: mean and population standard deviation in fp64
 * (sequential sums in model order), then the energy SA minimises:
 * kind 0 mean, kind 1 lower confidence bound mu - kappa sigma (UCB for a minimised cost,
 * fp64, rounded once), kind 2 -EI(mu, sigma, best) in fp32. */
float or_acquisition(int kind, int K, const float *f, float kappa, float best, float *mean_out, float *std_out)
{
    double mu = 0.0, v = 0.0;
    for (int k = 0; k < K; ++k) mu += (double)f[k];
    mu = mu / (double)K;
    for (int k = 0; k < K; ++k) { double e = (double)f[k] - mu; v += e * e; }
    double sd = sqrt(v / (double)K);
    if (mean_out) *mean_out = (float)mu;
    if (std_out) *std_out = (float)sd;
    if (kind == 1) return (float)(mu - (double)kappa * sd);
    if (kind == 2) return -or_expected_improvement((float)mu, (float)sd, best);
    return (float)mu;
}

int or_gbt_predict_acq(const or_gbt *models, int K, const float *X, int64_t n, int F, int kind, float kappa,
                       float best, float *score, float *mean, float *std)
{
    float f[64];
    if (K < 1 || K > 64) return -1;
    for (int64_t i = 0; i < n; ++i) {
        for (int k = 0; k < K; ++k) f[k] = or_gbt_score(&models[k], X + (size_t)i * F, NULL);
        score[i] = or_acquisition(kind, K, f, kappa, best, mean ? &mean[i] : NULL, std ? &std[i] : NULL);
    }
    return 0;
}

/* ======================================================================
 * Configuration features ("directly use configuration s as the model's input";
 * reading Q44): per knob in knob order, a split knob's ordered factor tuple (outer first), the
 * reorder knob's permutation index, the unroll knob's max-step value, the vectorize flag; as
 * fp32 columns, zero padded to OR_NKNOBF.
 * ==================================================================== */
int or_features_knobs(const or_space_set *s, const uint64_t *idx, int64_t n, float *out /* [n][OR_NKNOBF] */)
{
    for (int64_t i = 0; i < n; ++i) {
        int w = or_space_set_find(s, idx[i]);
        if (w < 0) return -2;
        const or_space *sp = &s->sp[w];
        int choices[OR_MAXKNOBS];
        or_decode(sp, idx[i] - s->offset[w], choices);
        float *x = out + (size_t)i * OR_NKNOBF;
        for (int c = 0; c < OR_NKNOBF; ++c) x[c] = 0.0f;
        int c = 0;
        for (int j = 0; j < sp->n_knobs; ++j) {
            if (sp->knob_kind[j] == 0) {
                int L = sp->axis_levels[sp->knob_axis[j]];
                for (int l = 0; l < L; ++l) x[c++] = (float)sp->fact[j][(size_t)choices[j] * L + l];
            } else if (sp->knob_kind[j] == 2) {
                x[c++] = (float)sp->unroll_vals[choices[j]];
            } else {
                x[c++] = (float)choices[j];
            }
        }
    }
    return 0;
}
