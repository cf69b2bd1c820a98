/*
 * oracle.h -- plain, slow CPU oracle for the AutoTVM hot path (arXiv 1805.08166).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_1805_08166_b200/) never includes, links or calls
 * anything here; the two share no code, headers, tables or constants.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named
 * beside it); "Qn" = reading n of DESIGN.md section 3 (taken from SURVEY.md
 * section 8(c) where the paper is silent).
 *
 * Every function here follows the paper's definition (or the DESIGN reading)
 * literally: explicit loop nests, enumeration of touched elements, pointer
 * walks of trees, sequential sums.  No blocking, fusion or closed forms.
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (no FTZ/DAZ).
 */
#ifndef AUTOTVM_ORACLE_H
#define AUTOTVM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_NFEAT 468       /* Appendix A feature vector length (Q14) */
#define OR_MAXLOOPS 18     /* T_CONV nest depth (Q3) */
#define OR_MAXKNOBS 9
#define OR_MAXW 16         /* workloads in one union space */
#define OR_NKNOBF 32       /* configuration-feature columns (Q44) */

/* workload e (P:45 matmul, Table 1 P:276-296 conv2d, MobileNet depthwise Q30) */
typedef struct {
    int32_t kind;                 /* 0 matmul C[n][m] = sum_k A[k][n] B[k][m]; 1 conv2d NCHW; 2 depthwise */
    int32_t n, m, k;              /* matmul extents */
    int32_t h, w, ic, oc, ksize, stride, pad;   /* conv / depthwise (dw uses ic as C) */
} or_workload;

/* one workload's schedule space S_e and its geometry */
typedef struct {
    or_workload wl;
    int tmpl;                      /* 0 T_MM, 1 T_CONV, 2 T_DW (Q3) */
    int n_axes;
    int64_t axis_ext[6];
    int axis_levels[6];
    int n_knobs;
    int knob_kind[OR_MAXKNOBS];    /* 0 split, 1 reorder, 2 unroll, 3 vectorize */
    int knob_axis[OR_MAXKNOBS];
    int radix[OR_MAXKNOBS];
    int *fact[OR_MAXKNOBS];        /* split knobs: [radix][levels] ordered factor tuples */
    uint64_t place[OR_MAXKNOBS];   /* mixed-radix place values, knob 0 fastest */
    uint64_t size;                 /* |S_e| */
    int unroll_vals[5];
    /* buffers b0 = output, b1 = first input, b2 = second input (O1) */
    int n_dims[3];
    int64_t shape[3][4];
    int64_t rowstride[3][4];
    int n_terms[3][4];
    int term_axis[3][4][2];
    int64_t term_mult[3][4][2];
} or_space;

typedef struct {
    int n;
    or_space sp[OR_MAXW];
    uint64_t offset[OR_MAXW + 1];
} or_space_set;

/* the lowered loop nest x = g(e, s), outer -> inner */
typedef struct {
    int n;
    int axis[OR_MAXLOOPS];
    int level[OR_MAXLOOPS];
    int64_t ext[OR_MAXLOOPS];
    int ann[OR_MAXLOOPS];          /* 0 serial 1 unroll 2 vectorize 3 parallel 4 blockIdx 5 vthread 6 threadIdx */
    int64_t coef[OR_MAXLOOPS];     /* coefficient of this loop variable inside its axis */
} or_nest;

/* per-loop context rows exposed for the Appendix-C pins */
typedef struct {
    int64_t length, top_down, bottom_up;
    int ann;
    uint64_t touch[3];
    float reuse[3];
    int64_t stride[3];
} or_loopctx;

/* GBT ensemble: complete trees of depth D in heap layout (Q18) */
typedef struct {
    int32_t n_trees, depth;
    const uint16_t *feat;   /* [T][2^D-1] */
    const float *thresh;    /* [T][2^D-1] */
    const float *leaf;      /* [T][2^D] */
    float base;
} or_gbt;

/* ---- space ---- */
int  or_space_set_create(const or_workload *w, int n, or_space_set *out);
void or_space_set_free(or_space_set *s);
int  or_space_set_find(const or_space_set *s, uint64_t gidx);       /* workload of a global index */
void or_decode(const or_space *sp, uint64_t idx, int *choices);
uint64_t or_encode(const or_space *sp, const int *choices);
uint64_t or_count_factorizations(int64_t n, int L);                 /* brute-force count (pins) */

/* ---- lowering + features ---- */
void or_lower(const or_space *sp, const int *choices, or_nest *out);
uint64_t or_touch(const or_space *sp, const or_nest *nest, int b, int k);
uint64_t or_touch_bruteforce(const or_space *sp, const or_nest *nest, int b, int k);
void or_context(const or_space *sp, const or_nest *nest, or_loopctx *rows);
void or_features_nest(const or_space *sp, const or_nest *nest, float *out);
int  or_features(const or_space_set *s, const uint64_t *idx, int64_t n, float *out /* [n][468] */);

/* ---- RNG and the shared-by-spec transcendental ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t or_mulhi64(uint64_t a, uint64_t b);
float or_exp_det(float a);
void or_exp_det_range(uint32_t first_bits, int64_t n, float *out);

/* ---- GBT inference ---- */
float or_gbt_score(const or_gbt *m, const float *x, uint8_t *slots /* [T] or NULL */);
int   or_gbt_predict(const or_gbt *m, const float *X /* [n][F] */, int64_t n, int F,
                     float *score, uint8_t *slots /* [T][n] or NULL */);

/* ---- parallel SA (Alg. 1) ---- */
int or_sa_explore(const or_space_set *s, const or_gbt *m,
                  int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                  uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                  int init, uint64_t *chain_idx, float *chain_energy,
                  uint32_t *accept_bits /* [n_chains][(n_steps+31)/32] or NULL */,
                  float *visited_E /* [n_chains][n_steps+1] */, uint64_t *visited_idx);

/* distinct top-K of a visited set, per workload (Q23) */
int or_topk_distinct(const or_space_set *s, const float *E, const uint64_t *idx, int64_t n,
                     const uint64_t *measured_sorted, int64_t n_measured, int32_t K,
                     uint64_t *out_idx /* [n_w][K] */, float *out_E, int32_t *out_n /* [n_w] */);

/* ---- diversity-aware selection, Eq. 3 + epsilon-greedy ---- */
int or_select(const or_space_set *s, int w, const uint64_t *pool_idx, const float *pool_E, int64_t n_pool,
              const uint64_t *measured_sorted, int64_t n_measured, int32_t b, float eps, float alpha,
              uint64_t seed, uint32_t round, uint64_t *out_idx, int32_t *out_n);

/* ---- histogram GBT refit under the rank loss, Eq. 2 ---- */
typedef struct {
    int32_t n_trees, depth, max_bins, group_size;
    float eta, lambda, min_child_weight;
    uint64_t seed;
    int32_t objective;          /* 0: rank loss, Eq. 2; 1: regression loss sum (f - c)^2 */
    const float *base_margin;   /* [n] initial predictions (transfer learning, Eq. 4); NULL -> 0 */
} or_fit_opts;

int or_fit_cuts(const float *X /* [n][F] */, int64_t n, int F, int max_bins,
                float *cuts /* [F][max_bins-1] */, int32_t *ncuts /* [F] */);
int or_group_positions(const uint16_t *gkey, int64_t n, uint64_t seed, int32_t tree,
                       int64_t *pos /* [n] position inside its workload run */);
int or_pair_gradients(const float *cost, const float *pred, const uint16_t *gkey, int64_t n,
                      uint64_t seed, int32_t tree, int32_t group_size, int64_t *g, int64_t *h);
int or_fit_hist(const float *X /* [n][F] */, int64_t n, int F, const float *cost, const uint16_t *gkey,
                const or_fit_opts *o, uint16_t *feat, float *thresh, float *leaf,
                float *pred_out /* [n] final fit predictions, nullable */,
                int64_t *hist0_out /* tree-0 root histogram [F][max_bins][2], nullable */);
double or_rank_loss(const float *cost, const float *pred, int64_t n);   /* Eq. 2 over all ordered pairs */
/* regression loss sum_i (f_i - c_i)^2: g_i = 2 (f_i - c_i), h_i = 2, quantised to 2^-32 */
int or_reg_gradients(const float *cost, const float *pred, int64_t n, int64_t *g, int64_t *h);

/* ---- transfer learning, Eq. 4: f(x) = f_global(x) + f_local(x) as ONE ensemble:
 * the trees of a then those of b (a tree shallower than max(depth) padded with pass-through
 * nodes (f 0, theta +inf: always left), its leaf copied to the leftmost descendant slot),
 * base = a.base + b.base (fp32).  Arrays sized for (a.n_trees + b.n_trees) trees of depth
 * max(a.depth, b.depth). */
int or_gbt_concat(const or_gbt *a, const or_gbt *b, uint16_t *feat, float *thresh, float *leaf, float *base);

/* ---- configuration features, the knob representation of P:229-232 (Q44) ---- */
int or_features_knobs(const or_space_set *s, const uint64_t *idx, int64_t n, float *out /* [n][OR_NKNOBF] */);

/* ---- bootstrap uncertainty, EI / UCB acquisition (Q40-Q43) ---- */
int or_bootstrap_indices(int64_t n, int32_t model, uint64_t seed, uint32_t round, int64_t *idx);
float or_expected_improvement(float mu, float sd, float best);
float or_acquisition(int kind /* 0 mean, 1 UCB (mu - kappa sigma), 2 -EI */, int K, const float *f, float kappa,
                     float best, float *mean_out, float *std_out);
/* SA whose energy is the acquisition over K models (kind 0 / K 1: plain f-hat, = or_sa_explore) */
int or_sa_explore_acq(const or_space_set *s, const or_gbt *models, int K, int kind, float kappa, float best,
                      int32_t n_chains, int32_t n_steps, uint64_t seed, uint32_t round,
                      uint32_t chain_id_base, const float *temps, const uint16_t *chain_workload,
                      int init, uint64_t *chain_idx, float *chain_energy,
                      uint32_t *accept_bits, float *visited_E, uint64_t *visited_idx);
int or_gbt_predict_acq(const or_gbt *models /* [K] */, int K, const float *X /* [n][F] */, int64_t n, int F,
                       int kind, float kappa, float best, float *score, float *mean, float *std);

#ifdef __cplusplus
}
#endif
#endif
