/*
 * at_b200.h -- C-ABI of the B200-native (sm_100a) AutoTVM hot path (arXiv 1805.08166).
 *
 * The six calls follow the paper's problem statement argmin_{s in S_e} f(g(e, s))
 * (Eq. 1) and Algorithm 1:
 *
 *   space_create      S_e for workload(s) e ........................ P:61
 *   features_extract  x = g(e, s) encoded as loop-context + relation
 *                     features, the input of f-hat .................. P:243-257
 *   gbt_predict       f-hat(x), the GBT cost model .................. P:129-133
 *   sa_explore        "run parallel simulated annealing to collect
 *                     candidates ... using energy function f-hat" ... Alg. 1
 *   select_topk       "greedy submodular optimization to pick a
 *                     (1-eps)b-subset" + "randomly sample eps b" ...... Alg. 1, Eq. 3
 *   gbt_fit_hist      "update f-hat using D" with the rank loss ....... Alg. 1, Eq. 2
 *
 * and the SURVEY §8(f) widenings, on the same kernels:
 *   gbt_fit_hist objective / d_base_margin   regression loss; f_local fitted on top of
 *                                            f_global (transfer learning, Eq. 4)
 *   gbt_concat        f_global + f_local as one ensemble ......... Eq. 4
 *   bootstrap_resample, gbt_predict_acq, at_sa_opts.acq
 *                     bootstrap uncertainty, EI / UCB acquisition .. P:208-215
 *   features_knobs    the configuration representation s .......... P:229-232
 *
 * Conventions
 *  - Every pointer named d_* is DEVICE memory owned by the caller; every other
 *    pointer is host memory owned by the caller.  The library never retains a
 *    caller pointer after the call returns, except for stream-ordered reads by
 *    work it enqueued on `stream`.
 *  - Opaque handles (at_space, at_gbt) own device copies of their tables; they
 *    are freed by the matching *_destroy.
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy default stream.
 *    Every call except *_create, *_destroy, *_info and gbt_export is asynchronous
 *    and stream-ordered; no call synchronizes the device unless stated.
 *  - Status codes: AT_OK (0) or a negative AT_E* code.  Arguments are validated on
 *    the host before anything is launched; on error nothing is launched and
 *    at_last_error() returns a message (thread-local).  No C++ exception crosses
 *    the ABI.  CUDA launch failures return AT_ECUDA.
 *  - Index errors found on the device ("errors: out-of-range index"): a
 *    global index >= |S| passed to features_extract / features_knobs, a persistent chain
 *    state or a chain workload outside its workload in sa_explore, a pool entry outside
 *    `workload` in select_topk.  The kernel clamps the entry to a valid one (its outputs
 *    for that entry are undefined) and raises the space's error word; the NEXT call on
 *    that space returns AT_ERANGE without launching anything (and clears the word), or
 *    space_check(sp, stream) synchronizes `stream` and reports it at once.
 *  - The library needs an sm_100a device (B200).  There is no CPU fallback.
 *  - Bit-exactness contract: indices, features, leaf slots,
 *    accept bits, top-k, selections, histograms and fitted trees are bit-identical
 *    to the CPU oracle (oracle/); GBT scores agree within 1e-6 relative.
 */
#ifndef AT_B200_H
#define AT_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define AT_API __attribute__((visibility("default")))
#else
#define AT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    AT_OK = 0,
    AT_EINVAL = -1,        /* malformed argument (null pointer, negative size, bad enum) */
    AT_ERANGE = -2,        /* an index outside [0, |S|) */
    AT_ENOMEM = -3,        /* device allocation failed */
    AT_ECUDA = -4,         /* a CUDA runtime / launch error */
    AT_EMISMATCH = -5,     /* sizes or leading dimensions that do not agree */
    AT_EUNSUPPORTED = -6,  /* a valid request outside what this build supports */
    AT_EEMPTY = -7         /* empty training set */
};

#define AT_NFEAT 468       /* feature columns, identical for every workload (Appendix A layout) */

typedef struct at_space_s *at_space;
typedef struct at_gbt_s *at_gbt;

/* Thread-local message describing the last non-AT_OK return on this thread. */
AT_API const char *at_last_error(void);

/* ------------------------------------------------------------------ workloads
 * e in E.  kind 0 = matmul C[n][m] = sum_k A[k][n] B[k][m] (paper
 * layout); kind 1 = conv2d NCHW batch 1, Out[oc][oh][ow] = sum Data[ic][y*S+ry][x*S+rx]
 * * Ker[oc][ic][ry][rx] over the zero-padded (h+2 pad) x (w+2 pad) input (Table 1,
 * P:276-296); kind 2 = depthwise conv (MobileNet), channels in `ic`.
 */
typedef struct {
    int32_t kind;
    int32_t n, m, k;                               /* matmul */
    int32_t h, w, ic, oc, ksize, stride, pad;      /* conv2d / depthwise */
} at_workload;

/* space_create -- build S_e for n_workloads workloads.
 * Templates (reading Q3): matmul -> T_MM [split_i(3), split_j(3), split_k(2),
 * unroll{1,2,4,8,16}]; conv2d -> T_CONV [tile_f/y/x (4 levels), tile_rc/ry/rx (2),
 * reorder (6), unroll{0,512,1500}, vectorize{0,1}]; depthwise -> T_DW [tile_c/y/x (4),
 * tile_ry/rx (2), reorder (6), unroll (3), vectorize (2)].  Split domains are all ordered
 * factorizations, lexicographic; flat idx = c_0 + r_0 (c_1 + r_1 (...)).  With
 * n_workloads > 1 the space is the union, global idx = offset_w + local idx.
 * Synchronous (uploads the tables).  Errors: AT_EINVAL (bad shape/kind, n_workloads
 * not in [1, 16]), AT_EUNSUPPORTED (a |S_w|, a loop-nest iteration count or a buffer
 * size >= 2^32). */
AT_API int space_create(const at_workload *w, int32_t n_workloads, at_space *out);

/* space_info -- host query.  size_total = |S| of the union; offsets[n_workloads+1]
 * (nullable); radices[n_workloads][9] (nullable, unused knobs 0); n_features = 468. */
AT_API int space_info(at_space sp, uint64_t *size_total, int32_t *n_workloads, int32_t *n_features,
               uint64_t *offsets, int32_t *radices);
AT_API int space_destroy(at_space sp);
/* space_check -- synchronizes `stream`, then returns AT_ERANGE if a kernel of an earlier call on
 * this space met an out-of-range index (see Conventions), else AT_OK.  Clears the error word. */
AT_API int space_check(at_space sp, void *stream);

/* features_extract -- for each global index d_idx[i], i < n: decode the knobs,
 * lower to the loop nest x = g(e, s) and write its 468 features as column i
 * of d_feat, SoA [468][ld] fp32 (feature f of candidate i at d_feat[f * ld + i]).
 * Layout (Appendix A): 18 loop rows x 19 (length, one-hot annotation x7, top-down,
 * bottom-up, per buffer touch/reuse/stride x3), 120 relation features
 * R_t = max_{k: touch_b(k) < 2^t} Z_k,{reuse_b, top-down}, total
 * iterations, 3 footprints, 2 zero pads.  Requires ld >= n and ld % 4 == 0.
 * An index >= |S| is detected on the device: its column is undefined and the next call on
 * the space (or space_check) returns AT_ERANGE.  n == 0 is a no-op. */
AT_API int features_extract(at_space sp, const uint64_t *d_idx, int64_t n, float *d_feat, int64_t ld,
                     void *stream);

/* features_knobs -- the configuration representation "directly use configuration s as the
 * model's input" (reading Q44), the baseline the loop-context features are compared
 * with: per knob in knob order a split knob's ordered factor tuple (outer factor first), the
 * reorder knob's permutation index, the unroll knob's max-step value, the vectorize flag, as fp32
 * columns of d_feat SoA [AT_KNOB_FEATURES][ld] (zero padded).  Models over it are created with
 * n_features = AT_KNOB_FEATURES and scored by gbt_predict. */
#define AT_KNOB_FEATURES 32
AT_API int features_knobs(at_space sp, const uint64_t *d_idx, int64_t n, float *d_feat, int64_t ld, void *stream);

/* ------------------------------------------------------------------ GBT model
 * Complete binary trees of depth D in heap layout (children 2i+1, 2i+2); node i of
 * tree t: feature feat[t][i], threshold thresh[t][i]; go left iff x[feat] < thresh
 * (x == thresh goes right); leaves leaf[t][2^D] with the learning rate folded in.
 * f-hat(x) = sum_t leaf_t(x) + base, summed in the canonical order (reading Q19):
 * p[q] = sum_{t = q mod 32, ascending t} leaf_t (fp32, from +0), then
 * p[q] += p[q ^ off] for off = 16, 8, 4, 2, 1, score = p[0] + base.
 * gbt_create copies HOST arrays feat [T][2^D-1] u16 (< n_features), thresh
 * [T][2^D-1] f32, leaf [T][2^D] f32.  1 <= depth <= 8, n_trees >= 1. */
AT_API int gbt_create(int32_t n_trees, int32_t depth, int32_t n_features, const uint16_t *feat,
               const float *thresh, const float *leaf, float base, at_gbt *out);
AT_API int gbt_info(at_gbt g, int32_t *n_trees, int32_t *depth, int32_t *n_features);
/* copies the ensemble back to HOST arrays (any may be NULL); synchronous */
AT_API int gbt_export(at_gbt g, uint16_t *feat, float *thresh, float *leaf, float *base);
AT_API int gbt_destroy(at_gbt g);

/* gbt_predict -- d_score[i] = f-hat(column i of d_feat [n_features][ld]), i < n.
 * d_leaf_slot (nullable) receives the leaf slot of every tree, u8 [T][n]. */
AT_API int gbt_predict(at_gbt g, const float *d_feat, int64_t n, int64_t ld, float *d_score,
                uint8_t *d_leaf_slot, void *stream);

/* ------------------------------------------------------------------ exploration
 * sa_explore -- n_chains Metropolis chains, n_steps steps each (Alg. 1 P:152-153;
 * "a batch of parallel Markov chains", states persistent across f-hat updates).
 * Chain c has global id g = chain_id_base + c; its random numbers are
 * Philox4x32-10(counter (g, step, round, tag), key seed) (reading Q28), so a chain's
 * trajectory does not depend on how chains are split across ranks.
 * Step s: pick the floor(u0 * n_ns / 2^32)-th non-singleton knob j, a new value
 * floor(u1 (r_j - 1) / 2^32) (+1 if >= the current), score the proposal, accept iff
 * E' <= E or (T_s > 0 and (u2 >> 8) 2^-24 < exp_det(-(E' - E) / T_s)) (readings Q20-Q22).
 * Collected set (Q23): the start state and every proposal, minus d_measured_sorted,
 * distinct by idx; per workload the k_out smallest (E, idx) are written to
 * d_out_idx / d_out_score [n_workloads][k_out], counts to d_out_n [n_workloads].
 */
typedef struct {
    int32_t n_chains, n_steps, k_out;
    int32_t init;                 /* 1: start from Philox(g, 0, round, SA_INIT) draws; 0: from d_chain_idx */
    uint64_t seed;
    uint32_t round;
    uint32_t chain_id_base;
    const float *d_temps;         /* [n_steps] temperatures T_s (caller schedule, Q21) */
    uint32_t *d_accept_bits;      /* nullable: [n_chains][(n_steps+31)/32], bit s = step s accepted */
    float *d_visited_E;           /* nullable: [n_chains][n_steps+1] energies of start + proposals */
    uint64_t *d_visited_idx;      /* nullable: [n_chains][n_steps+1] their global indices */
    const struct at_acq_opts_s *acq;   /* nullable: the energy is the acquisition over acq->n_models
                                          concatenated models (gbt_predict_acq) */
} at_sa_opts;

AT_API int sa_explore(at_space sp, at_gbt g,
               uint64_t *d_chain_idx,                /* [n_chains] in (init == 0) / out: final states */
               float *d_chain_energy,                /* [n_chains] out: final energies */
               const uint16_t *d_chain_workload,     /* [n_chains] workload of each chain; NULL -> 0 */
               const uint64_t *d_measured_sorted, int64_t n_measured,
               const at_sa_opts *o,
               uint64_t *d_out_idx, float *d_out_score, int32_t *d_out_n, void *stream);

/* topk_merge -- the rank-merge step of sa_explore (a7): distinct k_out smallest
 * (E, idx) per workload of the union of n_lists lists laid out [n_lists][n_workloads][k_in]
 * with valid counts d_in_n [n_lists][n_workloads] (e.g. all-gathered per-rank top-k). */
AT_API int topk_merge(at_space sp, const uint64_t *d_in_idx, const float *d_in_score, const int32_t *d_in_n,
               int32_t n_lists, int32_t k_in, const uint64_t *d_measured_sorted, int64_t n_measured,
               int32_t k_out, uint64_t *d_out_idx, float *d_out_score, int32_t *d_out_n, void *stream);

/* select_topk -- b candidates for measurement from the pool (Alg. 1):
 * greedy maximisation of Eq. 3 L(S) = -sum z(s) + alpha sum_j |U {s_j}| on scores
 * standardized over the pool (fp64, sequential), b - ceil(eps b) picks (ties: lower z,
 * then lower idx), then uniformly random unmeasured, unselected configurations of
 * workload `workload` (Philox tag EPS) until b or the space is exhausted (Q24-Q27).
 * Output order: greedy picks, then random picks; count to *d_out_n. */
typedef struct {
    int32_t b;
    float eps;
    float alpha;
    uint64_t seed;
    uint32_t round;
} at_select_opts;

AT_API int select_topk(at_space sp, int32_t workload, const uint64_t *d_pool_idx, const float *d_pool_score,
                int64_t n_pool, const uint64_t *d_measured_sorted, int64_t n_measured,
                const at_select_opts *o, uint64_t *d_out_idx, int32_t *d_out_n, void *stream);

/* select_topk_batch -- select_topk for workloads w0 .. w0 + n_w - 1 in ONE launch (one block per
 * workload), each from its own pool: pool q at d_pool_idx / d_pool_score + q * pool_stride with
 * d_pool_n[q] valid entries (device counts, e.g. the out_n of sa_explore / topk_merge; NULL ->
 * n_pool_max each).  Results d_out_idx [n_w][b], d_out_n [n_w]; bit-identical to n_w select_topk calls
 * with the same options. */
AT_API int select_topk_batch(at_space sp, int32_t w0, int32_t n_w, const uint64_t *d_pool_idx,
                             const float *d_pool_score, int64_t pool_stride, const int32_t *d_pool_n,
                             int64_t n_pool_max, const uint64_t *d_measured_sorted, int64_t n_measured,
                             const at_select_opts *o, uint64_t *d_out_idx, int32_t *d_out_n, void *stream);

/* ------------------------------------------------------------------ model update
 * gbt_fit_hist -- histogram GBT under the pairwise rank loss (Eq. 2), refit
 * from scratch (readings Q16, Q17, Q34-Q37): cuts per feature (<= max_bins-1),
 * per tree Philox-Feistel groups of group_size inside each workload, both orders of
 * every pair, int64 fixed-point (2^-32) gradients, per-level histograms, best split by
 * fp64 gain (ties: lower feature, lower bin), leaves -eta G / (H + lambda), fp32
 * prediction update in tree order.
 * d_feat is SoA [n_features][ld] of ALL n samples (replicated on every rank);
 * histograms are built over [hist_begin, hist_end) only and then summed by
 * o->allreduce (NULL -> single rank, the range must be [0, n)).  allreduce is called
 * once per tree level and once per tree for the leaves, on `stream`, with a device
 * buffer of `count` int64 to be summed in place across ranks.  Group keys < 1024.
 * Writes the fitted ensemble to *out (a new handle); d_pred_out (nullable) [n] gets
 * the fit's final training predictions; d_hist0_out (nullable) [n_features][max_bins][2]
 * gets tree 0's root histogram (after the reduction).  Errors: AT_EEMPTY (n == 0),
 * AT_EINVAL (non-finite cost), AT_EUNSUPPORTED (depth > 8, max_bins > 256, group key >= 1024).
 * Host synchronization: a single-rank fit (one fused launch for n <= 2048 samples, else the
 * histogram-subtraction path, whose layout is computed on the device and whose launches are sized
 * by upper bounds) reads every data-dependent size on the device and never blocks the host; its
 * input errors (non-finite cost, group key >= 1024) travel with the returned model -- every later
 * call on it (gbt_predict, sa_explore, gbt_export, gbt_concat, ...) returns AT_EINVAL.  Multi-rank
 * fits (the all-reduce count is the cut total) and the level-by-level path (AT_FIT_SUB=0) read the
 * cut counts back once and return those errors directly.  n_features <= 8192 on the subtraction
 * path (else level-by-level). */
typedef int (*at_allreduce_i64_fn)(int64_t *d_buf, int64_t count, void *ctx, void *stream);

typedef struct {
    int32_t n_trees, depth, max_bins, group_size;
    float eta, lambda, min_child_weight;
    uint64_t seed;
    at_allreduce_i64_fn allreduce;
    void *ctx;
    float *d_pred_out;
    int64_t *d_hist0_out;
    int32_t objective;            /* AT_OBJ_RANK (Eq. 2) or AT_OBJ_REG: sum_i (f_i - c_i)^2,
                                     g_i = 2 (f_i - c_i), h_i = 2 in 2^-32 fixed point; valid while
                                     sum_i |f_i - c_i| < 2^30 */
    const float *d_base_margin;   /* nullable [n]: initial predictions f_i (else 0); transfer
                                     learning fits f_local on top of f_global (Eq. 4) */
} at_fit_opts;
enum { AT_OBJ_RANK = 0, AT_OBJ_REG = 1 };

AT_API int gbt_fit_hist(const float *d_feat, int64_t n, int64_t ld, int32_t n_features,
                 const float *d_cost, const uint16_t *d_group_key,
                 int64_t hist_begin, int64_t hist_end, const at_fit_opts *o, at_gbt *out, void *stream);

/* ------------------------------------------------------------------ uncertainty
 * "We can use bootstrapping to get the model's uncertainty estimate" with EI / UCB acquisition
 * (readings Q40-Q43).
 * bootstrap_resample -- model `model`'s training multiset: output row r is input sample
 * (u * n) >> 32, u = word 0 of Philox(r, model, round, TAG_BOOT = 6) (n draws with replacement);
 * copies the features (SoA [n_features][ld] -> [n_features][ld_out]), costs and group keys, and
 * the drawn indices to d_idx_out (nullable).  Fit each model on its multiset with gbt_fit_hist,
 * then gbt_concat the K models (equal tree counts) for gbt_predict_acq.
 * gbt_predict_acq -- K = n_models equal-size models concatenated in g (model k = trees
 * [k T/K, (k+1) T/K)): each model's score in the canonical order (Q19) plus model_base[k] -- bit
 * for bit gbt_predict of that model alone -- then in fp64 over the K scores the mean mu and the
 * population std sigma (model order), and the energy to minimise: AT_ACQ_MEAN mu, AT_ACQ_UCB
 * mu - kappa sigma (the confidence bound of a minimised cost), AT_ACQ_EI -EI(mu, sigma; best)
 * with EI = d Phi(d / sigma) + sigma phi(d / sigma), d = best - mu (fp32, exp_det, A&S 7.1.26).
 * Writes d_score [n] and, when non-NULL, d_mean / d_std [n] (fp32). */
enum { AT_ACQ_MEAN = 0, AT_ACQ_UCB = 1, AT_ACQ_EI = 2 };
typedef struct at_acq_opts_s {
    int32_t n_models;             /* 1..8, divides the ensemble's tree count */
    int32_t kind;                 /* AT_ACQ_* */
    float kappa;                  /* UCB exploration weight */
    float best;                   /* EI incumbent (model scale), e.g. min mu over the measured set */
    float model_base[8];          /* base score of each model (gbt_concat sums the bases) */
} at_acq_opts;

AT_API int bootstrap_resample(const float *d_feat, int64_t n, int64_t ld, int32_t n_features, const float *d_cost,
                              const uint16_t *d_group_key, int32_t model, uint64_t seed, uint32_t round,
                              float *d_feat_out, int64_t ld_out, float *d_cost_out, uint16_t *d_key_out,
                              int64_t *d_idx_out, void *stream);
AT_API int gbt_predict_acq(at_gbt g, const float *d_feat, int64_t n, int64_t ld, const at_acq_opts *o, float *d_score,
                           float *d_mean, float *d_std, void *stream);

/* gbt_concat -- transfer learning, Eq. 4: f(x) = f_global(x) + f_local(x) as ONE
 * ensemble (a's trees, then b's), so gbt_predict / sa_explore score it unchanged.  A tree
 * shallower than max(depth) is padded with pass-through nodes (feature 0, threshold +inf:
 * always left), its leaves moved to the leftmost descendant slots (slot s -> s << (D - d)),
 * which leaves every tree's value unchanged; base = a.base + b.base (fp32).  The sum is taken
 * in the canonical order of the combined ensemble (Q19), i.e. equal to f_a(x) + f_b(x) up to
 * fp32 rounding.  Host-side construction like gbt_create; *out is a new handle.  Errors:
 * AT_EMISMATCH (different n_features). */
AT_API int gbt_concat(at_gbt a, at_gbt b, at_gbt *out);

/* at_exp_det_eval -- d_out[i] = exp_det(the fp32 whose bits are first_bits + i), i < n (u32
 * wrap-around).  exp_det is the deterministic fp32 exp of the Metropolis acceptance test (Alg. 1
 * P:152-153) and of Eq. 2's sigmoid, reading Q22: clamps at -87 / 88, n = rint(a log2 e),
 * two-step Cody-Waite reduction, degree-7 Horner polynomial with fma, times 2^n.  Exposed so that
 * the device implementation can be compared with the oracle's on all 2^32 inputs. */
AT_API int at_exp_det_eval(uint32_t first_bits, int64_t n, float *d_out, void *stream);

/* ------------------------------------------------------------------ instrumentation
 * at_launch_count: kernels this library launched since load (bench "gpu_launches").
 * at_prof_enable(1): from now on every launch of a kernel class is bracketed by CUDA
 * events recorded on the stream it is launched on; at_prof_query synchronizes on those
 * events and returns the class's launch count and summed device milliseconds since
 * the last at_prof_reset.  Kernel classes: */
enum {
    AT_K_FEATURES = 0, AT_K_PREDICT = 1, AT_K_SA = 2, AT_K_TOPK = 3, AT_K_SELECT = 4,
    AT_K_FIT_PREP = 5, AT_K_FIT_GRAD = 6, AT_K_FIT_HIST = 7, AT_K_FIT_SPLIT = 8, AT_K_FIT_UPDATE = 9,
    AT_K_FIT_GRAPH = 10,   /* a single-rank fit's trees, launched as one CUDA graph */
    AT_K_NCLASSES = 11
};
AT_API int64_t at_launch_count(void);
AT_API int at_prof_enable(int on);
AT_API int at_prof_reset(void);
AT_API int at_prof_query(int32_t kernel_class, int64_t *launches, double *total_ms);

#ifdef __cplusplus
}
#endif
#endif
