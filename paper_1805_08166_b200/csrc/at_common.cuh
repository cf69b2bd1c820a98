// at_common.cuh -- shared internals of the sm_100a library (never seen by the oracle).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/at_b200.h"

namespace at {

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);

#define AT_CUDA_TRY(expr)                                         \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::at::cuda_fail(_e, #expr); \
    } while (0)

#define AT_LAUNCH_CHECK(name)                                      \
    do {                                                           \
        cudaError_t _e = cudaGetLastError();                       \
        if (_e != cudaSuccess) return ::at::cuda_fail(_e, name);   \
    } while (0)

// launch accounting + optional per-class CUDA-event timing (at_prof_*)
void prof_begin(int cls, cudaStream_t s);
void prof_end(int cls, cudaStream_t s);
void note_launch();            // one library kernel launched (at_launch_count)
void pool_keep();              // keep freed stream-ordered scratch in the default pool (once per device)
void prof_suspend(bool on);   // while capturing a graph: count launches, record no events

struct ProfScope {
    int cls;
    cudaStream_t s;
    ProfScope(int c, cudaStream_t st) : cls(c), s(st) { prof_begin(cls, s); }
    ~ProfScope() { prof_end(cls, s); }
};

// device-side bounds checks of the data-dependent indices (tools/checks_run.sh builds a variant with
// -DAT_CHECKS and runs the GPU tests on it: compute-sanitizer is closed on the GPU pool)
#ifdef AT_CHECKS
#define AT_DCHECK(cond)                                                                                       \
    do {                                                                                                      \
        if (!(cond)) {                                                                                        \
            printf("AT_CHECKS %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond, (int)blockIdx.x, \
                   (int)threadIdx.x);                                                                         \
            __trap();                                                                                         \
        }                                                                                                     \
    } while (0)
#else
#define AT_DCHECK(cond) \
    do {                \
    } while (0)
#endif

// ---------------------------------------------------------------- constants
constexpr int NFEAT = 468;
constexpr int MAXLOOPS = 18;
constexpr int MAXKNOBS = 9;
constexpr int MAXW = 16;

enum Tag : uint32_t { TAG_SA_INIT = 0, TAG_SA_STEP = 1, TAG_EPS = 2, TAG_GROUP_PERM = 3, TAG_BOOT = 6 };

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG (Salmon et al., SC'11), counter (id, step, round, tag), key (seed lo, hi).
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ U4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
#else
        uint64_t p0 = 0xD2511F53ull * c0, p1 = 0xCD9E8D57ull * c2;
        uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
        uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return U4{c0, c1, c2, c3};
}

__host__ __device__ __forceinline__ U4 philox(uint64_t seed, uint32_t id, uint32_t step, uint32_t round,
                                              uint32_t tag)
{
    return philox10(id, step, round, tag, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// floor(a * b / 2^64)
__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// ---------------------------------------------------------------- exp_det (DESIGN reading Q22)
// fp32 RN ops only: clamp, n = rint(a log2e), two-step Cody-Waite reduction with fma,
// degree-7 Taylor polynomial in Horner form with fma, scale by the normal float 2^n.
__device__ __forceinline__ float exp_det(float a)
{
    if (a < -87.0f) return 0.0f;
    if (a > 88.0f) return __int_as_float(0x7f800000);
    float t = __fmul_rn(a, __int_as_float(0x3FB8AA3B));
    float n = rintf(t);
    float r = __fmaf_rn(-n, __int_as_float(0x3F317200), a);
    r = __fmaf_rn(-n, __int_as_float(0x35BFBE8E), r);
    float p = __int_as_float(0x39500D01);
    p = __fmaf_rn(p, r, __int_as_float(0x3AB60B61));
    p = __fmaf_rn(p, r, __int_as_float(0x3C088889));
    p = __fmaf_rn(p, r, __int_as_float(0x3D2AAAAB));
    p = __fmaf_rn(p, r, __int_as_float(0x3E2AAAAB));
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    int e = (int)n;
    return __fmul_rn(p, __int_as_float((e + 127) << 23));
}

// order-preserving float -> u32 (no NaNs on this path; -0 never produced, see DESIGN)
__host__ __device__ __forceinline__ uint32_t fkey(float f)
{
#ifdef __CUDA_ARCH__
    uint32_t b = __float_as_uint(f);
#else
    uint32_t b;
    memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float fkey_inv(uint32_t k)
{
    uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    memcpy(&f, &b, 4);
    return f;
#endif
}

// ---------------------------------------------------------------- device space description
// One workload's schedule space and loop-nest geometry, uploaded by space_create.
struct WlDev {
    int32_t tmpl;                 // 0 T_MM, 1 T_CONV, 2 T_DW
    int32_t n_knobs;
    uint32_t radix[MAXKNOBS];
    uint32_t place[MAXKNOBS];
    uint32_t size;                // |S_w| < 2^32
    uint32_t n_ns;                // number of non-singleton knobs
    uint8_t ns_list[MAXKNOBS];    // their knob ids in knob order
    uint8_t pad_[3];
    uint32_t fact_off[MAXKNOBS];  // u16 offset of the split knob's [radix][L] factor table
    uint32_t unroll_vals[5];
    // geometry (u32 everywhere; space_create guarantees no overflow)
    uint32_t S;                   // conv stride
    uint32_t str_out[3];          // rowstrides of b0 dims
    uint32_t str_in[3];           // rowstrides of b1 dims (Data / A)
    uint32_t str_ker[4];          // rowstrides of b2 dims (Ker / B)
    uint64_t offset;              // union offset
};

struct SpaceDev {
    int32_t n_w;
    uint64_t offset[MAXW + 1];
    WlDev w[MAXW];
    uint32_t *err;                // mapped host word: set by a kernel that met an out-of-range index
};

// an index outside the space (or a chain / pool entry outside its workload): the kernel clamps it
// to a valid one and raises the space's error word, which the next call on the space (or
// space_check) reports as AT_ERANGE
__device__ __forceinline__ void flag_range(const SpaceDev *S)
{
    *(volatile uint32_t *)S->err = 1u;
    __threadfence_system();
}

}  // namespace at

struct at_space_s {
    at::SpaceDev host;            // host mirror
    at::SpaceDev *d_space;        // device copy
    uint16_t *d_fact;             // device factor tables
    uint64_t total;
    // lazily grown scratch for sa_explore / topk_merge
    void *d_scratch;
    size_t scratch_bytes;
    uint32_t *h_err;              // mapped pinned word (device view in host.err); see flag_range
};

struct at_gbt_s {
    int32_t n_trees, depth, n_features;
    int32_t t_pad;                // allocation padded to a multiple of 16 trees (zero-filled), for bulk copies
    float base;
    uint2 *d_nodes;               // [t_pad][2^D-1] {feature, threshold bits}
    float *d_leaf;                // [t_pad][2^D]
    cudaStream_t last;            // stream of the last enqueued use: gbt_destroy frees stream-ordered
                                  // there (no device-wide sync from cudaFree inside a tuning loop)
    // rank form for deep ensembles (gbt.cu): node = k | (tile byte offset of f) << 16 with k the
    // 1-based index of its threshold among feature f's sorted distinct thresholds thr_val[thr_off[f] ..]; x < theta_k
    // <=> rank(x) < k, rank(x) = #{theta <= x}.  rk_state: 0 not built, 1 built, -1 unavailable
    uint32_t *d_rk_nodes;
    int32_t *d_thr_off;
    float *d_thr_val;
    int32_t rk_state;
    uint32_t *h_err;              // mapped word (fitted models): nonzero when the fit met a non-finite
                                  // cost or a group key >= 1024; every later call on the model
                                  // reports AT_EINVAL (gbt_fit_hist's small-fit path never syncs)
};

namespace at {
int scratch_reserve(at_space sp, size_t bytes, cudaStream_t s);
// AT_ERANGE (and clears the word) if a kernel enqueued earlier on this space met an out-of-range
// index and has already finished; AT_OK otherwise.  Never synchronizes.
int take_range_error(at_space sp);
// AT_EINVAL if the fit that produced g flagged bad input (see at_gbt_s::h_err); never synchronizes
int model_error(at_gbt g);
}
