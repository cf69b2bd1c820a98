// runtime.cu -- error state, launch accounting / event profiling, scratch memory.
#include <atomic>
#include <mutex>
#include <vector>

#include "at_common.cuh"

namespace at {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return AT_ECUDA;
}

// ---------------------------------------------------------------- profiling
static std::atomic<int64_t> g_launches{0};
static thread_local bool g_suspend = false;

void prof_suspend(bool on) { g_suspend = on; }
void note_launch() { g_launches.fetch_add(1); }

// Stream-ordered scratch (cudaMallocAsync / cudaFreeAsync: fit workspaces, rank tiles, model tables)
// stays in the device's default pool between calls instead of going back to the driver at every
// synchronisation (release threshold 0 by default), so a call inside a tuning loop does not pay
// for re-mapping its workspace.  Once per device.
void pool_keep()
{
    static int done_dev[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done_dev[dev]) return;
    cudaMemPool_t pool;
    uint64_t keep = ~0ull;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    done_dev[dev] = 1;
}
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
struct EvPair { cudaEvent_t a, b; };
static std::vector<EvPair> g_ev[AT_K_NCLASSES];
static std::vector<EvPair> g_pool;
static cudaEvent_t g_open[AT_K_NCLASSES];

static cudaEvent_t take_event()
{
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(int cls, cudaStream_t s)
{
    if (!g_prof_on.load() || g_suspend) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e;
    if (!g_pool.empty()) { e = g_pool.back().a; g_pool.pop_back(); } else e = take_event();
    cudaEventRecord(e, s);
    g_open[cls] = e;
}

void prof_end(int cls, cudaStream_t s)
{
    if (!g_prof_on.load() || g_suspend) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t e;
    if (!g_pool.empty()) { e = g_pool.back().a; g_pool.pop_back(); } else e = take_event();
    cudaEventRecord(e, s);
    g_ev[cls].push_back(EvPair{g_open[cls], e});
}

int scratch_reserve(at_space sp, size_t bytes, cudaStream_t s)
{
    if (sp->scratch_bytes >= bytes) return AT_OK;
    if (sp->d_scratch) {
        AT_CUDA_TRY(cudaStreamSynchronize(s));
        cudaFree(sp->d_scratch);
        sp->d_scratch = nullptr;
        sp->scratch_bytes = 0;
    }
    size_t want = bytes + bytes / 4;
    if (cudaMalloc(&sp->d_scratch, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(AT_ENOMEM, "scratch allocation of " + std::to_string(want) + " bytes failed");
    }
    sp->scratch_bytes = want;
    return AT_OK;
}

int model_error(at_gbt g)
{
    if (g && g->h_err && *(volatile uint32_t *)g->h_err)
        return fail(AT_EINVAL, *(volatile uint32_t *)g->h_err == 2u
                                   ? "this model's fit met a group key >= 1024: the model is undefined"
                                   : "this model's fit met a non-finite cost: the model is undefined");
    return AT_OK;
}

int take_range_error(at_space sp)
{
    if (sp->h_err && *(volatile uint32_t *)sp->h_err) {
        *(volatile uint32_t *)sp->h_err = 0u;
        return fail(AT_ERANGE, "an index outside the space (or outside its workload) was passed to an earlier call "
                               "on this space; its outputs for that entry are undefined");
    }
    return AT_OK;
}

__global__ void exp_det_kernel(uint32_t first, int64_t n, float *__restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = exp_det(__uint_as_float(first + (uint32_t)i));
}

}  // namespace at

extern "C" {

int at_exp_det_eval(uint32_t first_bits, int64_t n, float *d_out, void *stream)
{
    if (n < 0 || n > 0x100000000ll || (n > 0 && !d_out)) return at::fail(AT_EINVAL, "at_exp_det_eval: bad n / buffer");
    if (n == 0) return AT_OK;
    cudaStream_t s = (cudaStream_t)stream;
    at::exp_det_kernel<<<148 * 8, 256, 0, s>>>(first_bits, n, d_out);
    at::note_launch();
    AT_LAUNCH_CHECK("exp_det_kernel");
    return AT_OK;
}

int space_check(at_space sp, void *stream)
{
    if (!sp) return at::fail(AT_EINVAL, "space_check: null space");
    AT_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return at::take_range_error(sp);
}

const char *at_last_error(void) { return at::g_err.c_str(); }

int64_t at_launch_count(void) { return at::g_launches.load(); }

int at_prof_enable(int on)
{
    at::g_prof_on.store(on ? 1 : 0);
    return AT_OK;
}

int at_prof_reset(void)
{
    std::lock_guard<std::mutex> lk(at::g_prof_mu);
    for (int c = 0; c < AT_K_NCLASSES; ++c) {
        for (auto &p : at::g_ev[c]) {
            cudaEventSynchronize(p.b);
            at::g_pool.push_back(at::EvPair{p.a, nullptr});
            at::g_pool.push_back(at::EvPair{p.b, nullptr});
        }
        at::g_ev[c].clear();
    }
    return AT_OK;
}

int at_prof_query(int32_t cls, int64_t *launches, double *total_ms)
{
    if (cls < 0 || cls >= AT_K_NCLASSES) return at::fail(AT_EINVAL, "at_prof_query: bad kernel class");
    std::lock_guard<std::mutex> lk(at::g_prof_mu);
    double tot = 0.0;
    for (auto &p : at::g_ev[cls]) {
        cudaError_t e = cudaEventSynchronize(p.b);
        if (e != cudaSuccess) return at::cuda_fail(e, "at_prof_query");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        tot += ms;
    }
    if (launches) *launches = (int64_t)at::g_ev[cls].size();
    if (total_ms) *total_ms = tot;
    return AT_OK;
}

}  // extern "C"
