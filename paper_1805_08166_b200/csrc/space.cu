// space.cu -- space_create / space_info / space_destroy (DESIGN reading Q3).
//
// Split-knob domains (every ordered L-tuple with product = extent, lexicographic) are
// generated here from the prime factorisation of the extent: each prime's exponent is
// distributed over the L slots in every possible way, the tuples are multiplied out
// and sorted.  (The oracle enumerates them with nested divisor loops instead.)
#include <algorithm>
#include <array>
#include <cstring>
#include <vector>

#include "at_common.cuh"

namespace {

using Tuple = std::array<uint32_t, 4>;

void compositions(int e, int L, int i, std::array<int, 4> &cur, std::vector<std::array<int, 4>> &out)
{
    if (i == L - 1) {
        cur[i] = e;
        out.push_back(cur);
        return;
    }
    for (int x = 0; x <= e; ++x) {
        cur[i] = x;
        compositions(e - x, L, i + 1, cur, out);
    }
}

std::vector<Tuple> ordered_factorizations(uint32_t n, int L)
{
    std::vector<std::pair<uint32_t, int>> pf;
    uint32_t m = n;
    for (uint32_t p = 2; (uint64_t)p * p <= m; ++p) {
        int e = 0;
        while (m % p == 0) { m /= p; ++e; }
        if (e) pf.push_back({p, e});
    }
    if (m > 1) pf.push_back({m, 1});
    std::vector<Tuple> res(1, Tuple{1, 1, 1, 1});
    for (auto &pe : pf) {
        std::vector<std::array<int, 4>> comps;
        std::array<int, 4> cur{0, 0, 0, 0};
        compositions(pe.second, L, 0, cur, comps);
        std::vector<Tuple> nxt;
        for (auto &t : res)
            for (auto &c : comps) {
                Tuple u = t;
                for (int l = 0; l < L; ++l)
                    for (int k = 0; k < c[l]; ++k) u[l] *= pe.first;
                nxt.push_back(u);
            }
        res.swap(nxt);
    }
    std::sort(res.begin(), res.end(), [L](const Tuple &a, const Tuple &b) {
        for (int l = 0; l < L; ++l)
            if (a[l] != b[l]) return a[l] < b[l];
        return false;
    });
    return res;
}

struct Builder {
    std::vector<uint16_t> fact;
    int add_split(at::WlDev &W, int j, uint64_t extent, int L)
    {
        auto tabs = ordered_factorizations((uint32_t)extent, L);
        W.fact_off[j] = (uint32_t)fact.size();
        W.radix[j] = (uint32_t)tabs.size();
        for (auto &t : tabs)
            for (int l = 0; l < L; ++l) fact.push_back((uint16_t)t[l]);
        return 0;
    }
};

int build_workload(const at_workload &w, at::WlDev &W, Builder &B)
{
    std::memset(&W, 0, sizeof(W));
    const uint64_t LIM = 0xFFFFFFFFull;
    if (w.kind == 0) {
        if (w.n < 1 || w.m < 1 || w.k < 1) return at::fail(AT_EINVAL, "matmul extents must be >= 1");
        if (w.n > 65535 || w.m > 65535 || w.k > 65535) return at::fail(AT_EUNSUPPORTED, "extent > 65535");
        uint64_t iters = (uint64_t)w.n * w.m * w.k;
        if (iters > LIM || (uint64_t)w.n * w.m > LIM || (uint64_t)w.k * w.n > LIM || (uint64_t)w.k * w.m > LIM)
            return at::fail(AT_EUNSUPPORTED, "matmul iteration count >= 2^32");
        W.tmpl = 0;
        W.n_knobs = 4;
        B.add_split(W, 0, w.n, 3);
        B.add_split(W, 1, w.m, 3);
        B.add_split(W, 2, w.k, 2);
        W.radix[3] = 5;
        const uint32_t uv[5] = {1, 2, 4, 8, 16};
        std::memcpy(W.unroll_vals, uv, sizeof uv);
        W.S = 1;
        W.str_out[0] = (uint32_t)w.m; W.str_out[1] = 1;      // C[n][m]
        W.str_in[0] = (uint32_t)w.n;  W.str_in[1] = 1;       // A[k][n]
        W.str_ker[0] = (uint32_t)w.m; W.str_ker[1] = 1;      // B[k][m]
    } else if (w.kind == 1 || w.kind == 2) {
        if (w.h < 1 || w.w < 1 || w.ic < 1 || w.ksize < 1 || w.stride < 1 || w.pad < 0 || (w.kind == 1 && w.oc < 1))
            return at::fail(AT_EINVAL, "bad conv shape");
        uint64_t hp = (uint64_t)w.h + 2 * (uint64_t)w.pad, wp = (uint64_t)w.w + 2 * (uint64_t)w.pad;
        if (hp < (uint64_t)w.ksize || wp < (uint64_t)w.ksize) return at::fail(AT_EINVAL, "kernel larger than padded input");
        uint64_t oh = (hp - w.ksize) / w.stride + 1, ow = (wp - w.ksize) / w.stride + 1;
        uint64_t K = (uint64_t)w.ksize;
        uint64_t C = (uint64_t)w.ic, OC = (w.kind == 1) ? (uint64_t)w.oc : C;
        if (OC > 65535 || C > 65535 || oh > 65535 || ow > 65535 || K > 65535)
            return at::fail(AT_EUNSUPPORTED, "extent > 65535");
        uint64_t iters = (w.kind == 1) ? OC * oh * ow * C * K * K : C * oh * ow * K * K;
        uint64_t in_sz = C * hp * wp, out_sz = OC * oh * ow, ker_sz = (w.kind == 1) ? OC * C * K * K : C * K * K;
        if (iters > LIM || in_sz > LIM || out_sz > LIM || ker_sz > LIM)
            return at::fail(AT_EUNSUPPORTED, "conv iteration count or buffer size >= 2^32");
        const uint32_t uv[5] = {0, 512, 1500, 0, 0};
        std::memcpy(W.unroll_vals, uv, sizeof uv);
        W.S = (uint32_t)w.stride;
        W.str_out[0] = (uint32_t)(oh * ow); W.str_out[1] = (uint32_t)ow; W.str_out[2] = 1;
        W.str_in[0] = (uint32_t)(hp * wp);  W.str_in[1] = (uint32_t)wp;  W.str_in[2] = 1;
        if (w.kind == 1) {
            W.tmpl = 1;
            W.n_knobs = 9;
            B.add_split(W, 0, OC, 4);
            B.add_split(W, 1, oh, 4);
            B.add_split(W, 2, ow, 4);
            B.add_split(W, 3, C, 2);
            B.add_split(W, 4, K, 2);
            B.add_split(W, 5, K, 2);
            W.radix[6] = 6; W.radix[7] = 3; W.radix[8] = 2;
            W.str_ker[0] = (uint32_t)(C * K * K); W.str_ker[1] = (uint32_t)(K * K);
            W.str_ker[2] = (uint32_t)K; W.str_ker[3] = 1;
        } else {
            W.tmpl = 2;
            W.n_knobs = 8;
            B.add_split(W, 0, C, 4);
            B.add_split(W, 1, oh, 4);
            B.add_split(W, 2, ow, 4);
            B.add_split(W, 3, K, 2);
            B.add_split(W, 4, K, 2);
            W.radix[5] = 6; W.radix[6] = 3; W.radix[7] = 2;
            W.str_ker[0] = (uint32_t)(K * K); W.str_ker[1] = (uint32_t)K; W.str_ker[2] = 1;
        }
    } else {
        return at::fail(AT_EINVAL, "workload kind must be 0 (matmul), 1 (conv2d) or 2 (depthwise)");
    }
    uint64_t place = 1;
    W.n_ns = 0;
    for (int j = 0; j < W.n_knobs; ++j) {
        W.place[j] = (uint32_t)place;
        place *= W.radix[j];
        if (place > LIM) return at::fail(AT_EUNSUPPORTED, "|S_w| >= 2^32");
        if (W.radix[j] > 1) W.ns_list[W.n_ns++] = (uint8_t)j;
    }
    W.size = (uint32_t)place;
    return AT_OK;
}

}  // namespace

extern "C" {

int space_create(const at_workload *w, int32_t n_workloads, at_space *out)
{
    if (!w || !out) return at::fail(AT_EINVAL, "space_create: null pointer");
    if (n_workloads < 1 || n_workloads > at::MAXW) return at::fail(AT_EINVAL, "space_create: n_workloads not in [1,16]");
    *out = nullptr;
    at_space sp = new at_space_s();
    std::memset(&sp->host, 0, sizeof(sp->host));
    sp->d_space = nullptr;
    sp->d_fact = nullptr;
    sp->d_scratch = nullptr;
    sp->scratch_bytes = 0;
    sp->h_err = nullptr;
    Builder B;
    sp->host.n_w = n_workloads;
    uint64_t off = 0;
    for (int i = 0; i < n_workloads; ++i) {
        int rc = build_workload(w[i], sp->host.w[i], B);
        if (rc != AT_OK) { delete sp; return rc; }
        sp->host.w[i].offset = off;
        sp->host.offset[i] = off;
        off += sp->host.w[i].size;
    }
    sp->host.offset[n_workloads] = off;
    sp->total = off;
    if (B.fact.empty()) B.fact.push_back(0);
    // the range-error word: pinned, mapped (kernels store to it; the host reads it without a sync)
    if (cudaHostAlloc((void **)&sp->h_err, sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void **)&sp->host.err, sp->h_err, 0) != cudaSuccess) {
        cudaGetLastError();
        if (sp->h_err) cudaFreeHost(sp->h_err);
        delete sp;
        return at::fail(AT_ENOMEM, "space_create: mapped error word allocation failed");
    }
    *sp->h_err = 0u;
    if (cudaMalloc(&sp->d_space, sizeof(at::SpaceDev)) != cudaSuccess ||
        cudaMalloc(&sp->d_fact, B.fact.size() * sizeof(uint16_t)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(sp->d_space);
        cudaFreeHost(sp->h_err);
        delete sp;
        return at::fail(AT_ENOMEM, "space_create: device allocation failed");
    }
    cudaError_t e1 = cudaMemcpy(sp->d_space, &sp->host, sizeof(at::SpaceDev), cudaMemcpyHostToDevice);
    cudaError_t e2 = cudaMemcpy(sp->d_fact, B.fact.data(), B.fact.size() * sizeof(uint16_t), cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        cudaFree(sp->d_space);
        cudaFree(sp->d_fact);
        cudaFreeHost(sp->h_err);
        delete sp;
        return at::cuda_fail(e1 != cudaSuccess ? e1 : e2, "space_create upload");
    }
    *out = sp;
    return AT_OK;
}

int space_info(at_space sp, uint64_t *size_total, int32_t *n_workloads, int32_t *n_features, uint64_t *offsets,
               int32_t *radices)
{
    if (!sp) return at::fail(AT_EINVAL, "space_info: null space");
    if (size_total) *size_total = sp->total;
    if (n_workloads) *n_workloads = sp->host.n_w;
    if (n_features) *n_features = at::NFEAT;
    if (offsets)
        for (int i = 0; i <= sp->host.n_w; ++i) offsets[i] = sp->host.offset[i];
    if (radices)
        for (int i = 0; i < sp->host.n_w; ++i)
            for (int j = 0; j < at::MAXKNOBS; ++j)
                radices[i * at::MAXKNOBS + j] = j < sp->host.w[i].n_knobs ? (int32_t)sp->host.w[i].radix[j] : 0;
    return AT_OK;
}

int space_destroy(at_space sp)
{
    if (!sp) return AT_OK;
    cudaFree(sp->d_space);
    cudaFree(sp->d_fact);
    if (sp->d_scratch) cudaFree(sp->d_scratch);
    if (sp->h_err) cudaFreeHost(sp->h_err);
    delete sp;
    return AT_OK;
}

}  // extern "C"
