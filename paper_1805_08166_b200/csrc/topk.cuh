// topk.cuh -- host interface of the distinct top-K reduction (topk.cu).
#pragma once
#include "at_common.cuh"

namespace at {

struct TkArgs {
    int mode;                    // 0 SA keys, 1 (idx, score) lists
    const uint64_t *keys;        // mode 0: [steps + 1][n_chains] keys (fkey(E) << 32 | local idx)
    int64_t n_src;
    int64_t n_chains;
    const uint16_t *chain_w;     // mode 0: workload of each chain (nullable)
    const int32_t *chain_list;   // mode 0, optional: the chains of workload w (any order) ...
    const int32_t *list_n;       // ... and their number (device): only those chains' keys are read
    int w;
    uint64_t offset_w;
    const uint64_t *l_idx;       // mode 1
    const float *l_score;
    const int32_t *l_n;
    int n_w, k_in;
    const uint64_t *measured;
    int64_t n_measured;
    int K;
    uint64_t *out_idx;
    float *out_score;
    int32_t *out_n;
};

size_t topk_scratch_bytes(int64_t n_src, int K, int n_batch = 1);
// chain lists per workload: list[w * n_chains + j], j < cnt[w] (cnt zeroed by the caller)
void topk_chain_lists(const uint16_t *chain_w, int64_t n_chains, int n_w, int32_t *list, int32_t *cnt, cudaStream_t s);
// n_batch > 1: workloads a.w .. a.w + n_batch - 1 in one launch per pass, outputs in consecutive
// rows; offsets[w] = each workload's global index offset (nullptr: a.offset_w for all)
int topk_run(const TkArgs &a, uint64_t *scratch, cudaStream_t s, int n_batch = 1, const uint64_t *offsets = nullptr,
             const int32_t *fb = nullptr);
// threshold fast path for SA keys (mode 0): settles most workloads in 4 short launches; a row it cannot
// settle gets fb[y] = 1, and topk_run(..., fb) then reduces that row alone (the others return at once)
size_t topk_fast_scratch_bytes(int n_batch);
int topk_fast(const TkArgs &a, int n_batch, const uint64_t *offsets, int64_t per, uint8_t *scratch, int32_t *fb,
              cudaStream_t s);

}  // namespace at
