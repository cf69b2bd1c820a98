// walk_ceiling.cu -- microbenchmark of the GBT tree-walk inner loop on one B200 (sm_100a):
// the same node-step instruction pattern as gbt.cuh (LDS.64 node {feature, threshold}, IMAD to the
// feature's tile row, LDS feature, FSETP, SEL, IADD3), all data resident in shared memory, no
// barriers, NB independent walks per warp, W warps per block, one block per SM.  Reports lane
// node-steps per second and per SM clock: the achievable ceiling of the walk.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o walk_ceiling walk_ceiling.cu && ./walk_ceiling
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int D = 6, NI = (1 << D) - 1, T = 96, F = 468;

template <int NB>
__global__ void __launch_bounds__(1024, 1) walk_kernel(const uint2 *__restrict__ gnodes, int iters, unsigned long long *out)
{
    extern __shared__ __align__(16) unsigned char sm[];
    uint2 *nodes = (uint2 *)sm;                      // [T][NI]
    float *tile = (float *)(nodes + T * NI);         // [F][32]
    for (int i = threadIdx.x; i < T * NI; i += blockDim.x) nodes[i] = gnodes[i];
    for (int i = threadIdx.x; i < F * 32; i += blockDim.x) tile[i] = (float)((i * 2654435761u) >> 20);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t tile_lane = (uint32_t)__cvta_generic_to_shared(tile + lane);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(nodes);
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t a[NB], add_l[NB], add_r[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int t = (warp + (it * NB + j) * nw) % T;
            const uint32_t tb = base + (uint32_t)t * NI * 8u - 8u;
            add_l[j] = 0u - tb;
            add_r[j] = 8u - tb;
            a[j] = tb + 8u;
        }
#pragma unroll
        for (int d = 0; d < D; ++d) {
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                uint32_t nf, nt;
                float x;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nf), "=r"(nt) : "r"(a[j]));
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(tile_lane + (nf << 7)));
                a[j] = 2u * a[j] + (x < __uint_as_float(nt) ? add_l[j] : add_r[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < NB; ++j) acc += a[j] + add_l[j];
    }
    if (acc == 0x1234567ull) out[0] = acc;   // keep the walks alive
}

int main()
{
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    uint2 *h = new uint2[T * NI];
    for (int i = 0; i < T * NI; ++i) {
        const uint32_t f = (i * 2246822519u) % 466, th = (i * 3266489917u) >> 20;
        float thf = (float)th;
        h[i] = make_uint2(f, *(uint32_t *)&thf);
    }
    uint2 *g;
    unsigned long long *o;
    cudaMalloc(&g, sizeof(uint2) * T * NI);
    cudaMalloc(&o, 8);
    cudaMemcpy(g, h, sizeof(uint2) * T * NI, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(uint2) * T * NI + sizeof(float) * F * 32;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %d, \"results\": [\n", nsm, clk / 1000);
    bool first = true;
    auto run = [&](auto kern, int nb, int warps) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int iters = 2000;
        kern<<<nsm, warps * 32, smem>>>(g, 10, o);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        kern<<<nsm, warps * 32, smem>>>(g, iters, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (cudaGetLastError() != cudaSuccess) { printf("%s {\"NB\": %d, \"warps\": %d, \"error\": \"launch failed\"}", first ? " " : ",\n ", nb, warps); first = false; return; }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double steps = (double)nsm * warps * 32 * (double)iters * nb * D;
        printf("%s {\"NB\": %d, \"warps\": %d, \"ms\": %.3f, \"Gnode_steps_per_s\": %.1f, \"node_steps_per_clk_per_sm_at_1965\": %.2f}",
               first ? " " : ",\n ", nb, warps, ms, steps / ms / 1e6, steps / (ms * 1e-3) / nsm / 1.965e9);
        first = false;
    };
    run(walk_kernel<4>, 4, 16);
    run(walk_kernel<6>, 6, 16);
    run(walk_kernel<8>, 8, 16);
    run(walk_kernel<16>, 16, 16);
    run(walk_kernel<24>, 24, 16);
    run(walk_kernel<8>, 8, 24);
    run(walk_kernel<16>, 16, 24);
    run(walk_kernel<4>, 4, 32);
    run(walk_kernel<8>, 8, 32);
    run(walk_kernel<12>, 12, 32);
    printf("\n]}\n");
    return cudaGetLastError() != cudaSuccess;
}
