// Raw gather bandwidth of the sparse-attention access pattern (development tool):
// read N random 2 KB chunks (a (block, head) K tile and its V tile) with 128-bit loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench scripts/membench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void gather(const int4 *__restrict__ k, const int4 *__restrict__ v, const int *__restrict__ idx,
                       int n, int4 *out, int stride) {
    // one warp per chunk pair; each lane 4 x 16 B of K and of V
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    int4 acc = make_int4(0, 0, 0, 0);
    for (; w < n; w += (gridDim.x * blockDim.x) >> 5) {
        const size_t base = (size_t)idx[w] * stride;  // 2 KB = 128 int4 (stride 256: K and V adjacent)
        int4 a[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = k[base + lane + 32 * i];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[4 + i] = v[base + lane + 32 * i];
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc.x ^= a[i].x; acc.y ^= a[i].y; acc.z ^= a[i].z; acc.w ^= a[i].w; }
    }
    if (acc.x == 0x12345678) out[0] = acc;
}

int main(int argc, char **argv) {
    const size_t pool_chunks = argc > 1 ? atol(argv[1]) : 131072;  // 2 KB chunks per pool
    const int n = argc > 2 ? atoi(argv[2]) : 16384;                 // chunks per step
    const int reps = 6;
    const int inter = argc > 3 ? atoi(argv[3]) : 0;  // 1: K and V of an index adjacent (4 KB)
    std::vector<int4 *> K(reps), V(reps);
    std::vector<int *> I(reps);
    std::mt19937 rng(1);
    for (int r = 0; r < reps; ++r) {
        cudaMalloc(&K[r], pool_chunks * 2048 * (inter ? 2 : 1));
        cudaMemset(K[r], 1, pool_chunks * 2048 * (inter ? 2 : 1));
        if (inter) {
            V[r] = K[r] + 128;
        } else {
            cudaMalloc(&V[r], pool_chunks * 2048);
            cudaMemset(V[r], 1, pool_chunks * 2048);
        }
        std::vector<int> h(n);
        for (int i = 0; i < n; ++i) h[i] = rng() % pool_chunks;
        cudaMalloc(&I[r], n * 4);
        cudaMemcpy(I[r], h.data(), n * 4, cudaMemcpyHostToDevice);
    }
    int4 *out;
    cudaMalloc(&out, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int blocks_per_sm : {4, 8, 16}) {
        const int grid = sms * blocks_per_sm;
        for (int i = 0; i < 20; ++i) gather<<<grid, 256>>>(K[i % reps], V[i % reps], I[i % reps], n, out, inter ? 256 : 128);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int iters = 120;
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) gather<<<grid, 256>>>(K[i % reps], V[i % reps], I[i % reps], n, out, inter ? 256 : 128);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / iters;
        printf("gather %d x 4KB (pool %zu x 2KB, %s), %d blk/SM: %.2f us, %.0f GB/s\n", n, pool_chunks, inter ? "K|V adjacent" : "K, V separate",
               blocks_per_sm, us, n * 4096.0 / us / 1e3);
    }
    return 0;
}
