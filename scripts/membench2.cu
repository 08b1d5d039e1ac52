// Random-gather bandwidth vs chunk size (development tool): n_chunks random CB-byte chunks
// of K and of V (same total bytes for every CB), 128-bit loads, one warp per chunk pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membench2 scripts/membench2.cu
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

template <int CB>
__global__ void gather(const int4 *__restrict__ k, const int4 *__restrict__ v, const int *__restrict__ idx,
                       int n, int4 *out) {
    constexpr int PER = CB / 16 / 32 > 0 ? CB / 16 / 32 : 1;  // int4 per lane per chunk
    constexpr int LANES = CB / 16 < 32 ? CB / 16 : 32;
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    int4 acc = make_int4(0, 0, 0, 0);
    for (; w < n; w += (gridDim.x * blockDim.x) >> 5) {
        const size_t base = (size_t)idx[w] * (CB / 16);
        if (lane < LANES) {
            int4 a[2 * PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) a[i] = k[base + lane + 32 * i];
#pragma unroll
            for (int i = 0; i < PER; ++i) a[PER + i] = v[base + lane + 32 * i];
#pragma unroll
            for (int i = 0; i < 2 * PER; ++i) { acc.x ^= a[i].x; acc.y ^= a[i].y; }
        }
    }
    if (acc.x == 0x12345678) out[0] = acc;
}

template <int CB>
void run(size_t pool_bytes, size_t step_bytes) {
    const size_t chunks = pool_bytes / CB;
    const int n = (int)(step_bytes / 2 / CB);
    const int reps = 6;
    std::vector<int4 *> K(reps), V(reps);
    std::vector<int *> I(reps);
    std::mt19937 rng(1);
    for (int r = 0; r < reps; ++r) {
        cudaMalloc(&K[r], pool_bytes); cudaMemset(K[r], 1, pool_bytes);
        cudaMalloc(&V[r], pool_bytes); cudaMemset(V[r], 1, pool_bytes);
        std::vector<int> h(n);
        for (int i = 0; i < n; ++i) h[i] = rng() % chunks;
        cudaMalloc(&I[r], n * 4);
        cudaMemcpy(I[r], h.data(), n * 4, cudaMemcpyHostToDevice);
    }
    int4 *out; cudaMalloc(&out, 16);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {8, 16}) {
        const int grid = sms * bps;
        for (int i = 0; i < 20; ++i) gather<CB><<<grid, 256>>>(K[i % reps], V[i % reps], I[i % reps], n, out);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int iters = 60;
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) gather<CB><<<grid, 256>>>(K[i % reps], V[i % reps], I[i % reps], n, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / iters;
        printf("chunk %5d B x %6d x 2: %.2f us, %.0f GB/s (%d blk/SM)\n", CB, n, us, 2.0 * n * CB / us / 1e3, bps);
    }
    for (int r = 0; r < reps; ++r) { cudaFree(K[r]); cudaFree(V[r]); cudaFree(I[r]); }
}

int main() {
    const size_t pool = 512ull << 20, step = 128ull << 20;
    run<256>(pool, step); run<512>(pool, step); run<1024>(pool, step); run<2048>(pool, step); run<4096>(pool, step);
    return 0;
}
