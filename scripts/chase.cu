// Dependent-load latency vs working-set size (development tool): one thread chases a
// random cyclic permutation of 2 KB-strided slots over a region of `mb` MB; reports ns/hop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/chase scripts/chase.cu
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
__global__ void chase(const long long *p, long long start, int hops, long long *out, unsigned long long *ns) {
    long long i = start;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int h = 0; h < hops; ++h) i = __ldcg(p + i);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out = i;
    *ns = t1 - t0;
}
__global__ void flush(int4 *buf, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] = make_int4(i, 0, 0, 0);
}
int main() {
    const size_t stride = 2048 / 8;  // elements (2 KB)
    int4 *fb; size_t fbn = (512ull << 20) / 16; cudaMalloc(&fb, fbn * 16);
    long long *out; unsigned long long *ns; cudaMalloc(&out, 8); cudaMalloc(&ns, 8);
    for (size_t mb : {8, 64, 256, 1024, 4096, 16384}) {
        size_t n = (mb << 20) / 2048;
        long long *p; if (cudaMalloc(&p, (mb << 20)) != cudaSuccess) { printf("alloc fail %zu\n", mb); continue; }
        std::vector<long long> perm(n); for (size_t i = 0; i < n; ++i) perm[i] = i;
        std::mt19937_64 rng(1); std::shuffle(perm.begin() + 1, perm.end(), rng);
        std::vector<long long> h(n * stride, 0);
        for (size_t i = 0; i < n; ++i) h[perm[i] * stride] = perm[(i + 1) % n] * stride;
        cudaMemcpy(p, h.data(), n * stride * 8, cudaMemcpyHostToDevice);
        const int hops = 2000;
        for (int cold = 0; cold < 2; ++cold) {
            if (cold) flush<<<1184, 256>>>(fb, fbn);
            chase<<<1, 1>>>(p, 0, hops, out, ns);
            unsigned long long t; cudaMemcpy(&t, ns, 8, cudaMemcpyDeviceToHost);
            printf("%6zu MB %s: %.0f ns/hop\n", mb, cold ? "after L2 flush" : "warm-ish     ", (double)t / hops);
        }
        cudaFree(p);
    }
    return 0;
}
