// TMA / bulk-copy throughput microbenchmark (development tool).
// One producer lane per CTA streams CHUNK-byte cp.async.bulk copies of a contiguous (or
// randomly permuted) region into a STAGES-deep smem ring; one consumer warp waits on each
// stage's mbarrier and releases it.  Reports aggregate GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmabench scripts/tmabench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <stdint.h>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void *src, uint32_t n, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

template <int STAGES, int CONS, int LANES, int MODE>
__global__ void ringm(const char *src, const int *perm, long long nchunks, int chunk, unsigned long long *out) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) unsigned long long bars[2 * STAGES];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(bars), eb = fb + 8 * STAGES;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(fb + 8 * i, 1); mbar_init(eb + 8 * i, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long per = (nchunks + gridDim.x - 1) / gridDim.x;
    const long long c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
    const int n = (int)max(0LL, c1 - c0);
    if (warp == CONS) {
        for (int i0 = 0; i0 < n; i0 += LANES) {
            const int i = i0 + lane;
            const int mode = MODE;
            if (mode == 0) {  // lanes wait and issue
                if (lane < LANES && i < n) {
                    const int st = i % STAGES;
                    mbar_wait(eb + 8 * st, ((i / STAGES) & 1) ^ 1);
                    mbar_expect(fb + 8 * st, chunk);
                    const long long c = perm ? perm[c0 + i] : c0 + i;
                    bulk(sb + st * chunk, src + c * chunk, chunk, fb + 8 * st);
                }
            } else if (mode == 1) {  // lanes wait, lane 0 issues all
                if (lane < LANES && i < n) mbar_wait(eb + 8 * (i % STAGES), ((i / STAGES) & 1) ^ 1);
                __syncwarp();
                if (lane == 0)
                    for (int j = i0; j < min(n, i0 + LANES); ++j) {
                        const int st = j % STAGES;
                        mbar_expect(fb + 8 * st, chunk);
                        bulk(sb + st * chunk, src + (long long)(c0 + j) * chunk, chunk, fb + 8 * st);
                    }
            } else {  // lane 0 waits all, lanes issue
                if (lane == 0)
                    for (int j = i0; j < min(n, i0 + LANES); ++j)
                        mbar_wait(eb + 8 * (j % STAGES), ((j / STAGES) & 1) ^ 1);
                __syncwarp();
                if (lane < LANES && i < n) {
                    const int st = i % STAGES;
                    mbar_expect(fb + 8 * st, chunk);
                    bulk(sb + st * chunk, src + (long long)(c0 + i) * chunk, chunk, fb + 8 * st);
                }
            }
            __syncwarp();
        }
        return;
    }
    unsigned long long acc = 0;
    for (int i = warp; i < n; i += CONS) {
        const int st = i % STAGES;
        mbar_wait(fb + 8 * st, (i / STAGES) & 1);
        acc += smem[st * chunk + lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(eb + 8 * st);
    }
    if (acc == 0x1234567) out[0] = acc;
}

template <int STAGES, int CONS, int LANES, int MODE>
void runm(const char *src, const int *perm, size_t bytes, int chunk, int ctas_per_sm, int sms, unsigned long long *out, const char *tag) {
    const long long nchunks = bytes / chunk;
    const int smem = STAGES * chunk;
    cudaFuncSetAttribute(ringm<STAGES, CONS, LANES, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) ringm<STAGES, CONS, LANES, MODE><<<grid, (CONS + 1) * 32, smem>>>(src, perm, nchunks, chunk, out);
    cudaEventRecord(a);
    const int it = 50;
    for (int i = 0; i < it; ++i) ringm<STAGES, CONS, LANES, MODE><<<grid, (CONS + 1) * 32, smem>>>(src, perm, nchunks, chunk, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const cudaError_t e = cudaGetLastError();
    printf("mode %d %-6s multi-lane %d chunk %6d stages %2d ctas/SM %d: %8.1f GB/s (%s)\n", MODE, tag, LANES, chunk, STAGES, ctas_per_sm,
           bytes * (double)it / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
}

template <int STAGES, int CONS>
__global__ void ring(const char *src, const int *perm, long long nchunks, int chunk, unsigned long long *out) {
    extern __shared__ __align__(1024) char smem[];
    __shared__ __align__(8) unsigned long long bars[2 * STAGES];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(bars), eb = fb + 8 * STAGES;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(fb + 8 * i, 1); mbar_init(eb + 8 * i, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long per = (nchunks + gridDim.x - 1) / gridDim.x;
    const long long c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
    const int n = (int)max(0LL, c1 - c0);
    if (warp == CONS) {
        if (lane) return;
        for (int i = 0; i < n; ++i) {
            const int st = i % STAGES;
            mbar_wait(eb + 8 * st, ((i / STAGES) & 1) ^ 1);
            mbar_expect(fb + 8 * st, chunk);
            const long long c = perm ? perm[c0 + i] : c0 + i;
            bulk(sb + st * chunk, src + c * chunk, chunk, fb + 8 * st);
        }
        return;
    }
    unsigned long long acc = 0;
    for (int i = warp; i < n; i += CONS) {
        const int st = i % STAGES;
        mbar_wait(fb + 8 * st, (i / STAGES) & 1);
        acc += smem[st * chunk + lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(eb + 8 * st);
    }
    if (acc == 0x1234567) out[0] = acc;
}

template <int STAGES, int CONS>
void run(const char *src, const int *perm, size_t bytes, int chunk, int ctas_per_sm, int sms, unsigned long long *out, const char *tag) {
    const long long nchunks = bytes / chunk;
    const int smem = STAGES * chunk;
    cudaFuncSetAttribute(ring<STAGES, CONS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * ctas_per_sm;
    for (int i = 0; i < 3; ++i) ring<STAGES, CONS><<<grid, (CONS + 1) * 32, smem>>>(src, perm, nchunks, chunk, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    const int it = 10;
    for (int i = 0; i < it; ++i) ring<STAGES, CONS><<<grid, (CONS + 1) * 32, smem>>>(src, perm, nchunks, chunk, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const cudaError_t e = cudaGetLastError();
    printf("%-6s chunk %6d stages %2d ctas/SM %d: %8.1f GB/s (%s)\n", tag, chunk, STAGES, ctas_per_sm,
           bytes * (double)it / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
}

int main(int argc, char **argv) {
    if (argc > 1) {  // multi-lane issue stress
        const size_t bytes = 1ull << 30;
        char *src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
        unsigned long long *out; cudaMalloc(&out, 8);
        int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int m = atoi(argv[1]);
        if (m == 0) runm<16, 6, 8, 0>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 1) runm<16, 6, 8, 1>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 2) runm<16, 6, 8, 2>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 3) runm<16, 6, 1, 0>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 4) run<16, 6>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 5) runm<16, 4, 1, 0>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 6) run<16, 4>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        if (m == 7) runm<16, 4, 8, 0>(src, nullptr, bytes, 4096, 2, sms, out, "seq");
        return 0;
    }
    const size_t bytes = 1ull << 30;
    char *src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
    unsigned long long *out; cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int chunk : {2048, 4096, 8192, 16384}) {
        run<8, 4>(src, nullptr, bytes, chunk, 1, sms, out, "seq");
        run<8, 4>(src, nullptr, bytes, chunk, 2, sms, out, "seq");
        run<16, 4>(src, nullptr, bytes, chunk, 1, sms, out, "seq");
        if (chunk <= 8192) run<16, 4>(src, nullptr, bytes, chunk, 2, sms, out, "seq");
    }
    for (int chunk : {2048, 4096}) {
        const long long n = bytes / chunk;
        std::vector<int> h(n);
        for (long long i = 0; i < n; ++i) h[i] = (int)i;
        std::mt19937 rng(3);
        for (long long i = n - 1; i > 0; --i) std::swap(h[i], h[rng() % (i + 1)]);
        int *perm; cudaMalloc(&perm, n * 4);
        cudaMemcpy(perm, h.data(), n * 4, cudaMemcpyHostToDevice);
        run<16, 4>(src, perm, bytes, chunk, 1, sms, out, "random");
        run<16, 4>(src, perm, bytes, chunk, 2, sms, out, "random");
        run<32, 4>(src, perm, bytes, chunk, 1, sms, out, "random");
        cudaFree(perm);
    }
    return 0;
}
