// atomtest.cu — latency of a shared-memory histogram build until its counts are readable
// (development tool).  Variants: atomicAdd(+1), red.shared.add with a register value,
// atomicAdd with return, plain stores.  Clocks are read with the loaded count as an input
// operand, so they cannot move above the load.
#include <cstdio>
#include <vector>
#include <random>
__device__ long long g_t[148 * 8];
__device__ __forceinline__ long long clk_after(int v) {
    long long t;
    asm volatile("{ .reg .u32 tmp; mov.u32 tmp, %1; mov.u64 %0, %%clock64; }" : "=l"(t) : "r"(v) : "memory");
    return t;
}
__global__ void __launch_bounds__(160) k(const unsigned *keys_g, int n, int mode, int one) {
    __shared__ int hist[2048];
    __shared__ unsigned keys[2048];
    __shared__ int sink;
    for (int i = threadIdx.x; i < 2048; i += 160) { hist[i] = 0; keys[i] = keys_g[blockIdx.x * 2048 + i]; }
    __syncthreads();
    const long long t0 = clk_after(0);
    if (mode == 0) {
        for (int i = threadIdx.x; i < n; i += 160) atomicAdd(&hist[keys[i] & 2047], 1);
    } else if (mode == 1) {
        for (int i = threadIdx.x; i < n; i += 160) {
            const unsigned a = (unsigned)__cvta_generic_to_shared(&hist[keys[i] & 2047]);
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(one) : "memory");
        }
    } else if (mode == 2) {
        int acc = 0;
        for (int i = threadIdx.x; i < n; i += 160) acc += atomicAdd(&hist[keys[i] & 2047], 1);
        if (acc == -7) sink = acc;
    } else {
        for (int i = threadIdx.x; i < n; i += 160) hist[keys[i] & 2047] = 1;
    }
    const long long t1 = clk_after(0);
    __syncthreads();
    const long long t2 = clk_after(0);
    const int v = hist[(threadIdx.x * 16) & 2047];
    const long long t3 = clk_after(v);
    if (threadIdx.x == 0) { g_t[blockIdx.x * 8] = t1 - t0; g_t[blockIdx.x * 8 + 1] = t2 - t1; g_t[blockIdx.x * 8 + 2] = t3 - t2; }
}
int main() {
    std::mt19937 r(1);
    std::vector<unsigned> h(148 * 2048);
    for (auto &x : h) x = r();
    unsigned *d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const char *nm[4] = {"atomicAdd+1", "red.shared.add", "atomicAdd ret", "store"};
    for (int n : {256, 2048})
        for (int mode = 0; mode < 4; ++mode) {
            for (int it = 0; it < 3; ++it) k<<<148, 160>>>(d, n, mode, 1);
            cudaDeviceSynchronize();
            long long t[148 * 8]; cudaMemcpyFromSymbol(t, g_t, sizeof(t));
            double a = 0, b = 0, c = 0; for (int i = 0; i < 148; ++i) { a += t[i * 8]; b += t[i * 8 + 1]; c += t[i * 8 + 2]; }
            printf("n %4d %-15s issue %6.0f  bar %6.0f  first load %6.0f cycles\n", n, nm[mode], a / 148, b / 148, c / 148);
        }
}
