// cta_topk microbenchmark (development tool): one CTA per row selects k of n random scores
// held in shared memory; reports clock64 cycles per phase (CTA 0) and checks the result.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_12211_b200/csrc -o /tmp/selbench scripts/selbench.cu
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
__device__ long long g_prof[16];
#define TS_TOPK_PROF(i) if (threadIdx.x == 0 && blockIdx.x == 0) g_prof[i] = clock64();
#include "score_select.cuh"
using namespace ts;
template <int NT>
__global__ void __launch_bounds__(NT) bench(const float *scores, int n, int k, int *out, long long *cyc) {
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t *keys = sm;
    int *hist = reinterpret_cast<int *>(sm + ((n + 3) & ~3));
    int *red = hist + kSsHist;
    uint32_t *cand = reinterpret_cast<uint32_t *>(red + 64);
    long long t0 = clock64();
    const float *row = scores + (size_t)blockIdx.x * n;
    for (int i = threadIdx.x; i < kSsHist; i += NT) hist[i] = 0;
    uint32_t mn = 0xffffffffu, mx = 0;
    for (int i = threadIdx.x; i < ((n + 3) & ~3); i += NT) {
        const uint32_t key = i < n ? score_key(row[i]) : 0u;
        keys[i] = key;
        if (i < n) { mn = min(mn, key); mx = max(mx, key); }
    }
    __syncthreads();
    block_minmax<NT>(mn, mx, red);
    long long t1 = clock64();
    int *o = out + (size_t)blockIdx.x * k;
    const int kk = (n <= 512 ? cta_topk<NT, 0, 9>(keys, n, k, mn, mx, hist, red, cand, [&](int pos, int i) { o[pos] = i; }) : cta_topk<NT, 0, 11>(keys, n, k, mn, mx, hist, red, cand, [&](int pos, int i) { o[pos] = i; }));
    __syncthreads();
    long long t2 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = kk; }
}
int main() {
    for (auto cfg : std::vector<std::pair<int,int>>{{256, 32}, {2048, 128}, {8192, 64}}) {
        const int n = cfg.first, k = cfg.second, rows = 16;
        std::vector<float> h(rows * n);
        std::mt19937 rng(3); std::normal_distribution<float> nd(10.f, 3.f);
        for (auto &x : h) x = nd(rng);
        float *d; int *out; long long *cyc;
        cudaMalloc(&d, h.size() * 4); cudaMalloc(&out, rows * k * 4); cudaMalloc(&cyc, 64);
        cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        const size_t sm = ((n + 3) & ~3) * 4 + kSsHist * 4 + 64 * 4 + 512 + 64;
        cudaFuncSetAttribute(bench<160>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(bench<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int nt : {160, 512}) {
            for (int it = 0; it < 3; ++it) {
                if (nt == 160) bench<160><<<rows, 160, sm>>>(d, n, k, out, cyc);
                else bench<512><<<rows, 512, sm>>>(d, n, k, out, cyc);
            }
            long long c[3]; cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
            std::vector<int> o(k); cudaMemcpy(o.data(), out, k * 4, cudaMemcpyDeviceToHost);
            std::vector<int> idx(n); for (int i = 0; i < n; ++i) idx[i] = i;
            std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return h[a] > h[b]; });
            std::vector<int> ref(idx.begin(), idx.begin() + k); std::sort(ref.begin(), ref.end());
            long long pr[16]; cudaMemcpyFromSymbol(pr, g_prof, sizeof(pr));
            printf("   phases:"); for (int i = 1; i < 7; ++i) printf(" %d:%lld", i, pr[i] ? pr[i] - pr[0] : -1); printf("\n");
            cudaMemset(cyc, 0, 8); long long z[16] = {0}; cudaMemcpyToSymbol(g_prof, z, sizeof(z));
            printf("n %5d k %4d NT %3d: prep %6lld cyc, topk %6lld cyc, kk %lld, %s (%s)\n", n, k, nt, c[0], c[1], c[2],
                   ref == o ? "exact" : "MISMATCH", cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
